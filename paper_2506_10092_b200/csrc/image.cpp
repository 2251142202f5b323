// Column images: the reference's dump_column byte format (column.cpp:513-563)
// as the shard on-disk / wire format of device columns.
//
//   line 1: {"encoding":..,"total_size":..,"value_type":..,"widths":{"value":W,
//            "position":8}, + per-encoding counts / storage / center}\n
//   body  : the column's arrays back to back, in the reference's order
//           plain v | rle v s e | index v p | plain+index base v2 p2 |
//           rle+index v s e v2 p2
//
// rq_col_dump_image downloads a device column into one malloc'd image;
// rq_col_load_image parses the header and uploads the body sections straight
// from the image (no host re-layout).
#include <cstdlib>
#include <cstring>
#include <string>

#include "rq_internal.hpp"

namespace rqb {
namespace {

const char* enc_name(int e) {
  switch (e) {
    case RQ_ENC_PLAIN: return "plain";
    case RQ_ENC_RLE: return "rle";
    case RQ_ENC_INDEX: return "index";
    case RQ_ENC_PLAIN_INDEX: return "plain+index";
    case RQ_ENC_RLE_INDEX: return "rle+index";
    default: return "?";
  }
}

const char* dt_name(int d) {  // dtype.hpp:27-37
  static const char* names[] = {"i8", "i16", "i32", "i64", "f32", "f64"};
  return d >= 0 && d < 6 ? names[d] : "?";
}

int dt_from_name(const std::string& s) {
  for (int d = 0; d < 6; ++d)
    if (s == dt_name(d)) return d;
  fail("column image: unknown dtype '" + s + "'");
  return -1;
}

int enc_from_name(const std::string& s) {
  for (int e = 0; e <= RQ_ENC_RLE_INDEX; ++e)
    if (s == enc_name(e)) return e;
  fail("column image: unknown encoding '" + s + "'");
  return -1;
}

// flat lookups in the one-line header (keys are unique in it)
bool hdr_find(const std::string& h, const std::string& key, size_t& at) {
  const std::string pat = "\"" + key + "\":";
  const size_t p = h.find(pat);
  if (p == std::string::npos) return false;
  at = p + pat.size();
  return true;
}
std::string hdr_str(const std::string& h, const std::string& key) {
  size_t at;
  if (!hdr_find(h, key, at) || at >= h.size() || h[at] != '"') fail("column image: header lacks \"" + key + "\"");
  const size_t end = h.find('"', at + 1);
  if (end == std::string::npos) fail("column image: unterminated string");
  return h.substr(at + 1, end - at - 1);
}
bool hdr_int(const std::string& h, const std::string& key, int64_t& v) {
  size_t at;
  if (!hdr_find(h, key, at)) return false;
  char* end = nullptr;
  v = std::strtoll(h.c_str() + at, &end, 10);
  if (end == h.c_str() + at) fail("column image: bad integer for \"" + key + "\"");
  return true;
}
int64_t hdr_req(const std::string& h, const std::string& key) {
  int64_t v = 0;
  if (!hdr_int(h, key, v)) fail("column image: header lacks \"" + key + "\"");
  return v;
}

}  // namespace
}  // namespace rqb

using namespace rqb;

extern "C" {

int rq_col_dump_image(rq_ctx_t c, rq_col_t col, void** out, int64_t* nbytes) {
  rq_host_column h{};
  int st = rq_col_describe(col, &h);
  if (st) return st;
  return api_guard([&] {
    require(out != nullptr && nbytes != nullptr, "null argument");
    const int vt = h.encoding == RQ_ENC_PLAIN || h.encoding == RQ_ENC_PLAIN_INDEX ? h.logical : h.dtype;
    std::string hdr = std::string("{\"encoding\":\"") + enc_name(h.encoding) + "\"" +
                      ",\"total_size\":" + std::to_string(h.total_size) + ",\"value_type\":\"" + dt_name(vt) + "\"" +
                      ",\"widths\":{\"value\":" + std::to_string(dt_width(vt)) + ",\"position\":8}";
    const int64_t w = dt_width(h.dtype), w2 = dt_width(h.dtype2);
    int64_t body = 0;
    switch (h.encoding) {
      case RQ_ENC_PLAIN:
        hdr += std::string(",\"storage\":\"") + dt_name(h.dtype) + "\"";
        if (h.has_center) hdr += ",\"center\":" + std::to_string(h.center);
        body = h.n * w;
        break;
      case RQ_ENC_RLE:
        hdr += ",\"runs\":" + std::to_string(h.n);
        body = h.n * (w + 16);
        break;
      case RQ_ENC_INDEX:
        hdr += ",\"points\":" + std::to_string(h.n);
        body = h.n * (w + 8);
        break;
      case RQ_ENC_PLAIN_INDEX:
        hdr += std::string(",\"storage\":\"") + dt_name(h.dtype) + "\",\"outliers\":" + std::to_string(h.n2);
        if (h.has_center) hdr += ",\"center\":" + std::to_string(h.center);
        body = h.n * w + h.n2 * (w2 + 8);
        break;
      default:
        hdr += ",\"runs\":" + std::to_string(h.n) + ",\"points\":" + std::to_string(h.n2);
        body = h.n * (w + 16) + h.n2 * (w2 + 8);
        break;
    }
    hdr += "}\n";
    const int64_t total = static_cast<int64_t>(hdr.size()) + body;
    char* img = static_cast<char*>(std::malloc(static_cast<size_t>(total > 0 ? total : 1)));
    require(img != nullptr, "column image: host allocation failed");
    std::memcpy(img, hdr.data(), hdr.size());
    char* p = img + hdr.size();
    auto take = [&](int64_t bytes) {
      char* q = p;
      p += bytes;
      return q;
    };
    h.v = take(h.n * w);
    if (h.encoding == RQ_ENC_RLE || h.encoding == RQ_ENC_RLE_INDEX) {
      h.s = reinterpret_cast<int64_t*>(take(h.n * 8));
      h.e = reinterpret_cast<int64_t*>(take(h.n * 8));
    } else if (h.encoding == RQ_ENC_INDEX) {
      h.p = reinterpret_cast<int64_t*>(take(h.n * 8));
    }
    if (h.encoding == RQ_ENC_PLAIN_INDEX || h.encoding == RQ_ENC_RLE_INDEX) {
      h.v2 = take(h.n2 * w2);
      h.p2 = reinterpret_cast<int64_t*>(take(h.n2 * 8));
    }
    const int rc = rq_col_download(c, col, &h);
    if (rc) {
      std::free(img);
      fail(rq_last_error());
    }
    *out = img;
    *nbytes = total;
  });
}

int rq_col_load_image(rq_ctx_t c, const void* image, int64_t nbytes, rq_col_t* out) {
  rq_host_column h{};
  int rc = api_guard([&] {
    require(image != nullptr && out != nullptr && nbytes > 0, "column image: null or empty");
    const char* b = static_cast<const char*>(image);
    const void* nl = std::memchr(b, '\n', static_cast<size_t>(nbytes));
    require(nl != nullptr, "column image: no header line");
    const std::string hdr(b, static_cast<const char*>(nl) - b);
    const char* p = static_cast<const char*>(nl) + 1;
    const char* end = b + nbytes;
    h.encoding = enc_from_name(hdr_str(hdr, "encoding"));
    h.total_size = hdr_req(hdr, "total_size");
    const int vt = dt_from_name(hdr_str(hdr, "value_type"));
    require(hdr_req(hdr, "position") == 8, "column image: positions must be 8 bytes");
    int64_t center = 0;
    h.has_center = hdr_int(hdr, "center", center) ? 1 : 0;
    h.center = center;
    auto take = [&](int64_t bytes) {
      require(bytes >= 0 && end - p >= bytes, "column image: body shorter than its header says");
      const char* q = p;
      p += bytes;
      return const_cast<char*>(q);
    };
    switch (h.encoding) {
      case RQ_ENC_PLAIN:
        h.dtype = dt_from_name(hdr_str(hdr, "storage"));
        h.logical = vt;
        h.n = h.total_size;
        h.v = take(h.n * dt_width(h.dtype));
        break;
      case RQ_ENC_RLE:
      case RQ_ENC_RLE_INDEX:
        h.dtype = h.logical = vt;
        h.n = hdr_req(hdr, "runs");
        h.v = take(h.n * dt_width(vt));
        h.s = reinterpret_cast<int64_t*>(take(h.n * 8));
        h.e = reinterpret_cast<int64_t*>(take(h.n * 8));
        if (h.encoding == RQ_ENC_RLE_INDEX) {
          h.dtype2 = vt;
          h.n2 = hdr_req(hdr, "points");
          h.v2 = take(h.n2 * dt_width(vt));
          h.p2 = reinterpret_cast<int64_t*>(take(h.n2 * 8));
        }
        break;
      case RQ_ENC_INDEX:
        h.dtype = h.logical = vt;
        h.n = hdr_req(hdr, "points");
        h.v = take(h.n * dt_width(vt));
        h.p = reinterpret_cast<int64_t*>(take(h.n * 8));
        break;
      default:  // plain+index: outliers in the logical dtype
        h.dtype = dt_from_name(hdr_str(hdr, "storage"));
        h.logical = h.dtype2 = vt;
        h.n = h.total_size;
        h.n2 = hdr_req(hdr, "outliers");
        h.v = take(h.n * dt_width(h.dtype));
        h.v2 = take(h.n2 * dt_width(vt));
        h.p2 = reinterpret_cast<int64_t*>(take(h.n2 * 8));
        break;
    }
    require(p == end, "column image: trailing bytes after the body");
  });
  if (rc) return rc;
  return rq_col_upload(c, &h, out);
}

void rq_image_free(void* image) { std::free(image); }

}  // extern "C"
