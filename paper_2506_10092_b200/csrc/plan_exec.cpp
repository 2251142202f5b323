// plan_exec.cpp — the query runner on the device (§8f row 4).
//
// Restates runq::query (plan.cpp:13-105 parse_plan_json, runner.cpp:86-373
// Exec::eval / Exec::dispatch / materialize) over the device operators of
// this library: every plan node keeps its columns resident in HBM (no
// decompression between nodes), string literals resolve against the column's
// dictionary (runner.cpp:106-112), joins recode dictionaries (runner.cpp:
// 198-226), and the plan shape the runner spends its time in — a GroupAgg
// over a Filter over a Scan — is recognised and run as ONE fused call
// (group_aggregate_exprs with the WHERE conjuncts pushed into the segment
// construction) when its predicate and aggregate expressions fit; any other
// shape runs node by node exactly as Exec does. Result columns are
// materialised as decoded rows (materialize, runner.cpp:354-373).
//
// The JSON reader accepts what plan.cpp reads (objects, arrays, strings,
// integers, floats, booleans, null).
#include <algorithm>
#include <cctype>
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <map>
#include <memory>
#include <optional>
#include <string>
#include <unordered_map>
#include <vector>

#include "rq_internal.hpp"

namespace rqb {
namespace planx {

inline void req(bool ok, const std::string& msg) {
  if (!ok) fail(msg);
}

// ---- JSON -------------------------------------------------------------------

struct J {
  enum Kind { NUL, BOOL, INT, FLT, STR, ARR, OBJ } k = NUL;
  bool b = false;
  int64_t i = 0;
  double f = 0.0;
  std::string s;
  std::vector<J> a;
  std::vector<std::pair<std::string, J>> o;
  const J* get(const std::string& key) const {
    for (const auto& kv : o)
      if (kv.first == key) return &kv.second;
    return nullptr;
  }
  const J& at(const std::string& key) const {
    const J* v = get(key);
    req(v != nullptr, "plan: missing field '" + key + "'");
    return *v;
  }
  const std::string& str() const {
    require(k == STR, "plan: expected a string");
    return s;
  }
};

struct JsonReader {
  const std::string& t;
  size_t p = 0;
  explicit JsonReader(const std::string& text) : t(text) {}
  void ws() {
    while (p < t.size() && (t[p] == ' ' || t[p] == '\n' || t[p] == '\t' || t[p] == '\r')) ++p;
  }
  char peek() {
    ws();
    require(p < t.size(), "plan: unexpected end of JSON");
    return t[p];
  }
  void expect(char c) {
    req(peek() == c, std::string("plan: expected '") + c + "' in JSON");
    ++p;
  }
  std::string string_lit() {
    expect('"');
    std::string out;
    while (true) {
      require(p < t.size(), "plan: unterminated string");
      char c = t[p++];
      if (c == '"') break;
      if (c == '\\') {
        require(p < t.size(), "plan: bad escape");
        char e = t[p++];
        switch (e) {
          case 'n': out += '\n'; break;
          case 't': out += '\t'; break;
          case 'r': out += '\r'; break;
          case 'b': out += '\b'; break;
          case 'f': out += '\f'; break;
          case 'u': {
            require(p + 4 <= t.size(), "plan: bad \\u escape");
            const unsigned cp = static_cast<unsigned>(std::strtoul(t.substr(p, 4).c_str(), nullptr, 16));
            p += 4;
            if (cp < 0x80) {
              out += static_cast<char>(cp);
            } else if (cp < 0x800) {
              out += static_cast<char>(0xc0 | (cp >> 6));
              out += static_cast<char>(0x80 | (cp & 0x3f));
            } else {
              out += static_cast<char>(0xe0 | (cp >> 12));
              out += static_cast<char>(0x80 | ((cp >> 6) & 0x3f));
              out += static_cast<char>(0x80 | (cp & 0x3f));
            }
            break;
          }
          default: out += e;
        }
      } else {
        out += c;
      }
    }
    return out;
  }
  J value() {
    const char c = peek();
    J v;
    if (c == '{') {
      ++p;
      v.k = J::OBJ;
      if (peek() == '}') {
        ++p;
        return v;
      }
      while (true) {
        std::string key = string_lit();
        expect(':');
        v.o.emplace_back(std::move(key), value());
        if (peek() == ',') {
          ++p;
          continue;
        }
        expect('}');
        return v;
      }
    }
    if (c == '[') {
      ++p;
      v.k = J::ARR;
      if (peek() == ']') {
        ++p;
        return v;
      }
      while (true) {
        v.a.push_back(value());
        if (peek() == ',') {
          ++p;
          continue;
        }
        expect(']');
        return v;
      }
    }
    if (c == '"') {
      v.k = J::STR;
      v.s = string_lit();
      return v;
    }
    if (t.compare(p, 4, "true") == 0) {
      p += 4;
      v.k = J::BOOL;
      v.b = true;
      return v;
    }
    if (t.compare(p, 5, "false") == 0) {
      p += 5;
      v.k = J::BOOL;
      return v;
    }
    if (t.compare(p, 4, "null") == 0) {
      p += 4;
      return v;
    }
    // number: integer unless it has a fraction or exponent (nlohmann's split)
    const size_t start = p;
    if (t[p] == '-' || t[p] == '+') ++p;
    bool flt = false;
    while (p < t.size() && (std::isdigit(static_cast<unsigned char>(t[p])) || t[p] == '.' || t[p] == 'e' ||
                            t[p] == 'E' || ((t[p] == '-' || t[p] == '+') && (t[p - 1] == 'e' || t[p - 1] == 'E')))) {
      if (t[p] == '.' || t[p] == 'e' || t[p] == 'E') flt = true;
      ++p;
    }
    require(p > start, "plan: invalid JSON value");
    const std::string num = t.substr(start, p - start);
    if (flt) {
      v.k = J::FLT;
      v.f = std::strtod(num.c_str(), nullptr);
    } else {
      v.k = J::INT;
      v.i = std::strtoll(num.c_str(), nullptr, 10);
    }
    return v;
  }
};

// ---- plan (plan.hpp:13-80) ----------------------------------------------------

struct Expr;
using ExprP = std::shared_ptr<const Expr>;
struct Expr {
  enum Kind { COL, LIT, BIN, NOT } k = COL;
  std::string name;  // COL: column; BIN: operator spelling
  int lit = 0;       // LIT: 0 int, 1 float, 2 string
  int64_t li = 0;
  double lf = 0.0;
  std::string ls;
  ExprP l, r;  // BIN: lhs / rhs; NOT: l
};

struct Node;
using NodeP = std::shared_ptr<const Node>;
struct Agg {
  int fn = RQ_SUM;
  ExprP expr;  // null: count(*)
  std::string name;
};
struct Node {
  enum Kind { SCAN, FILTER, PROJECT, JOIN, GROUP } k = SCAN;
  std::string table;
  std::vector<std::string> columns;
  ExprP pred;
  std::vector<std::pair<ExprP, std::string>> items;
  NodeP input, left, right;
  std::string left_on, right_on;
  bool semi = false;
  std::vector<std::string> keys;
  std::vector<Agg> aggs;
};

int agg_from_name(const std::string& n) {  // groupby.cpp:9-18
  if (n == "sum") return RQ_SUM;
  if (n == "count") return RQ_COUNT;
  if (n == "min") return RQ_MIN;
  if (n == "max") return RQ_MAX;
  if (n == "avg") return RQ_AVG;
  if (n == "std") return RQ_STD;
  if (n == "var") return RQ_VAR;
  fail("unknown aggregate function: " + n);
}

int binop_from_name(const std::string& n) {  // align.cpp:258-270
  if (n == "+") return RQ_ADD;
  if (n == "-") return RQ_SUB;
  if (n == "*") return RQ_MUL;
  if (n == "/") return RQ_DIV;
  if (n == "<") return RQ_LT;
  if (n == "<=") return RQ_LE;
  if (n == "==" || n == "=") return RQ_EQ;
  if (n == "!=" || n == "<>") return RQ_NE;
  if (n == ">=") return RQ_GE;
  if (n == ">") return RQ_GT;
  fail("unknown operator: " + n);
}

ExprP parse_expr(const J& j) {  // plan.cpp:13-32
  require(j.k == J::OBJ, "expression must be a JSON object");
  auto e = std::make_shared<Expr>();
  if (const J* c = j.get("col")) {
    e->k = Expr::COL;
    e->name = c->str();
    return e;
  }
  if (const J* v = j.get("lit")) {
    e->k = Expr::LIT;
    if (v->k == J::INT) {
      e->lit = 0;
      e->li = v->i;
    } else if (v->k == J::FLT) {
      e->lit = 1;
      e->lf = v->f;
    } else if (v->k == J::STR) {
      e->lit = 2;
      e->ls = v->s;
    } else {
      fail("literal must be a number or string");
    }
    return e;
  }
  require(j.get("op") != nullptr, "expression needs col, lit, or op");
  const std::string op = j.at("op").str();
  if (op == "not") {
    e->k = Expr::NOT;
    e->l = parse_expr(j.at("arg"));
    return e;
  }
  e->k = Expr::BIN;
  e->name = op;
  e->l = parse_expr(j.at("lhs"));
  e->r = parse_expr(j.at("rhs"));
  return e;
}

std::vector<std::string> strings(const J& j) {
  require(j.k == J::ARR, "plan: expected an array of strings");
  std::vector<std::string> out;
  for (const auto& x : j.a) out.push_back(x.str());
  return out;
}

NodeP parse_node(const J& j) {  // plan.cpp:34-92
  require(j.k == J::OBJ && j.get("node"), "plan node needs a 'node' field");
  const std::string kind = j.at("node").str();
  auto n = std::make_shared<Node>();
  if (kind == "scan") {
    n->k = Node::SCAN;
    n->table = j.at("table").str();
    if (const J* c = j.get("columns")) n->columns = strings(*c);
  } else if (kind == "filter") {
    n->k = Node::FILTER;
    n->pred = parse_expr(j.at("pred"));
    n->input = parse_node(j.at("input"));
  } else if (kind == "project") {
    n->k = Node::PROJECT;
    for (const auto& it : j.at("exprs").a) n->items.emplace_back(parse_expr(it.at("expr")), it.at("as").str());
    n->input = parse_node(j.at("input"));
  } else if (kind == "join") {
    n->k = Node::JOIN;
    n->left = parse_node(j.at("left"));
    n->right = parse_node(j.at("right"));
    n->left_on = j.at("on").at("left").str();
    n->right_on = j.at("on").at("right").str();
    if (const J* kd = j.get("kind")) {
      req(kd->str() == "inner" || kd->str() == "semi", "join kind must be inner or semi: " + kd->str());
      n->semi = kd->str() == "semi";
    }
  } else if (kind == "group_agg") {
    n->k = Node::GROUP;
    if (const J* k = j.get("keys")) n->keys = strings(*k);
    for (const auto& a : j.at("aggs").a) {
      Agg g;
      g.fn = agg_from_name(a.at("fn").str());
      if (const J* x = a.get("expr")) g.expr = parse_expr(*x);
      else require(g.fn == RQ_COUNT, "only count may omit expr");
      g.name = a.at("as").str();
      n->aggs.push_back(std::move(g));
    }
    require(!n->aggs.empty(), "group_agg needs at least one aggregate");
    n->input = parse_node(j.at("input"));
  } else {
    fail("unknown plan node kind: " + kind);
  }
  return n;
}

}  // namespace planx

// ---- catalog ------------------------------------------------------------------

struct DictD {  // runq::Dictionary (dictionary.hpp:16-43): codes in first-occurrence order
  std::vector<std::string> s;
  std::unordered_map<std::string, int64_t> code;
  std::optional<int64_t> find(const std::string& x) const {
    auto it = code.find(x);
    if (it == code.end()) return std::nullopt;
    return it->second;
  }
};
using DictP = std::shared_ptr<const DictD>;

struct CatColD {
  std::string name;
  std::shared_ptr<const DCol> col;
  DictP dict;
  bool is_date = false;
};
struct TableD {
  std::string name;
  int64_t rows = 0;
  std::vector<CatColD> cols;
};
struct CatalogD {
  std::vector<TableD> tables;
  const TableD& at(const std::string& n) const {
    for (const auto& t : tables)
      if (t.name == n) return t;
    fail("no table named " + n);
  }
};

struct ResultD {  // runq::query::ResultTable (runner.hpp:42-48)
  std::vector<std::string> names;
  std::vector<DictP> dicts;
  std::vector<DArr> columns;
  int64_t rows = 0;
  int fused = 0;  // GroupAgg nodes run through the fused call
};

namespace planx {

struct CCol {
  std::string name;
  std::shared_ptr<const DCol> col;
  DictP dict;
  bool is_date = false;
};
struct CSet {
  int64_t rows = 0;
  std::vector<CCol> cols;
  const CCol& at(const std::string& n) const {
    for (const auto& c : cols)
      if (c.name == n) return c;
    fail("no column named " + n);
  }
};
struct EvalV {
  std::shared_ptr<const DCol> col;
  std::shared_ptr<DMask> mask;
  bool has_scalar = false;
  Scalar scalar;
  DictP dict;
  bool is_date = false;
  bool is_col() const { return col != nullptr; }
};

int64_t days_from_civil(int64_t y, unsigned m, unsigned d) {  // proleptic Gregorian, 1970-01-01 = 0
  y -= m <= 2;
  const int64_t era = (y >= 0 ? y : y - 399) / 400;
  const unsigned yoe = static_cast<unsigned>(y - era * 400);
  const unsigned doy = (153 * (m + (m > 2 ? -3 : 9)) + 2) / 5 + d - 1;
  const unsigned doe = yoe * 365 + yoe / 4 - yoe / 100 + doy;
  return era * 146097 + static_cast<int64_t>(doe) - 719468;
}

int64_t parse_date_literal(const std::string& tok) {  // ingest.cpp:72-89
  auto bad = [&]() { fail("parse error at row -1, column 0: not a date (YYYY-MM-DD): '" + tok + "'"); };
  if (tok.size() != 10 || tok[4] != '-' || tok[7] != '-') bad();
  for (size_t i : {0, 1, 2, 3, 5, 6, 8, 9})
    if (!std::isdigit(static_cast<unsigned char>(tok[i]))) bad();
  const int y = std::atoi(tok.substr(0, 4).c_str()), m = std::atoi(tok.substr(5, 2).c_str()),
            d = std::atoi(tok.substr(8, 2).c_str());
  static const int mdays[] = {31, 28, 31, 30, 31, 30, 31, 31, 30, 31, 30, 31};
  const bool leap = (y % 4 == 0 && y % 100 != 0) || y % 400 == 0;
  if (m < 1 || m > 12 || d < 1 || d > mdays[m - 1] + (m == 2 && leap ? 1 : 0)) bad();
  return days_from_civil(y, static_cast<unsigned>(m), static_cast<unsigned>(d));
}

Scalar resolve_string_literal(const std::string& s, const EvalV& col_side) {  // runner.cpp:106-112
  Scalar k;
  if (col_side.is_date) {
    k.i = parse_date_literal(s);
    return k;
  }
  req(col_side.dict != nullptr, "string literal '" + s + "' compared against a non-string column");
  k.i = col_side.dict->find(s).value_or(-1);
  return k;
}

DCol recode_column(const CtxPtr& ctx, const DCol& col, const DictD& from, const DictD& to) {  // runner.cpp:198-226
  std::vector<int64_t> xlat(from.s.size());
  for (size_t c = 0; c < from.s.size(); ++c) xlat[c] = to.find(from.s[c]).value_or(-1);
  DArr table = upload_arr(ctx, RQ_I64, xlat.data(), static_cast<int64_t>(xlat.size()));
  auto remap = [&](const DArr& v) { return gather(ctx, table, cast_values(ctx, v, RQ_I64)); };
  switch (col.enc) {
    case RQ_ENC_PLAIN: {
      DCol out;
      out.enc = RQ_ENC_PLAIN;
      out.v = remap(decode_plain(ctx, col));
      out.logical = RQ_I64;
      out.total = col.total;
      return out;
    }
    case RQ_ENC_RLE:
    case RQ_ENC_INDEX: {
      DCol out = col;
      out.v = remap(col.v);
      return out;
    }
    default: return recode_column(ctx, normalize_basic(ctx, col), from, to);
  }
}

struct Exec {
  const CtxPtr& ctx;
  const CatalogD& cat;
  int fused = 0;

  EvalV eval(const CSet& ds, const Expr& e);
  std::shared_ptr<DMask> eval_mask(const CSet& ds, const Expr& e) {
    EvalV v = eval(ds, e);
    require(v.mask != nullptr, "predicate must be boolean");
    return v.mask;
  }
  CSet run(const Node& n);
  bool try_fused_group(const Node& n, CSet& out);
};

EvalV Exec::eval(const CSet& ds, const Expr& e) {  // runner.cpp:114-193
  EvalV v;
  if (e.k == Expr::COL) {
    const CCol& c = ds.at(e.name);
    v.col = c.col;
    v.dict = c.dict;
    v.is_date = c.is_date;
    return v;
  }
  if (e.k == Expr::LIT) {
    if (e.lit == 0) {
      v.has_scalar = true;
      v.scalar.i = e.li;
    } else if (e.lit == 1) {
      v.has_scalar = true;
      v.scalar.is_float = true;
      v.scalar.f = e.lf;
    }
    return v;  // string literal: resolved by the parent
  }
  if (e.k == Expr::NOT) {
    std::shared_ptr<DMask> a = eval_mask(ds, *e.l);
    v.mask = std::make_shared<DMask>(mask_not(ctx, *a));
    return v;
  }
  if (e.name == "and" || e.name == "or") {
    std::shared_ptr<DMask> l = eval_mask(ds, *e.l);
    std::shared_ptr<DMask> r = eval_mask(ds, *e.r);
    v.mask = std::make_shared<DMask>(e.name == "and" ? mask_and(ctx, *l, *r) : mask_or(ctx, *l, *r));
    return v;
  }
  EvalV l = eval(ds, *e.l);
  EvalV r = eval(ds, *e.r);
  const int op = binop_from_name(e.name);
  if (e.l->k == Expr::LIT && e.l->lit == 2) {
    require(r.is_col(), "string literal needs a column operand");
    l.scalar = resolve_string_literal(e.l->ls, r);
    l.has_scalar = true;
  }
  if (e.r->k == Expr::LIT && e.r->lit == 2) {
    require(l.is_col(), "string literal needs a column operand");
    r.scalar = resolve_string_literal(e.r->ls, l);
    r.has_scalar = true;
  }
  const bool cmp = op >= RQ_LT;
  auto col_result = [&](DCol c) { v.col = std::make_shared<DCol>(std::move(c)); };
  if (l.is_col() && r.is_col()) {
    if (cmp) v.mask = std::make_shared<DMask>(compare(ctx, *l.col, *r.col, op));
    else col_result(arith(ctx, *l.col, *r.col, op));
  } else if (l.is_col() && r.has_scalar) {
    if (cmp) v.mask = std::make_shared<DMask>(compare_scalar(ctx, *l.col, r.scalar, op, false));
    else col_result(arith_scalar(ctx, *l.col, r.scalar, op, false));
  } else if (l.has_scalar && r.is_col()) {
    if (cmp) v.mask = std::make_shared<DMask>(compare_scalar(ctx, *r.col, l.scalar, op, true));
    else col_result(arith_scalar(ctx, *r.col, l.scalar, op, true));
  } else {
    fail("expression must reference at least one column");
  }
  return v;
}

// WHERE → conjuncts `col op k` / `col IN (...)` over the scan's columns
// (and-trees of comparisons; an or-tree of equalities on one column).
bool to_conjuncts(const Expr& e, const CSet& in, std::vector<XPred>& out) {
  if (e.k == Expr::BIN && e.name == "and") return to_conjuncts(*e.l, in, out) && to_conjuncts(*e.r, in, out);
  auto col_lit = [&](const Expr& x, const CCol*& c, Scalar& k, int& op) -> bool {
    if (x.k != Expr::BIN || x.name == "and" || x.name == "or") return false;
    op = binop_from_name(x.name);
    if (op < RQ_LT) return false;
    const Expr* ce = x.l.get();
    const Expr* le = x.r.get();
    bool rev = false;
    if (ce->k != Expr::COL) {
      std::swap(ce, le);
      rev = true;
    }
    if (ce->k != Expr::COL || le->k != Expr::LIT) return false;
    c = &in.at(ce->name);
    EvalV side;
    side.dict = c->dict;
    side.is_date = c->is_date;
    if (le->lit == 2) k = resolve_string_literal(le->ls, side);
    else if (le->lit == 1) k.is_float = true, k.f = le->lf;
    else k.i = le->li;
    if (rev) {  // k op col  ==  col op' k
      switch (op) {
        case RQ_LT: op = RQ_GT; break;
        case RQ_LE: op = RQ_GE; break;
        case RQ_GT: op = RQ_LT; break;
        case RQ_GE: op = RQ_LE; break;
        default: break;
      }
    }
    return true;
  };
  const CCol* c = nullptr;
  Scalar k;
  int op = 0;
  if (col_lit(e, c, k, op)) {
    XPred q;
    q.col = c->col.get();
    q.op = op;
    q.k = k;
    out.push_back(q);
    return true;
  }
  if (e.k == Expr::BIN && e.name == "or") {  // IN-list: equalities on one column
    std::vector<const Expr*> st{&e}, leaves;
    while (!st.empty()) {
      const Expr* x = st.back();
      st.pop_back();
      if (x->k == Expr::BIN && x->name == "or") {
        st.push_back(x->r.get());
        st.push_back(x->l.get());
      } else {
        leaves.push_back(x);
      }
    }
    XPred q;
    for (const Expr* x : leaves) {
      const CCol* cc = nullptr;
      Scalar kk;
      int o = 0;
      if (!col_lit(*x, cc, kk, o) || o != RQ_EQ) return false;
      if (q.col && q.col != cc->col.get()) return false;
      q.col = cc->col.get();
      q.in.push_back(kk);
    }
    out.push_back(q);
    return true;
  }
  return false;
}

// aggregate expression → left-deep chain of ≤ 3 terms (col / col op lit / lit op col)
bool to_xexpr(const Expr& e, const CSet& in, XExpr& x) {
  auto term = [&](const Expr& t, XTerm& out) -> bool {
    if (t.k == Expr::COL) {
      out.col = in.at(t.name).col.get();
      return true;
    }
    if (t.k != Expr::BIN) return false;
    const int op = binop_from_name(t.name);
    if (op > RQ_DIV) return false;
    const Expr* l = t.l.get();
    const Expr* r = t.r.get();
    if (l->k == Expr::COL && r->k == Expr::LIT && r->lit != 2) {
      out.col = in.at(l->name).col.get();
      out.sop = op;
      out.rev = false;
      if (r->lit == 1) out.k.is_float = true, out.k.f = r->lf;
      else out.k.i = r->li;
      return true;
    }
    if (r->k == Expr::COL && l->k == Expr::LIT && l->lit != 2) {
      out.col = in.at(r->name).col.get();
      out.sop = op;
      out.rev = true;
      if (l->lit == 1) out.k.is_float = true, out.k.f = l->lf;
      else out.k.i = l->li;
      return true;
    }
    return false;
  };
  XTerm t;
  if (term(e, t)) {
    x.terms.push_back(t);
    return true;
  }
  if (e.k != Expr::BIN) return false;
  const int op = binop_from_name(e.name);
  if (op > RQ_DIV) return false;
  XTerm rt;
  if (!term(*e.r, rt)) return false;
  if (!to_xexpr(*e.l, in, x)) return false;
  if (x.terms.size() >= 3) return false;
  x.terms.push_back(rt);
  x.ops.push_back(op);
  return true;
}

// group_agg(filter(scan)) or group_agg(scan) as one fused call
bool Exec::try_fused_group(const Node& n, CSet& out) {
  const Node* in_node = n.input.get();
  ExprP pred;
  if (in_node->k == Node::FILTER) {
    pred = in_node->pred;
    in_node = in_node->input.get();
  }
  if (in_node->k != Node::SCAN) return false;
  CSet in = run(*in_node);
  std::vector<XPred> preds;
  if (pred && !to_conjuncts(*pred, in, preds)) return false;
  std::vector<XExpr> exprs;
  std::vector<int> fns;
  for (const auto& a : n.aggs) {
    if (a.fn != RQ_SUM && a.fn != RQ_AVG && a.fn != RQ_COUNT) return false;
    XExpr x;
    if (a.expr && !to_xexpr(*a.expr, in, x)) return false;
    exprs.push_back(x);
    fns.push_back(a.fn);
  }
  std::vector<const DCol*> keys;
  for (const auto& k : n.keys) keys.push_back(in.at(k).col.get());
  // The fused pass intersects one segment table with the coverage of every
  // operand of every expression (and the WHERE). The runner instead
  // (runner.cpp:302-336) aligns keys with all data jointly — including, for
  // count(*), the scan's FIRST column (in.cols.front()) — and without keys
  // aggregates each expression over its own coverage. The two agree when the
  // columns whose coverage differs are full-coverage; otherwise take the
  // runner's generic path (the no-key case is checked inside
  // group_aggregate_exprs, which the C ABI shares).
  bool has_count_star = false;
  for (auto& x : exprs) has_count_star |= x.terms.empty();
  if (keys.empty()) {  // count(*) without keys needs a column for the row count
    if (has_count_star) return false;
  } else if (has_count_star) {
    if (in.cols.empty() || !col_full_coverage(ctx, *in.cols.front().col)) return false;
  }
  bool was_fused = false;
  GroupAggOut r = group_aggregate_exprs(ctx, nullptr, keys, exprs, fns, &was_fused, preds.empty() ? nullptr : &preds,
                                        /*fused_only=*/true);
  if (!was_fused) return false;  // the generic path runs next (same result); counted only when fused
  ++fused;
  out.rows = r.n_groups;
  for (size_t k = 0; k < n.keys.size(); ++k) {
    const CCol& src = in.at(n.keys[k]);
    DCol c;
    c.enc = RQ_ENC_PLAIN;
    c.v = r.keys[k];
    c.logical = c.v.dt;
    c.total = c.v.n;
    out.cols.push_back({n.keys[k], std::make_shared<DCol>(std::move(c)), src.dict, src.is_date});
  }
  for (size_t i = 0; i < n.aggs.size(); ++i) {
    DCol c;
    c.enc = RQ_ENC_PLAIN;
    c.v = r.vals[i];
    c.logical = c.v.dt;
    c.total = c.v.n;
    out.cols.push_back({n.aggs[i].name, std::make_shared<DCol>(std::move(c)), nullptr, false});
  }
  return true;
}

CSet Exec::run(const Node& n) {  // runner.cpp:228-352
  CSet out;
  switch (n.k) {
    case Node::SCAN: {
      const TableD& t = cat.at(n.table);
      out.rows = t.rows;
      for (const auto& c : t.cols) {
        if (!n.columns.empty() && std::find(n.columns.begin(), n.columns.end(), c.name) == n.columns.end())
          continue;
        out.cols.push_back({c.name, c.col, c.dict, c.is_date});
      }
      if (!n.columns.empty())
        req(out.cols.size() == n.columns.size(), "scan: a requested column is missing from " + n.table);
      return out;
    }
    case Node::FILTER: {
      CSet in = run(*n.input);
      std::shared_ptr<DMask> m = eval_mask(in, *n.pred);
      out.rows = in.rows;
      for (const auto& c : in.cols)
        out.cols.push_back({c.name, std::make_shared<DCol>(filter(ctx, *c.col, *m)), c.dict, c.is_date});
      return out;
    }
    case Node::PROJECT: {
      CSet in = run(*n.input);
      out.rows = in.rows;
      for (const auto& it : n.items) {
        EvalV v = eval(in, *it.first);
        require(v.is_col(), "projection must be a column expression");
        out.cols.push_back({it.second, v.col, v.dict, v.is_date});
      }
      return out;
    }
    case Node::JOIN: {
      CSet left = run(*n.left);
      CSet right = run(*n.right);
      const CCol& lc = left.at(n.left_on);
      const CCol& rc = right.at(n.right_on);
      std::shared_ptr<const DCol> right_key = rc.col;
      if (lc.dict && rc.dict && lc.dict != rc.dict)
        right_key = std::make_shared<DCol>(recode_column(ctx, *rc.col, *rc.dict, *lc.dict));
      if (n.semi) {
        DMask m = semi_join_mask(ctx, *lc.col, *right_key);
        out.rows = left.rows;
        for (const auto& c : left.cols)
          out.cols.push_back({c.name, std::make_shared<DCol>(filter(ctx, *c.col, m)), c.dict, c.is_date});
        return out;
      }
      JoinResultD jr = get_join_index(ctx, *lc.col, *right_key);
      out.rows = jr.cardinality;
      for (const auto& c : left.cols)
        out.cols.push_back({c.name, std::make_shared<DCol>(apply_join_index(ctx, *c.col, jr.left)), c.dict,
                            c.is_date});
      for (const auto& c : right.cols) {
        for (const auto& existing : out.cols)
          req(existing.name != c.name, "join: duplicate output column name '" + c.name + "'; project first");
        out.cols.push_back({c.name, std::make_shared<DCol>(apply_join_index(ctx, *c.col, jr.right)), c.dict,
                            c.is_date});
      }
      return out;
    }
    default: {
      if (try_fused_group(n, out)) return out;
      out = CSet{};
      CSet in = run(*n.input);
      std::vector<const DCol*> key_cols;
      for (const auto& k : n.keys) key_cols.push_back(in.at(k).col.get());
      std::vector<DCol> data(n.aggs.size());
      std::vector<int> fns;
      for (size_t i = 0; i < n.aggs.size(); ++i) {
        const Agg& a = n.aggs[i];
        fns.push_back(a.fn);
        if (a.expr) {
          EvalV v = eval(in, *a.expr);
          require(v.is_col(), "aggregate input must be a column expression");
          data[i] = *v.col;
        } else {
          require(!in.cols.empty(), "count(*) on empty column set");
          data[i] = *in.cols.front().col;
        }
      }
      std::vector<const DCol*> dp;
      for (auto& d : data) dp.push_back(&d);
      if (n.keys.empty()) {
        out.rows = 1;
        for (size_t i = 0; i < n.aggs.size(); ++i) {
          AggOut a = aggregate_column(ctx, normalize_basic(ctx, data[i]), fns[i]);
          DArr r = a.dtype == RQ_F64 ? upload_arr(ctx, RQ_F64, &a.f, 1) : upload_arr(ctx, RQ_I64, &a.i, 1);
          DCol c;
          c.enc = RQ_ENC_PLAIN;
          c.v = r;
          c.logical = r.dt;
          c.total = 1;
          out.cols.push_back({n.aggs[i].name, std::make_shared<DCol>(std::move(c)), nullptr, false});
        }
        return out;
      }
      GroupAggOut r = group_aggregate(ctx, key_cols, dp, fns, true);
      out.rows = r.n_groups;
      for (size_t k = 0; k < n.keys.size(); ++k) {
        const CCol& src = in.at(n.keys[k]);
        DCol c;
        c.enc = RQ_ENC_PLAIN;
        c.v = r.keys[k];
        c.logical = c.v.dt;
        c.total = c.v.n;
        out.cols.push_back({n.keys[k], std::make_shared<DCol>(std::move(c)), src.dict, src.is_date});
      }
      for (size_t i = 0; i < n.aggs.size(); ++i) {
        DCol c;
        c.enc = RQ_ENC_PLAIN;
        c.v = r.vals[i];
        c.logical = c.v.dt;
        c.total = c.v.n;
        out.cols.push_back({n.aggs[i].name, std::make_shared<DCol>(std::move(c)), nullptr, false});
      }
      return out;
    }
  }
}

// to_rows (column.cpp:331-376): covered positions and values in row order
void to_rows(const CtxPtr& ctx, const DCol& c, DArr& pos, DArr& vals) {
  switch (c.enc) {
    case RQ_ENC_PLAIN:
      pos = iota(ctx, c.total);
      vals = decode_plain(ctx, c);
      return;
    case RQ_ENC_PLAIN_INDEX:
      pos = iota(ctx, c.total);
      vals = decode_plain_index(ctx, c);
      return;
    case RQ_ENC_RLE: {
      DArr s = c.s.n || c.e.n == 0 ? c.s : starts_from_ends(ctx, c.e);
      DArr idx;
      expand_runs(ctx, s, c.e, &pos, &idx);
      vals = gather(ctx, c.v, idx);
      return;
    }
    case RQ_ENC_INDEX:
      pos = c.p;
      vals = c.v;
      return;
    default: to_rows(ctx, normalize_basic(ctx, c), pos, vals);
  }
}

}  // namespace planx

ResultD run_plan(const CtxPtr& ctx, const CatalogD& cat, const std::string& json) {
  planx::J j = planx::JsonReader(json).value();
  planx::NodeP plan = planx::parse_node(j.get("plan") ? j.at("plan") : j);
  planx::Exec ex{ctx, cat};
  KTimer timer(ctx, "run_plan");
  planx::CSet ds = ex.run(*plan);
  ResultD out;  // materialize (runner.cpp:354-373)
  out.rows = -1;
  out.fused = ex.fused;
  DArr ref_pos;
  for (const auto& c : ds.cols) {
    DArr pos, vals;
    planx::to_rows(ctx, *c.col, pos, vals);
    if (out.rows < 0) {
      out.rows = pos.n;
      ref_pos = pos;
    } else {
      require(pos.n == ref_pos.n, "internal: output columns disagree on covered rows");
    }
    out.names.push_back(c.name);
    out.dicts.push_back(c.dict);
    out.columns.push_back(vals);
  }
  if (out.rows < 0) out.rows = 0;
  return out;
}

}  // namespace rqb

// ---- C ABI ------------------------------------------------------------------------

struct rq_catalog_s {
  rqb::CatalogD cat;
  std::map<std::string, rqb::DictP> dicts;  // shared by name so equal dictionaries stay identical
};
struct rq_result_s {
  rqb::ResultD r;
};

namespace {
rqb::CtxPtr ctx_of(rq_ctx_t c) {
  if (!c || !c->ctx) rqb::fail("null context");
  RQ_CUDA_CHECK(cudaSetDevice(c->ctx->device));
  return c->ctx;
}
const rqb::DCol& col_of(rq_col_t c) {
  if (!c) rqb::fail("null column handle");
  return c->c;
}
}  // namespace

extern "C" {

int rq_catalog_create(rq_catalog_t* out) {
  return rqb::api_guard([&] {
    rqb::require(out != nullptr, "null out");
    *out = new rq_catalog_s{};
  });
}

int rq_catalog_destroy(rq_catalog_t c) {
  return rqb::api_guard([&] { delete c; });
}

int rq_catalog_add_column(rq_catalog_t c, const char* table, const char* column, rq_col_t col,
                          const char* const* dict, int64_t dict_n, const char* dict_name, int32_t is_date) {
  return rqb::api_guard([&] {
    rqb::require(c && table && column && col, "null argument");
    rqb::TableD* t = nullptr;
    for (auto& x : c->cat.tables)
      if (x.name == table) t = &x;
    if (!t) {
      c->cat.tables.push_back({table, 0, {}});
      t = &c->cat.tables.back();
    }
    const rqb::DCol& d = col_of(col);
    rqb::require(t->cols.empty() || t->rows == d.total, "catalog: column length differs from its table");
    t->rows = d.total;
    rqb::DictP dp;
    if (dict_n > 0 || dict_name) {
      const std::string key = dict_name ? dict_name : std::string(table) + "." + column;
      auto it = c->dicts.find(key);
      if (it != c->dicts.end() && dict_n == 0) {
        dp = it->second;
      } else {
        auto nd = std::make_shared<rqb::DictD>();
        for (int64_t i = 0; i < dict_n; ++i) {
          nd->code.emplace(dict[i], static_cast<int64_t>(nd->s.size()));
          nd->s.emplace_back(dict[i]);
        }
        dp = nd;
        c->dicts[key] = dp;
      }
    }
    t->cols.push_back({column, std::make_shared<rqb::DCol>(d), dp, is_date != 0});
  });
}

int rq_run_plan(rq_ctx_t ctx, rq_catalog_t c, const char* plan_json, rq_result_t* out) {
  return rqb::api_guard([&] {
    rqb::require(c && plan_json && out, "null argument");
    *out = new rq_result_s{rqb::run_plan(ctx_of(ctx), c->cat, plan_json)};
  });
}

int rq_result_info(rq_result_t r, int32_t* n_cols, int64_t* rows, int32_t* fused_nodes) {
  return rqb::api_guard([&] {
    rqb::require(r != nullptr, "null result");
    if (n_cols) *n_cols = static_cast<int32_t>(r->r.columns.size());
    if (rows) *rows = r->r.rows;
    if (fused_nodes) *fused_nodes = r->r.fused;
  });
}

int rq_result_column(rq_result_t r, int32_t i, const char** name, rq_arr_t* values) {
  return rqb::api_guard([&] {
    rqb::require(r != nullptr && i >= 0 && i < static_cast<int32_t>(r->r.columns.size()), "result column out of range");
    if (name) *name = r->r.names[static_cast<size_t>(i)].c_str();
    if (values) *values = rqb::wrap_arr(r->r.columns[static_cast<size_t>(i)]);
  });
}

int rq_result_free(rq_result_t r) {
  return rqb::api_guard([&] { delete r; });
}

}  // extern "C"
