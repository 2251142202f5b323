"""Validates the streaming oracle (oracle/streaming.py) against the
unmodified reference library at up to 100M rows on the same seeded tables
("validate it against the library at <=100M rows on identical
seeds first, then use it as the at-scale oracle"). Test infrastructure.

    python tools/validate_streaming_oracle.py [c3=100e6] [q1=10e6] [q6=100e6] [c5=100e6]

Prints one line per configuration: rows, reference seconds, oracle seconds,
groups, and whether the full tables agree (ints exact, f64 1e-9 relative).
"""
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))

from oracle import streaming as S  # noqa: E402
from oracle.refpy import Ref, RefAPI  # noqa: E402
from paper_2506_10092_b200 import datagen as G  # noqa: E402
from paper_2506_10092_b200 import queries as Q  # noqa: E402
from test_oracle_streaming_cpu import tables_equal  # noqa: E402


def main():
    sizes = {"c3": 100_000_000, "q1": 10_000_000, "q6": 100_000_000, "c5": 100_000_000}
    for a in sys.argv[1:]:
        k, v = a.split("=")
        sizes[k] = int(float(v))
    ref, so = Ref(), S.StreamingOracle()
    api = RefAPI(ref)
    for name, n in sizes.items():
        if name == "c3":
            k, x, y, z, w = G.c3_tables(n, 42)
            t0 = time.time()
            ks, vs, _ = ref.group_aggregate([ref.normalize_basic(k)],
                                            [ref.normalize_basic(c) for c in (x, k, z, y, w)], G.C3_FNS)
            tr = time.time() - t0
            t0 = time.time()
            got = S.c3({"k": k, "x": x, "y": y, "z": z, "w": w}, so)
            to = time.time() - t0
            del k, x, y, z, w
        elif name == "q1":
            t = Q.lineitem_q1(n, 43)
            t0 = time.time()
            ks, vs, _ = Q.q1(api, t)
            tr = time.time() - t0
            t0 = time.time()
            got = S.q1(t, Q.Q1_CUTOFF, so)
            to = time.time() - t0
        elif name == "q6":
            t = Q.lineitem_q6(n, 42)
            t0 = time.time()
            want = Q.q6(api, t)
            tr = time.time() - t0
            t0 = time.time()
            g = S.q6(t, Q.Q6_WHERE, so)
            to = time.time() - t0
            ok = abs(g - want) <= 1e-9 * max(1.0, abs(g), abs(want))
            print(f"{name}: rows={n} reference={tr:.1f}s oracle={to:.2f}s value={g!r} ref={want!r} "
                  f"match={ok}", flush=True)
            continue
        else:
            t = Q.production_table(n, 5)
            t0 = time.time()
            ks, vs, _ = Q.c5_query(api, t)
            tr = time.time() - t0
            t0 = time.time()
            got = S.c5(t, Q.C5_IN, Q.C5_LT, so)
            to = time.time() - t0
        try:
            tables_equal(got, ks, vs)
            ok = True
        except AssertionError as e:
            ok = f"MISMATCH {e}"
        print(f"{name}: rows={n} reference={tr:.1f}s oracle={to:.2f}s groups={len(got[0][0])} "
              f"checksum(first agg)={int(got[1][0].astype('int64').sum()) if got[1][0].dtype.kind != 'f' else float(got[1][0].sum())} "
              f"match={ok}", flush=True)


if __name__ == "__main__":
    main()
