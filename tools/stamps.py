import re, sys
rows = [l for l in open(sys.argv[1]) if l.startswith("STAMP")]
rows = rows[-12:]
vals = []
for l in rows:
    m = dict(re.findall(r"(\w+) (\d+)", l))
    vals.append(m)
t0 = min(int(v["start"]) for v in vals)
for v in vals:
    print(" ".join(f"{k}={(int(v[k]) - t0) / 1000:.2f}" if k in ("start", "search", "full", "cons_end", "prod_end", "ticket") else f"{k}={v[k]}" for k in ("cta", "start", "search", "full", "cons_end", "prod_end", "ticket", "last")))
