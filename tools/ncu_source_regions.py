"""Split an `ncu --page source --csv` dump of one kernel into code regions by executed-
instruction count (the main k loop is the run of instructions executed most often) and
report the stall samples inside and outside it.
  python tools/ncu_source_regions.py <source.csv>"""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
h = rows[1]
src, smp, nis, ex = h.index("Source"), h.index("Warp Stall Sampling (All Samples)"), \
    h.index("Warp Stall Sampling (Not-issued Samples)"), h.index("Instructions Executed")
stall_cols = [i for i, c in enumerate(h) if c.startswith("stall_")]
data = [(r[src].strip(), int(r[smp] or 0), int(r[nis] or 0), int(r[ex] or 0), r) for r in rows[2:] if len(r) > ex]
tot = sum(d[1] for d in data)
mx = max(d[3] for d in data)
hot = [d for d in data if d[3] >= 0.5 * mx]
print(f"instructions {len(data)}, samples {tot}, hottest executed count {mx}")
print(f"hot region: {len(hot)} instr, samples {sum(d[1] for d in hot)} ({100.0 * sum(d[1] for d in hot) / tot:.1f}%), "
      f"not-issued {sum(d[2] for d in hot)}")
cold = [d for d in data if d[3] < 0.5 * mx]
print(f"rest: {len(cold)} instr, samples {sum(d[1] for d in cold)} ({100.0 * sum(d[1] for d in cold) / tot:.1f}%)")
def ops(ds):
    m = {}
    for d in ds:
        op = d[0].split()[0] if not d[0].startswith("@") else d[0].split()[1]
        op = op.split(".")[0]
        m[op] = m.get(op, 0) + d[1]
    return sorted(m.items(), key=lambda kv: -kv[1])[:8]
print("hot by opcode:", ops(hot))
print("rest by opcode:", ops(cold))
if stall_cols:
    for name, ds in (("hot", hot), ("rest", cold)):
        agg = {h[i]: sum(int(d[4][i] or 0) for d in ds) for i in stall_cols}
        print(name, sorted(agg.items(), key=lambda kv: -kv[1])[:8])
