"""Summarise a stream-kernel event log (tools/trace_stream.py output)."""
import sys
import numpy as np
EV = {1: "start", 2: "issue", 3: "issueR", 4: "skip", 5: "consume", 6: "resPiece", 7: "pdone", 8: "xch",
      9: "decide", 10: "resDone", 11: "rowEnd", 12: "end", 13: "plan"}
d = np.load(sys.argv[1])
buf = d["buf"].astype(np.uint64)
grid = buf.shape[0]
recs = []
for c in range(grid):
    n = int(buf[c, 0])
    r = buf[c, 1:n + 1]
    typ = (r >> np.uint64(56)).astype(int)
    arg = ((r >> np.uint64(40)) & np.uint64(0xFFFF)).astype(int)
    t = (r & np.uint64(0xFFFFFFFFFF)).astype(np.int64)
    recs.append((typ, arg, t))
t0 = min(r[2].min() for r in recs if len(r[2]))
def us(x): return (x - t0) / 1000.0
ends = [us(r[2][r[0] == 12]).max() for r in recs]
starts = [us(r[2][r[0] == 1]).min() for r in recs]
print(f"CTAs {grid}; start med {np.median(starts):.2f} max {max(starts):.2f}; end min {min(ends):.1f} med {np.median(ends):.1f} max {max(ends):.1f} us")
cta = int(sys.argv[2]) if len(sys.argv) > 2 else 0
typ, arg, t = recs[cta]
o = np.argsort(t)
print(f"--- CTA {cta} timeline (first 120 events)")
for i in o[:120]:
    print(f"{us(t[i]):8.2f} {EV.get(typ[i], typ[i]):9s} {arg[i] & 0x3FFF:5d} {'R' if arg[i] & 0x8000 else ''}{'S' if arg[i] & 0x4000 else ''}")
# per-row latencies: issue(first) -> consume(last) -> pdone -> xch -> decide -> rowEnd
rows = {}
for c in range(grid):
    typ, arg, t = recs[c]
    for ty, a, tt in zip(typ, arg, t):
        key = (c, a & 0x3FFF)
        rows.setdefault(key, {}).setdefault(ty, []).append(us(tt))
def stat(name, f):
    v = [f(r) for r in rows.values()]
    v = np.array([x for x in v if x is not None])
    if len(v): print(f"{name:28s} n={len(v):5d} med {np.median(v):7.2f} p90 {np.percentile(v, 90):7.2f} max {v.max():7.2f} us")
stat("issue first->last consume", lambda r: max(r[5]) - min(r[2]) if 2 in r and 5 in r else None)
stat("last consume->pdone", lambda r: min(r[7]) - max(r[5]) if 5 in r and 7 in r else None)
stat("pdone->xch", lambda r: min(r[8]) - min(r[7]) if 7 in r and 8 in r else None)
stat("xch->decide", lambda r: min(r[9]) - min(r[8]) if 8 in r and 9 in r else None)
stat("decide->resDone", lambda r: min(r[10]) - min(r[9]) if 9 in r and 10 in r else None)
stat("resDone->rowEnd", lambda r: min(r[11]) - min(r[10]) if 10 in r and 11 in r else None)
stat("decide->rowEnd (no resid)", lambda r: min(r[11]) - min(r[9]) if 9 in r and 11 in r and 10 not in r else None)
stat("issueR first->last", lambda r: max(r[3]) - min(r[3]) if 3 in r else None)
# producer issue rate
typ, arg, t = recs[cta]
iss = np.sort(us(t[typ == 2]))
if len(iss) > 1: print(f"CTA {cta}: {len(iss)} main issues, {np.sum(typ==3)} resid issues, {np.sum(typ==4)} skips; issue gaps med {np.median(np.diff(iss)):.3f} us; span {iss[0]:.1f}-{iss[-1]:.1f}")

# clock64 accounting (cycles; 8 stats warps / 4 row warps summed)
ctr = buf[:, -16:].astype(np.float64)
names_n = 16
names = ["stats wait full", "stats total", "stats main pieces", "stats resid pieces", "planner wait empty",
         "planner wait pfree", "planner total", "row wait pdone", "row wait xch", "row wait resdone",
         "row wait xres", "row total", "stats compute", "stats trywait fails", "issuers wait plan", "issuers wait empty"]
print("--- clock64 accounting, median over CTAs (cycles; stats summed over 8 warps, rows over 4)")
for i, nm in enumerate(names):
    print(f"{nm:22s} {np.median(ctr[:, i]):14.0f}")
