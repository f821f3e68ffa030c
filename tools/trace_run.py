"""Timeline of one fused sd_verify call (sd_debug_trace) -> gpurun_out/trace_<config>.json."""
import argparse, json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import paper_2601_21622_b200 as sd
from paper_2601_21622_b200 import _lib
from workload import CONFIGS, make_batch_torch

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="c2")
ap.add_argument("--out", default="gpurun_out")
a = ap.parse_args()
c = CONFIGS[a.config]
dev = torch.device("cuda:0")
bs = [make_batch_torch(c["V"], c["k"], c["B"], c["T"], c["kappa"], c["seed"] + i, dev) for i in range(4)]
G = torch.cuda.get_device_properties(0).multi_processor_count
rows = c["B"] * (c["k"] + 1)
buf = torch.zeros(4 * G + 2 * rows + c["B"] + G * 64, dtype=torch.int64, device=dev)
for i in range(6):
    b = bs[i % 4]
    sd.verify(b["p"], b["q"], b["ids"], c["T"], seed=1, round=i)
torch.cuda.synchronize()
_lib.load().sd_debug_trace(buf.data_ptr())
b = bs[1]
L, tok, st = sd.verify(b["p"], b["q"], b["ids"], c["T"], seed=1, round=99)
torch.cuda.synchronize()
_lib.load().sd_debug_trace(None)
t = buf.cpu().numpy().astype(np.float64)
t0 = t[:G].min()
rel = lambda x: np.where(x > 0, (x - t0) / 1000.0, np.nan)
out = dict(G=G, rows=rows, B=c["B"], k=c["k"], L=L.cpu().tolist(),
           cta_start=rel(t[:G]).tolist(), p1_end=rel(t[G:2*G]).tolist(),
           prod_end=rel(t[2*G:3*G]).tolist(), cta_exit=rel(t[3*G:4*G]).tolist(),
           decide=rel(t[4*G:4*G+rows]).tolist(), pass_end=rel(t[4*G+rows:4*G+2*rows]).tolist(),
           done=rel(t[4*G+2*rows:4*G+2*rows+c["B"]]).tolist())
wc = buf.cpu().numpy()[4*G+2*rows+c["B"]:].reshape(G, 16, 4).astype(np.float64)
ep = wc[:, 14, :]; de = wc[:, 15, :]
out["warp_counters"] = wc.tolist()
json.dump(out, open(os.path.join(a.out, f"trace_{a.config}.json"), "w"))
worst = np.argsort(-(de[:, 0] + de[:, 1]))[:5]
for g in worst:
    print("cta %3d: decider rows %d (%.0f cyc) searches %d (%.0f cyc) | p1_end %.1f | epi entries %d" % (
        g, de[g, 2], de[g, 0], de[g, 3], de[g, 1], out["p1_end"][g], ep[g, 2]))
print("epilogue: publish cycles med %.0f of total %.0f; entries %.0f batches %.0f" % (np.median(ep[:,0]), np.median(ep[:,1]), np.median(ep[:,2]), np.median(ep[:,3])))
print("decider: rows %.1f cycles/row %.0f; searches %.2f cycles/search %.0f; max total %.0f" % (de[:,2].mean(), de[:,0].sum()/max(de[:,2].sum(),1), de[:,3].mean(), de[:,1].sum()/max(de[:,3].sum(),1), (de[:,0]+de[:,1]).max()))
cons = wc[:, :12, :]; prod = wc[:, 12, :]
print("consumer: wait frac med %.2f  items/warp med %.1f  resid items/warp %.2f  total cycles med %.0f" % (
    np.median(cons[:, :, 0] / np.maximum(cons[:, :, 1], 1)), np.median(cons[:, :, 2]), cons[:, :, 3].mean(), np.median(cons[:, :, 1])))
print("producer: empty-wait cycles med %.0f  slots %.0f" % (np.median(prod[:, 0]), np.median(prod[:, 2])))
json.dump(out, open(os.path.join(a.out, f"trace_{a.config}.json"), "w"))
def q(x):
    x = np.array(x, dtype=float); x = x[~np.isnan(x)]
    return f"n={len(x)} min={x.min():.1f} med={np.median(x):.1f} max={x.max():.1f}" if len(x) else "n=0"
for k in ("cta_start", "p1_end", "prod_end", "cta_exit", "decide", "pass_end", "done"):
    print(f"{k:10s} {q(out[k])} (us)")
