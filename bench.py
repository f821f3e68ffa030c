#!/usr/bin/env python
"""bench.py -- verified tokens/s of the StarSD speculative-sampling verify step on B200.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config c2] [--impl ours|reference]

A step is one sd_verify call (the whole hot path, rows a1-a10 of SURVEY 8(a)) over one batch of
synthetic logits that is already resident in HBM.  The default workload is BASELINE.json
configs[2] -- the Llama-3 shape north_star's target is quoted on (V=128256, k=7, B=128 per
verifier, T=1, fp32, kappa=30).  Eight distinct batches (7.9 GB > the 126 MB L2) are rotated so
no step reads L2-resident inputs of the previous one.
K steps are captured in one CUDA graph and timed with CUDA events on the launching stream (device
timestamps inside the same graph give the dominant kernel's span for the roofline).
Multi-GPU runs (torchrun, N > 1) run the star of PAPER.md Alg. 1: rank 0 drafts, ranks 1..N-1
verify over NCCL (--mode dp: independent verifiers instead); --star-loopback N emulates a 1 -> N
star on one GPU.  Times are the max over ranks.

Printed: one JSON line (rank 0).  See DESIGN.md "Measurement" for every field.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "verified tokens/s (spec-sampling verify)"
UNIT = "verified tokens/s"


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=2000)
    ap.add_argument("--warmup", type=int, default=20)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="c3")
    ap.add_argument("--dtype", default="f32", choices=["f32", "bf16"])
    ap.add_argument("--temperature", type=float, default=None)
    ap.add_argument("--nbatch", type=int, default=8)
    ap.add_argument("--e2e-steps", type=int, default=20)
    ap.add_argument("--cpu-seconds", type=float, default=10.0)
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--mode", default="auto", choices=["auto", "star", "dp"],
                    help="N > 1: star (rank 0 drafts, ranks 1..N-1 verify; default) or dp "
                         "(independent verifiers)")
    ap.add_argument("--star-loopback", type=int, default=0,
                    help="emulate a 1 -> N star in one process on one GPU (loopback transport)")
    ap.add_argument("--payload", default="full", choices=["full", "qmeta"])
    ap.add_argument("--slots", type=int, default=2)
    ap.add_argument("--draft-hidden", type=int, default=4096)
    ap.add_argument("--o-alone", type=float, default=0.0,
                    help="standalone target tokens/ms for the N_max admission bound")
    ap.add_argument("--batches", default="",
                    help="star: per-verifier batch sizes, comma-separated (C4 heterogeneous star)")
    ap.add_argument("--kappas", default="",
                    help="star: per-verifier draft/target agreement kappa, comma-separated (C4)")
    ap.add_argument("--target-ms", type=float, default=0.0,
                    help="star: the verifiers' target-model forward per round, as a device spin "
                         "of this many ms before each verify (Z of Eq. 6; 0 = verify only)")
    ap.add_argument("--trace-seconds", type=float, default=0.0,
                    help="star loopback: drive the verifiers' cohorts by a seeded bursty arrival "
                         "trace for this many seconds (BASELINE C5)")
    ap.add_argument("--burst-rate", type=float, default=20.0, help="C5: bursts per second per verifier")
    ap.add_argument("--burst-mean", type=float, default=16.0, help="C5: mean requests per burst")
    return ap.parse_args()


def dist_env():
    return (int(os.environ.get("RANK", 0)), int(os.environ.get("WORLD_SIZE", 1)),
            int(os.environ.get("LOCAL_RANK", 0)))


def workload(args):
    from workload import CONFIGS
    c = dict(CONFIGS[args.config])
    if args.temperature is not None:
        c["T"] = args.temperature
    return c


def esize(dtype):
    return 4 if dtype == "f32" else 2


def algorithmic_bytes(L, V, k, e, greedy):
    """bytes the method itself must move for one request with accept length L
    (lazy: rows up to the first rejection), plus ids and outputs."""
    import numpy as np
    L = np.asarray(L, np.int64)
    rows = (L + 1) if greedy else (L + 1) + np.minimum(L + 1, k)
    return rows * V * e + 4 * k + 4 * (k + 2)


def load_peaks():
    try:
        m = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
        return float(m["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback"


# ------------------------------------------------------------------------------- clocks ----
class ClockSampler:
    """NVML SM-clock and throttle-reason sampling during the timed region."""
    REASONS = {0x4: "sw_power_cap", 0x8: "hw_slowdown", 0x20: "sw_thermal_slowdown",
               0x40: "hw_thermal_slowdown", 0x80: "hw_power_brake_slowdown",
               0x2: "applications_clocks_setting", 0x1: "gpu_idle"}

    def __init__(self, index, period=0.002):
        self.index, self.period = index, period
        self.samples, self.reasons = [], set()
        self._stop = threading.Event()
        self._first = threading.Event()
        self.max_mhz = None
        self.ok = False
        try:
            import pynvml
            pynvml.nvmlInit()
            self.nv = pynvml
            self.h = pynvml.nvmlDeviceGetHandleByIndex(index)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
            self.ok = True
        except Exception:
            self.nv = None

    def _run(self):
        nv = self.nv
        while not self._stop.is_set():
            try:
                self.samples.append(nv.nvmlDeviceGetClockInfo(self.h, nv.NVML_CLOCK_SM))
                r = nv.nvmlDeviceGetCurrentClocksEventReasons(self.h)
                for bit, name in self.REASONS.items():
                    if r & bit and bit != 0x1:
                        self.reasons.add(name)
            except Exception:
                pass
            self._first.set()
            time.sleep(self.period)

    def __enter__(self):
        if self.ok:
            self.t = threading.Thread(target=self._run, daemon=True)
            self.t.start()
            self._first.wait(timeout=2.0)      # sampling is live before the timed region
        return self

    def __exit__(self, *a):
        if self.ok:
            self._stop.set()
            self.t.join()

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": self.max_mhz, "reasons": sorted(self.reasons),
                    "samples": 0}
        return {"sm_mhz": statistics.median(self.samples), "sm_max_mhz": self.max_mhz,
                "reasons": sorted(self.reasons), "samples": len(self.samples)}


# --------------------------------------------------------------------------- CPU oracle ----
def oracle_rate(d, T, seconds, seed, cores, per_step=None, steps=None):
    """Time the CPU oracle (as it stands) on bounded samples of the workload: each step
    verifies `per_step` consecutive requests of the batch (rotating).  Returns tokens/s and a
    description of the sample."""
    import numpy as np
    import oracle
    B = d["ids"].shape[0]
    per_step = per_step or min(B, cores)
    n, tok, t0, i = 0, 0, time.perf_counter(), 0
    while True:
        lo = (i * per_step) % B
        idx = [(lo + j) % B for j in range(per_step)]
        L, _, st = oracle.verify(d["p"][idx], None if T == 0 else d["q"][idx], d["ids"][idx], T,
                                 seed=seed, round=i, rid_base=lo, n_threads=cores)
        tok += int((L + 1)[st & oracle.HARD_FAULTS == 0].sum())
        n += per_step
        i += 1
        el = time.perf_counter() - t0
        if (steps is not None and i >= steps) or (steps is None and el >= seconds):
            break
    return tok / el, dict(requests=n, steps=i, per_step=per_step, seconds=el)


def parity_sample(dev_batch, d0, T, V, cores, n=32):
    """After the timed region: one GPU verify of batch 0 (seed 21622, round 0) against the oracle
    on its first n requests, with the C-13 rule (tests/parity.py): exact unless the oracle's fp64
    margins are below 1e-6 (a tie).  Returns the counts (mismatches must be 0)."""
    import numpy as np
    import torch
    import oracle
    import paper_2601_21622_b200 as sd
    L, tok, st = sd.verify(dev_batch["p"], None if T == 0 else dev_batch["q"], dev_batch["ids"], T,
                           seed=21622, round=0, request_id_base=0, vocab=V)
    torch.cuda.synchronize()
    n = min(n, int(L.shape[0]))
    gL, gt, gs = L[:n].cpu().numpy(), tok[:n].cpu().numpy(), st[:n].cpu().numpy()
    rL, rt, rs, tr = oracle.verify(d0["p"][:n], None if T == 0 else d0["q"][:n], d0["ids"][:n], T,
                                   seed=21622, round=0, rid_base=0, V=V, trace=True,
                                   n_threads=cores)
    exact = ties = bad = 0
    for b in range(n):
        same = gL[b] == rL[b] and np.array_equal(gt[b], rt[b]) and gs[b] == rs[b]
        tie = T > 0 and not (rs[b] & oracle.HARD_FAULTS) and (
            tr[b].mu_a < 1e-6 or tr[b].mu_s < 1e-6 or tr[b].R < 5e-8)
        if same:
            exact += 1
        elif tie:
            ties += 1
        else:
            bad += 1
    return {"requests": n, "bit_exact": exact, "ties": ties, "mismatches": bad,
            "rule": "C-13 (DESIGN.md): bit-exact L, tokens, status outside fp64 margins < 1e-6"}


def host_batch(d):
    import numpy as np
    import torch
    out = {}
    for key in ("p", "q", "ids"):
        t = d[key]
        if t is None:
            out[key] = None
        elif isinstance(t, np.ndarray):
            out[key] = t
        else:
            t = t.cpu()
            out[key] = (t.view(torch.int16).numpy().view(np.uint16)
                        if t.dtype == torch.bfloat16 else t.numpy())
    return out


def run_reference(args):
    """--impl reference: the CPU oracle (the tier's reference arm) timed as it stands on this
    host's cores, on the same config/metric; rank 0 only."""
    rank, world, _ = dist_env()
    if rank != 0:
        return
    import numpy as np
    from workload import make_batch
    c = workload(args)
    d = make_batch(V=c["V"], k=c["k"], B=c["B"], T=c["T"], kappa=c["kappa"] or 30.0,
                   seed=c["seed"], dtype=args.dtype)
    cores = len(os.sched_getaffinity(0))
    per = max(1, min(c["B"], cores))
    oracle_rate(d, c["T"], 0, 1, cores, per_step=per, steps=max(1, args.warmup))
    rate, info = oracle_rate(d, c["T"], 0, 1, cores, per_step=per, steps=args.steps)
    sample = (f"{args.steps} steps x {per} requests of the {args.config} batch "
              f"(V={c['V']}, k={c['k']}, T={c['T']}), oracle threads={cores}")
    line = {"impl": "reference", "metric": METRIC, "value": rate, "unit": UNIT,
            "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": 1000 * info["seconds"] / info["steps"], "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": config_block(args, c),
            "cpu_baseline": {"value": rate, "unit": UNIT, "cores": cores, "kind": "oracle",
                             "sample": sample},
            "e2e": {"value": rate, "unit": UNIT, "h2d_bytes_per_step": 0,
                    "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def config_block(args, c):
    return {"workload": f"{args.config}: {c['name']}", "vocab": c["V"], "k": c["k"],
            "batch_per_gpu": c["B"], "temperature": c["T"], "kappa": c["kappa"],
            "logits": args.dtype, "inputs": "synthetic log-Dirichlet logits (DESIGN.md recipe)",
            "l2": f"rotating {args.nbatch} distinct resident input batches (> 126 MB L2)",
            "parallelism": f"dp{args.gpus} (one verifier per GPU, requests sharded)"}


# --------------------------------------------------------------------------------- ours ----
def run_ours(args):
    import numpy as np
    import torch
    import torch.distributed as dist

    import paper_2601_21622_b200 as sd
    from paper_2601_21622_b200 import _lib
    from paper_2601_21622_b200.dp import reduce_max_sum, request_id_base
    from workload import make_batch_torch

    rank, world, local = dist_env()
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        dist.init_process_group("nccl", device_id=dev)
    c = workload(args)
    V, k, B, T = c["V"], c["k"], c["B"], c["T"]
    greedy = T == 0.0
    e = esize(args.dtype)

    batches = [make_batch_torch(V, k, B, T, c["kappa"] or 30.0, c["seed"] + 1000 * rank + i, dev,
                                dtype=args.dtype) for i in range(args.nbatch)]
    torch.cuda.synchronize()
    K, W = args.steps, max(3, args.warmup)
    L_all = torch.empty(K, B, dtype=torch.int32, device=dev)
    tok_all = torch.empty(K, B, k + 1, dtype=torch.int32, device=dev)
    st_all = torch.empty(K, B, dtype=torch.int32, device=dev)
    ws = sd.Workspace(B, k, V, T, batches[0]["p"].dtype, dev)
    rid0 = request_id_base(rank)

    def step(i, out):
        bt = batches[i % args.nbatch]
        return sd.verify(bt["p"], None if greedy else bt["q"], bt["ids"], T, seed=21622,
                         round=i, request_id_base=rid0, out=out, workspace=ws)

    # warm-up (eager), then capture K steps into one graph (the timed one) and the same K steps
    # into a second graph with per-step profiling events around k_row_stats (the roofline's kernel
    # time; event nodes between the kernels would otherwise sit inside the timed step)
    wout = (L_all[0], tok_all[0], st_all[0])
    for i in range(W):
        step(i, wout)
    torch.cuda.synchronize()
    # the timed graph carries device timestamps (sd_profile_timestamps: %globaltimer folded with
    # atomic min at the first k_row_stats CTA start and at the first CTA of the second kernel to
    # see k_row_stats complete) -- the dominant kernel's span per step, no event nodes
    from paper_2601_21622_b200 import _lib as _l
    ts = torch.full((K, 2), -1, dtype=torch.int64, device=dev)
    g = torch.cuda.CUDAGraph()
    cs = torch.cuda.Stream(dev)
    cs.wait_stream(torch.cuda.current_stream(dev))
    with torch.cuda.stream(cs):
        _l.check(_l.load().sd_profile_timestamps(ts.data_ptr(), K), "sd_profile_timestamps")
        with torch.cuda.graph(g, stream=cs):
            for i in range(K):
                step(i, (L_all[i], tok_all[i], st_all[i]))
        _l.check(_l.load().sd_profile_timestamps(None, 0), "sd_profile_timestamps")
    torch.cuda.synchronize()
    evs = []
    for _ in range(2 * K):
        ev = torch.cuda.Event(enable_timing=True)
        ev.record()
        evs.append(ev)
    torch.cuda.synchronize()
    import ctypes
    handles = (ctypes.c_void_p * (2 * K))(*[ev.cuda_event for ev in evs])
    L = _lib.load()
    gp = torch.cuda.CUDAGraph()
    with torch.cuda.stream(cs):
        _lib.check(L.sd_profile_events(handles, K), "sd_profile_events")
        with torch.cuda.graph(gp, stream=cs):
            for i in range(K):
                step(i, (L_all[i], tok_all[i], st_all[i]))
        _lib.check(L.sd_profile_events(None, 0), "sd_profile_events")
    torch.cuda.synchronize()
    g.replay()                       # one untimed replay each (graph upload / first-touch)
    gp.replay()
    torch.cuda.synchronize()
    ts.fill_(-1)
    torch.cuda.synchronize()

    t0, t1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    with ClockSampler(local) as clk:
        t0.record()
        g.replay()
        t1.record()
        torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    ms = t0.elapsed_time(t1)
    tsh = ts.cpu().numpy().view(np.uint64)
    gp.replay()                      # the evented replay: k_row_stats event pairs (cross-check)
    torch.cuda.synchronize()
    kA_ev = [evs[2 * i].elapsed_time(evs[2 * i + 1]) for i in range(K)]
    if (tsh != np.uint64(2**64 - 1)).all():
        kA = list(((tsh[:, 1] - tsh[:, 0]).astype(np.float64) / 1e6))
        kA_src = "device timestamps in the timed graph (sd_profile_timestamps)"
    else:                            # (a variant without timestamp hooks)
        kA = kA_ev
        kA_src = "CUDA events around the kernel (separate replay)"

    Lh = L_all.cpu().numpy()
    sth = st_all.cpu().numpy()
    ok = (sth & 7) == 0
    tokens = int((Lh + 1)[ok].sum())
    alg = float(algorithmic_bytes(Lh, V, k, e, greedy).sum())
    (ms_max,), (tokens_all,) = reduce_max_sum([ms], [tokens], dev)
    value = tokens_all / (ms_max / 1000.0)

    # dominant kernel (k_row_stats on the two-launch path; the stream variant's kernel): algorithmic
    # bytes of the whole step per launch / its CUDA-event time on the launching stream
    pl = sd.plan(B, k, V, T, torch.float32 if args.dtype == "f32" else torch.bfloat16)
    kname = "k_row_stats"
    kA_mean_ms = statistics.fmean(kA)
    alg_per_launch = alg / K
    peak, peak_kind = load_peaks()
    achieved_gbs = alg_per_launch / (kA_mean_ms / 1000.0) / 1e9
    traffic = None
    prof = os.path.join(ROOT, "profiles", f"ncu_{args.config}_{args.dtype}.json")
    if os.path.exists(prof):
        try:
            traffic = json.load(open(prof)).get(f"{kname}_dram_bytes_per_launch")
        except Exception:
            traffic = None

    # e2e: host (pinned) inputs -> device -> verify -> host results, every step
    e2e = None
    if not args.no_e2e:
        hb = []
        for i in range(2):
            bt = batches[i]
            hb.append({x: (bt[x].cpu().pin_memory() if bt[x] is not None else None)
                       for x in ("p", "q", "ids")})
        staging = {}
        for i in range(2):
            sd.verify_host(hb[i]["p"], None if greedy else hb[i]["q"], hb[i]["ids"], T,
                           seed=21622, round=i, request_id_base=rid0, device=dev,
                           staging=staging)
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()
        E = args.e2e_steps
        etok = 0
        zc_bytes = 0.0
        s0 = torch.cuda.Event(enable_timing=True)
        s1 = torch.cuda.Event(enable_timing=True)
        s0.record()
        for i in range(E):
            h = hb[i % 2]
            Lo, _, so = sd.verify_host(h["p"], None if greedy else h["q"], h["ids"], T,
                                       seed=21622, round=i, request_id_base=rid0, device=dev,
                                       staging=staging)
            etok += int((Lo + 1)[(so & 7) == 0].sum())
            Ln = Lo.numpy()
            # zero copy: the rows the lazy path reads in place + the sampler's stop
            # row pair (p_L, q_L) or bonus row p_k -- a lower bound: ncu shows ~1.1x (rows of the
            # next position that load before a stop lands)
            zc_bytes += float(algorithmic_bytes(Ln, V, k, e, greedy).sum())
            if not greedy and staging.get("p_stage") is None:
                zc_bytes += float(((Ln < k) + 1).sum()) * V * e
        s1.record()
        torch.cuda.synchronize()
        ems = s0.elapsed_time(s1)
        (ems,), (etok_all,) = reduce_max_sum([ems], [etok], dev)
        zero_copy = staging.get("p") is None                         # (verify_host's zero-copy path)
        if zero_copy:
            h2d = int(zc_bytes / E) + hb[0]["ids"].numel() * 4
        else:
            h2d = sum(hb[0][x].numel() * hb[0][x].element_size() for x in ("p", "q", "ids")
                      if hb[0][x] is not None and not (greedy and x == "q"))   # no q at T = 0
        d2h = B * 4 + B * (k + 1) * 4 + B * 4
        e2e = {"value": etok_all / (ems / 1000.0), "unit": UNIT, "h2d_bytes_per_step": h2d,
               "d2h_bytes_per_step": d2h, "steps": E,
               "h2d_mode": ("zero copy: the kernels read the pinned host logits in place over PCIe "
                            "(only the rows the lazy path needs, each once: the sampler reads its "
                            "stop rows from a device stage, sd_verify_staged); bytes = those rows, "
                            "a lower bound" if zero_copy else
                            "pinned host -> device copies of p, q, ids")}

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu:
        d0 = host_batch(batches[0])
        cores = len(os.sched_getaffinity(0))
        rate, info = oracle_rate(d0, T, args.cpu_seconds, 21622, cores)
        # the oracle on one core as well (a shorter bounded sample)
        rate1, info1 = oracle_rate(d0, T, min(5.0, args.cpu_seconds), 21622, 1, per_step=1)
        cpu = {"value": rate, "unit": UNIT, "cores": cores, "kind": "oracle",
               "sample": f"{info['requests']} requests of batch 0 ({info['steps']} calls x "
                         f"{info['per_step']}), {info['seconds']:.1f} s on {cores} threads",
               "single_core": {"value": rate1, "cores": 1,
                               "sample": f"{info1['requests']} requests, {info1['seconds']:.1f} s"},
               "parity_sample": parity_sample(batches[0], d0, T, V, cores)}

    if rank == 0:
        clocks = clk.summary()
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": K,
            "warmup": W, "ms_per_step": ms_max / K, "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": args.dtype, "data": "synthetic",
            "config": config_block(args, c),
            "roofline": {"bound": "hbm", "kernel": kname, "achieved": achieved_gbs,
                         "peak": peak, "peak_kind": peak_kind, "unit": "GB/s",
                         "frac": achieved_gbs / peak, "traffic": traffic,
                         "alg_bytes_per_launch": alg_per_launch,
                         "kernel_ms_mean": kA_mean_ms, "kernel_ms_source": kA_src,
                         "kernel_ms_events": statistics.fmean(kA_ev),
                         "step_gbs": alg_per_launch / (ms_max / K / 1000.0) / 1e9,
                         "step_frac": alg_per_launch / (ms_max / K / 1000.0) / 1e9 / peak},
            "cpu_baseline": cpu,
            "e2e": e2e,
            "gpu_launches": K * pl["launches"],
            "kernel_plan": pl,
            "clocks": clocks,
            "accept": {"mean_L": float(Lh.mean()), "mean_emitted": float((Lh + 1).mean()),
                       "L_hist": np.bincount(Lh.ravel().astype(np.int64), minlength=k + 1).tolist(),
                       "fault_requests": int((~ok).sum())},
        }
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


# --------------------------------------------------------------------------------- star ----
def run_star(args):
    """The 1 -> N-1 star (Alg. 1) on one node: rank 0 is the
    draft, ranks 1..N-1 verify over per-pair NCCL communicators (or --star-loopback N: one process
    plays the draft and N virtual verifiers on one GPU).  Draft service per verifier-round (SURVEY
    8(d) B10): k LM-head-shaped bf16 GEMMs [B, H] x [H, V] (the draft model's cost, S(d) = d t_s,
    Eq. 5) plus sd_draft_sample (NEXT-2) of the round's draft tokens from its q rows.  q rows come
    from a seeded pool both sides regenerate identically (the verifier holds the matching target
    rows), so acceptance follows the workload's kappa.  A step = one round for every (verifier,
    slot) stream; W untimed steps, then K timed ones, each phase drained.  value = verified tokens
    (L+1, all verifiers) / the max over ranks of each rank's CUDA-event window."""
    import numpy as np
    import torch
    import torch.distributed as dist

    import paper_2601_21622_b200 as sd
    from paper_2601_21622_b200 import star
    from workload import make_batch_torch

    rank, world, local = dist_env()
    loop = args.star_loopback > 0
    nver = args.star_loopback if loop else world - 1
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if not loop:
        dist.init_process_group("nccl", device_id=dev)
    c = workload(args)
    V, k, B, T = c["V"], c["k"], c["B"], c["T"]
    # per-verifier batch and agreement (C4: a heterogeneous star; default: all equal)
    lst = lambda txt, cast, dflt: ([cast(x) for x in txt.split(",")] if txt else [dflt])  # noqa: E731
    Bl, Kl = lst(args.batches, int, B), lst(args.kappas, float, c["kappa"] or 30.0)
    Bv = {v: Bl[(v - 1) % len(Bl)] for v in range(1, nver + 1)}
    Kv = {v: Kl[(v - 1) % len(Kl)] for v in range(1, nver + 1)}
    B = max(Bv.values())                                                   # the star's max batch
    tdt = torch.float32 if args.dtype == "f32" else torch.bfloat16
    npool, slots = 2, args.slots
    K, W = args.steps, max(3, args.warmup)

    def pool_batch(v, i):
        return make_batch_torch(V, k, Bv[v], T, Kv[v], c["seed"] + 7919 * v + i, dev,
                                dtype=args.dtype)

    ids_x = star.exchange_ids(rank, world) if not loop else None
    h = star.Star(0 if loop else rank, nver + 1, B, k, V, T, seed=21622, n_slots=slots, dtype=tdt,
                  device=dev, ids=ids_x, transport="loopback" if loop else "nccl",
                  timeout_ms=120000, payload=args.payload, target_ms=args.target_ms)
    rid = lambda v, s: (v << 32) + s * B                                  # noqa: E731
    pidx = lambda r, s: (r + s) % npool                                    # noqa: E731
    total_rounds = W + K
    s_main = torch.cuda.current_stream(dev)
    if rank == 0:
        qpool, ppool = {}, {}
        for v in range(1, nver + 1):
            for i in range(npool):
                bt = pool_batch(v, i)
                qpool[(v, i)] = bt["q"]
                if loop:
                    ppool[(v, i)] = bt["p"]
                del bt
        Wt = (torch.randn(args.draft_hidden, V, device=dev, dtype=torch.bfloat16) * 0.02)
        hid = torch.randn(B, args.draft_hidden, device=dev, dtype=torch.bfloat16)
        bufs = {(v, s): (torch.empty(Bv[v], dtype=torch.int32, device=dev),
                         torch.empty(Bv[v], k + 1, dtype=torch.int32, device=dev))
                for v in range(1, nver + 1) for s in range(slots)}
        drafted = {}
        tok_acc = torch.zeros((), dtype=torch.int64, device=dev)
        per_v = torch.zeros(nver + 1, dtype=torch.int64, device=dev)
        Lhost = {}

        def draft_and_submit(v, s, r):
            q = qpool[(v, pidx(r, s))]
            h.draft_begin(verifier=v)
            for _ in range(k):                                             # S(d) = d t_s
                torch.matmul(hid[:Bv[v]], Wt)
            ids, qm, _ = sd.draft_sample(q, T, seed=21622, round=r, request_id_base=rid(v, s),
                                         want_qmeta=args.payload == "qmeta")
            h.draft_end()
            L, tok = bufs[(v, s)]
            drafted[(v, s)] = (ids, qm, q)                                 # alive until the return
            h.submit(v, s, r, ids, q, L, tok, request_id_base=rid(v, s),
                     p=ppool[(v, pidx(r, s))] if loop else None, qmeta=qm)

        def phase(r0, r1, count):
            nonlocal tok_acc
            for s in range(slots):
                for v in range(1, nver + 1):
                    draft_and_submit(v, s, r0)
            left = nver * slots * (r1 - r0)
            while left:
                got = h.poll(timeout_us=120_000_000)
                if got is None:
                    raise RuntimeError("star: no return within 120 s")
                v, s, r = got
                left -= 1
                L, _ = bufs[(v, s)]
                if count:
                    n = (L + 1).sum()
                    tok_acc += n
                    per_v[v] += n
                    Lhost.setdefault(v, []).append(L.to("cpu", non_blocking=True))
                if r + 1 < r1:
                    draft_and_submit(v, s, r + 1)

        phase(0, W, False)
        torch.cuda.synchronize()
        if not loop:
            dist.barrier()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        with ClockSampler(local) as clk:
            e0.record(s_main)
            phase(W, total_rounds, True)
            e1.record(s_main)
            torch.cuda.synchronize()
        ms = e0.elapsed_time(e1)
        tokens = float(tok_acc.item())
        alg = 0.0                                            # verifier-side algorithmic bytes
        for v, Ls in Lhost.items():
            for Lt in Ls:
                h.observe(v, Lt.numpy())
                alg += float(algorithmic_bytes(Lt.numpy(), V, k, esize(args.dtype), T == 0.0).sum())
        st = h.stats()
        try:
            pred = h.predict(args.o_alone)
        except sd.StarsdError:
            pred = None
        perv = (per_v.cpu().numpy()[1:] / (ms / 1000.0)).tolist()
    else:
        ppool = {i: pool_batch(rank, i)["p"] for i in range(npool)}
        outs = {s: (torch.empty(Bv[rank], dtype=torch.int32, device=dev),
                    torch.empty(Bv[rank], k + 1, dtype=torch.int32, device=dev)) for s in range(slots)}

        def serve_phase(r0, r1):
            for r in range(r0, r1):
                for s in range(slots):
                    # the slot's previous results must have left before its buffers are reused
                    if r > r0:
                        while h.poll(timeout_us=120_000_000) is None:
                            raise RuntimeError("star verifier: send not done within 120 s")
                    L, tok = outs[s]
                    h.serve(s, r, Bv[rank], ppool[pidx(r, s)], L, tok, request_id_base=rid(rank, s))
            for _ in range(slots):
                if h.poll(timeout_us=120_000_000) is None:
                    raise RuntimeError("star verifier: send not done within 120 s")

        serve_phase(0, W)
        torch.cuda.synchronize()
        dist.barrier()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(s_main)
        serve_phase(W, total_rounds)
        e1.record(s_main)
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1)
        tokens = 0.0
    if not loop:
        from paper_2601_21622_b200.dp import reduce_max_sum
        (ms,), (tokens,) = reduce_max_sum([ms], [tokens], dev)
    if rank == 0:
        value = tokens / (ms / 1000.0)
        S_ms = pred["service_ms"] if pred else None
        Z_ms = pred["return_ms"] if pred else None
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": 1 if loop else world,
            "steps": K, "warmup": W, "ms_per_step": ms / K, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": args.dtype, "data": "synthetic",
            "config": {"workload": f"{args.config}: {c['name']}, star 1 -> {nver}"
                                   + (" (loopback on one GPU)" if loop else ""),
                       "vocab": V, "k": k, "batch_per_verifier": [Bv[v] for v in range(1, nver + 1)],
                       "temperature": T, "kappa": [Kv[v] for v in range(1, nver + 1)],
                       "logits": args.dtype, "slots": slots,
                       "payload": args.payload, "target_ms": args.target_ms,
                       "draft_standin": f"{k} x bf16 GEMM [{B},{args.draft_hidden}]x[{args.draft_hidden},{V}]"
                                        " + sd_draft_sample per verifier-round",
                       "parallelism": f"star: rank 0 draft, {nver} verifiers"},
            "star": {"busy_fraction": st["busy_fraction"], "mean_idle_ms": st["mean_idle_ms"],
                     "mean_wait_ms": st["mean_wait_ms"], "rounds": st["rounds"],
                     "per_verifier_tokens_s": perv,
                     "predicted": pred,
                     "closed_form_busy": (min(1.0, nver * S_ms / (S_ms + Z_ms))
                                          if S_ms and Z_ms is not None else None)},
            # the verifiers' HBM roofline averaged over the window: algorithmic bytes of every
            # verify (realized L) / window / verifier GPUs (loopback: one GPU plays
            # all roles, so the fraction also carries the draft's GEMMs and sampling)
            "roofline": {"bound": "hbm", "kernel": "k_row_stats (verifier side, window average)",
                         "achieved": alg / (ms / 1000.0) / 1e9 / (1 if loop else nver),
                         "peak": load_peaks()[0], "peak_kind": load_peaks()[1], "unit": "GB/s",
                         "frac": alg / (ms / 1000.0) / 1e9 / (1 if loop else nver) / load_peaks()[0],
                         "traffic": None, "alg_bytes_per_round": alg / max(1, K)},
            "e2e": None,
            # our kernels in the window: per verifier-round, sd_verify (2) on the verifier and
            # sd_draft_sample (2, + the q-metadata gather with the lazy payload) on the draft
            "gpu_launches": K * nver * slots * (4 + (1 if args.payload == "qmeta" else 0)),
            "clocks": clk.summary(),
        }
        print(json.dumps(line), flush=True)
    h.close()
    if not loop:
        dist.barrier()
        dist.destroy_process_group()


def run_star_trace(args):
    """BASELINE config 5 on one GPU (loopback star, N virtual verifiers): requests arrive by a
    seeded compound-Poisson trace (workload.bursty_trace: bursts at --burst-rate per second per
    verifier, Geometric(--burst-mean) requests per burst, 64..512 tokens each).  Each verifier
    keeps --slots cohorts of up to B requests; a cohort with active requests issues its next round
    when its previous one returned (closed loop), the draft serving rounds FIFO from Q_in
    (Alg. 1); a round's batch is the cohort's current size; each request emits L+1 tokens per
    round until its length is reached.  Reports the draft busy fraction overall and per 100 ms
    window, per-verifier tokens/s and completed requests."""
    import numpy as np
    import torch

    import paper_2601_21622_b200 as sd
    from paper_2601_21622_b200 import star
    from workload import make_batch_torch
    from workload.trace import bursty_trace

    nver = args.star_loopback
    dev = torch.device("cuda", 0)
    torch.cuda.set_device(dev)
    c = workload(args)
    V, k, B, T = c["V"], c["k"], c["B"], c["T"]
    slots = args.slots
    tdt = torch.float32 if args.dtype == "f32" else torch.bfloat16
    h = star.Star(0, nver + 1, B, k, V, T, seed=21622, n_slots=slots, dtype=tdt, device=dev,
                  transport="loopback", timeout_ms=120000, payload=args.payload)
    pool = {v: make_batch_torch(V, k, B, T, c["kappa"] or 30.0, c["seed"] + 7919 * v, dev,
                                dtype=args.dtype) for v in range(1, nver + 1)}
    Wt = torch.randn(args.draft_hidden, V, device=dev, dtype=torch.bfloat16) * 0.02
    hid = torch.randn(B, args.draft_hidden, device=dev, dtype=torch.bfloat16)
    bufs = {(v, s_): (torch.empty(B, dtype=torch.int32, device=dev),
                      torch.empty(B, k + 1, dtype=torch.int32, device=dev))
            for v in range(1, nver + 1) for s_ in range(slots)}
    trace = bursty_trace(nver, args.trace_seconds, burst_rate_hz=args.burst_rate,
                         burst_mean=args.burst_mean)
    nxt = {v: 0 for v in trace}
    pending = {v: [] for v in trace}                                 # arrived, not yet in a cohort
    cohort = {(v, s_): [] for v in trace for s_ in range(slots)}     # [remaining tokens]
    inflight = {(v, s_): None for v in trace for s_ in range(slots)}
    rnd = {(v, s_): 0 for v in trace for s_ in range(slots)}
    tokens = np.zeros(nver + 1)
    done = np.zeros(nver + 1, dtype=np.int64)
    win_tok = {}
    keep = {}

    def submit(v, s_, now):
        n = len(cohort[(v, s_)])
        q = pool[v]["q"][:n]
        h.draft_begin(verifier=v)
        for _ in range(k):                                                 # S(d) = d t_s
            torch.matmul(hid[:n], Wt)
        r = rnd[(v, s_)]
        ids, qm, _ = sd.draft_sample(q, T, seed=21622, round=r, request_id_base=(v << 32) + s_ * B,
                                     want_qmeta=args.payload == "qmeta")
        h.draft_end()
        L, tok = bufs[(v, s_)]
        keep[(v, s_)] = (ids, qm)
        h.submit(v, s_, r, ids, q, L[:n], tok[:n], request_id_base=(v << 32) + s_ * B,
                 p=pool[v]["p"][:n], qmeta=qm)
        inflight[(v, s_)] = n
        rnd[(v, s_)] = r + 1

    t0 = time.perf_counter()
    now_ms = lambda: (time.perf_counter() - t0) * 1000.0                  # noqa: E731
    end_ms = args.trace_seconds * 1000.0
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    with ClockSampler(0) as clk:
        while True:
            t = now_ms()
            if t < end_ms:
                for v in trace:                                           # arrivals wait ...
                    while nxt[v] < len(trace[v]) and trace[v][nxt[v]][0] <= t:
                        pending[v].append(trace[v][nxt[v]][1])
                        nxt[v] += 1
                for (v, s_), n in inflight.items():                       # ... for an idle cohort
                    if n is None:
                        room = B - len(cohort[(v, s_)])
                        cohort[(v, s_)] += pending[v][:room]
                        del pending[v][:room]
                        if cohort[(v, s_)]:
                            submit(v, s_, t)
            elif all(n is None for n in inflight.values()):
                break
            got = h.poll(timeout_us=200)
            while got is not None:
                v, s_, r = got
                n = inflight[(v, s_)]
                Lh = bufs[(v, s_)][0][:n].cpu().numpy()
                rem = cohort[(v, s_)]
                emit = np.minimum(Lh + 1, np.asarray(rem))
                tokens[v] += emit.sum()
                w = int(now_ms() // 100)
                win_tok[w] = win_tok.get(w, 0) + int(emit.sum())
                rem = [x - e for x, e in zip(rem, emit) if x - e > 0]
                done[v] += n - len(rem)
                cohort[(v, s_)] = rem
                inflight[(v, s_)] = None
                got = h.poll(timeout_us=0)
        e1.record()
        torch.cuda.synchronize()
    ms = e0.elapsed_time(e1)
    st = h.stats()
    line = {
        "metric": METRIC, "value": float(tokens.sum()) / (ms / 1000.0), "unit": UNIT, "n_gpus": 1,
        "steps": int(sum(rnd.values())), "warmup": 0, "ms_per_step": ms / max(1, sum(rnd.values())),
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": args.dtype,
        "data": "synthetic",
        "config": {"workload": f"c5: bursty arrival trace, star 1 -> {nver} (loopback on one GPU)",
                   "vocab": V, "k": k, "max_batch_per_cohort": B, "slots": slots,
                   "temperature": T, "kappa": c["kappa"], "payload": args.payload,
                   "trace": {"seconds": args.trace_seconds, "burst_rate_hz": args.burst_rate,
                             "burst_mean": args.burst_mean, "tokens_per_request": "64..512",
                             "requests": int(sum(len(x) for x in trace.values()))}},
        "star": {"busy_fraction": st["busy_fraction"], "mean_wait_ms": st["mean_wait_ms"],
                 "rounds": st["rounds"],
                 "per_verifier_tokens_s": (tokens[1:] / (ms / 1000.0)).tolist(),
                 "completed_requests": done[1:].tolist(),
                 "tokens_per_100ms": [win_tok.get(i, 0) for i in range(int(ms // 100) + 1)]},
        "roofline": None, "e2e": None,
        "gpu_launches": int(sum(rnd.values())) * (4 + (1 if args.payload == "qmeta" else 0)),
        "clocks": clk.summary(),
    }
    print(json.dumps(line), flush=True)
    h.close()


def main():
    args = parse()
    if args.star_loopback > 0 and args.trace_seconds > 0:
        run_star_trace(args)
        return
    if args.impl == "reference":
        run_reference(args)
        return
    world = dist_env()[1]
    if args.star_loopback > 0 or (world > 1 and args.mode in ("auto", "star")):
        run_star(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
