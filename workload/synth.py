"""Seeded synthetic logits / draft ids (see package docstring; no verify arithmetic here)."""
from __future__ import annotations

import itertools

import numpy as np

# BASELINE.json:configs as concrete workloads (SURVEY.md 8(d) "Configs as concrete workloads").
CONFIGS = {
    "c1": dict(name="tiny exhaustive", V=8, k=4, B=1, T=1.0, kappa=None, seed=21622001),
    "c2": dict(name="Vicuna-7B shape", V=32000, k=5, B=64, T=1.0, kappa=30.0, seed=21622002),
    "c2g": dict(name="Vicuna-7B shape, greedy", V=32000, k=5, B=64, T=0.0, kappa=30.0,
                seed=21622002),
    "c3": dict(name="Llama-3 shape", V=128256, k=7, B=128, T=1.0, kappa=30.0, seed=21622003),
    "c3g": dict(name="Llama-3 shape, greedy", V=128256, k=7, B=128, T=0.0, kappa=30.0,
                seed=21622003),
    "c5": dict(name="bursty trace row shape", V=128256, k=5, B=128, T=1.0, kappa=30.0,
               seed=21622005),
}

ZIPF_S = 1.2      # target prior exponent
TARGET_A = 10.0   # target Dirichlet concentration
CLAMP = -1.0e4    # logits are clamped to >= CLAMP (finite)


def bf16_bits(x: np.ndarray) -> np.ndarray:
    """Round fp32 -> bf16 (round-to-nearest-even), returned as raw uint16 bits."""
    u = np.ascontiguousarray(x, np.float32).view(np.uint32).astype(np.uint64)
    r = (u + 0x7FFF + ((u >> 16) & 1)) >> 16
    return r.astype(np.uint16)


def log_dirichlet(alpha: np.ndarray, rng: np.random.Generator) -> np.ndarray:
    """log of a Dirichlet(alpha) draw along the last axis, in log space so that tiny
    concentrations never underflow: log G(a) = log G(a+1) + log(U)/a."""
    alpha = np.asarray(alpha, np.float64)
    g1 = rng.standard_gamma(alpha + 1.0)
    u = rng.random(alpha.shape)
    with np.errstate(divide="ignore"):
        lg = np.log(g1) + np.log(u) / alpha
    m = lg.max(axis=-1, keepdims=True)
    return lg - (m + np.log(np.exp(lg - m).sum(axis=-1, keepdims=True)))


def _zipf_prior(rows: int, V: int, rng: np.random.Generator) -> np.ndarray:
    w = np.arange(1, V + 1, dtype=np.float64) ** (-ZIPF_S)
    w /= w.sum()
    out = np.empty((rows, V))
    for r in range(rows):
        out[r] = w[rng.permutation(V)]
    return out


def _gumbel_argmax(z: np.ndarray, T: float, rng: np.random.Generator) -> np.ndarray:
    """Draft-side sample x ~ softmax(z/T) (Gumbel-max), or argmax z when T == 0."""
    if T == 0.0:
        return np.argmax(z, axis=-1).astype(np.int32)
    g = -np.log(-np.log(rng.random(z.shape)))
    return np.argmax(z.astype(np.float64) / T + g, axis=-1).astype(np.int32)


def make_batch(V: int, k: int, B: int, T: float, kappa: float, seed: int, dtype: str = "f32",
               ld: int | None = None):
    """Independent rows (C-15).  Returns dict(p [B,k+1,ld], q [B,k,ld], ids [B,k], V, k, T).

    dtype "f32" -> float32 logits; "bf16" -> uint16 raw bf16 bits (ids drawn from the bf16
    values, which are what the verifier sees).  ld >= V pads rows (padding filled with NaN so
    a kernel that reads it is caught)."""
    rng = np.random.default_rng(seed)
    rows_p = B * (k + 1)
    logp = log_dirichlet(TARGET_A * _zipf_prior(rows_p, V, rng), rng).reshape(B, k + 1, V)
    logq = log_dirichlet(kappa * np.exp(logp[:, :k, :]), rng)
    zp = np.maximum(logp, CLAMP).astype(np.float32)
    zq = np.maximum(logq, CLAMP).astype(np.float32)
    if dtype == "bf16":
        zp_b, zq_b = bf16_bits(zp), bf16_bits(zq)
        zq_seen = (zq_b.astype(np.uint32) << 16).view(np.float32)
        ids = _gumbel_argmax(zq_seen, T, np.random.default_rng(seed + 1))
        zp, zq = zp_b, zq_b
    else:
        ids = _gumbel_argmax(zq, T, np.random.default_rng(seed + 1))
    if ld is not None and ld > V:
        pad = np.float32(np.nan) if dtype == "f32" else np.uint16(0x7FC0)
        zp2 = np.full((B, k + 1, ld), pad, dtype=zp.dtype)
        zq2 = np.full((B, k, ld), pad, dtype=zq.dtype)
        zp2[..., :V] = zp
        zq2[..., :V] = zq
        zp, zq = zp2, zq2
    return dict(p=zp, q=zq, ids=ids, V=V, k=k, T=T)


def make_batch_torch(V: int, k: int, B: int, T: float, kappa: float, seed: int, device,
                     dtype: str = "f32"):
    """Same recipe as make_batch, drawn with torch on `device` (fast for the 128K vocabulary).
    Not bit-identical to make_batch (different RNG); both are seeded and deterministic."""
    import torch

    g = torch.Generator(device=device)
    g.manual_seed(seed)
    rows_p = B * (k + 1)
    w = torch.arange(1, V + 1, device=device, dtype=torch.float64).pow(-ZIPF_S)
    w = w / w.sum()
    perm = torch.argsort(torch.rand(rows_p, V, generator=g, device=device), dim=-1)
    alpha = (TARGET_A * w)[perm]

    def logdir(a):
        g1 = torch._standard_gamma(a + 1.0, generator=g)
        u = torch.rand(a.shape, generator=g, device=device, dtype=torch.float64)
        lg = torch.log(g1) + torch.log(u) / a
        return lg - torch.logsumexp(lg, dim=-1, keepdim=True)

    logp = logdir(alpha).reshape(B, k + 1, V)
    del alpha, perm
    logq = logdir(kappa * torch.exp(logp[:, :k, :]))
    zp = torch.clamp(logp, min=CLAMP).float()
    zq = torch.clamp(logq, min=CLAMP).float()
    del logp, logq
    if dtype == "bf16":
        zp, zq = zp.bfloat16(), zq.bfloat16()
    zsee = zq.float()
    if T == 0.0:
        ids = torch.argmax(zsee, dim=-1)
    else:
        u = torch.rand(zsee.shape, generator=g, device=device, dtype=torch.float64)
        ids = torch.argmax(zsee.double() / T - torch.log(-torch.log(u)), dim=-1)
    return dict(p=zp.contiguous(), q=zq.contiguous(), ids=ids.to(torch.int32).contiguous(),
                V=V, k=k, T=T)


def make_tiny_tables(V: int = 8, k: int = 4, seed: int = 21622001, alpha: float = 1.0):
    """Prefix-conditioned tables for the tiny exhaustive config (C1): one target logit row per
    prefix of length 0..k and one draft row per prefix of length 0..k-1, each
    log-Dirichlet(alpha * 1)."""
    rng = np.random.default_rng(seed)
    P, Q = {}, {}
    for n in range(k + 1):
        for pre in itertools.product(range(V), repeat=n):
            P[pre] = np.maximum(log_dirichlet(np.full(V, alpha), rng), CLAMP).astype(np.float32)
    for n in range(k):
        for pre in itertools.product(range(V), repeat=n):
            Q[pre] = np.maximum(log_dirichlet(np.full(V, alpha), rng), CLAMP).astype(np.float32)
    return P, Q


def tiny_batch(P, Q, paths):
    """Rows along the given draft paths: p[b][j] = P[path[:j]], q[b][j] = Q[path[:j]]."""
    paths = np.asarray(paths, np.int32)
    B, k = paths.shape
    V = len(next(iter(P.values())))
    p = np.empty((B, k + 1, V), np.float32)
    q = np.empty((B, k, V), np.float32)
    for b in range(B):
        pre = tuple(int(x) for x in paths[b])
        for j in range(k + 1):
            p[b, j] = P[pre[:j]]
        for j in range(k):
            q[b, j] = Q[pre[:j]]
    return p, q
