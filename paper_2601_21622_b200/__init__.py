"""paper_2601_21622_b200 -- B200-native StarSD verify path (arXiv 2601.21622).

Thin Python binding over libstarsd.so (include/starsd.h).  This module only marshals torch
tensors into the C ABI (pointers, shapes, the current CUDA stream); every step of the verify
path runs in the sm_100a kernels.  PyTorch provides device memory and streams, nothing else.
"""
from __future__ import annotations

import ctypes

import torch

from . import _lib
from ._lib import StarsdError, check

__all__ = ["verify", "verify_qmeta", "tree_verify", "verify_host", "verify_trace", "draft_sample", "draft_qmeta",
           "qmeta_fields", "workspace_size", "draft_workspace_size", "plan", "philox_words",
           "Workspace", "StarsdError", "version"]

FAULT_BAD_DRAFT_ID, FAULT_NONFINITE, FAULT_EMPTY_ROW = 1, 2, 4
FAULT_ZERO_Q, FAULT_ZERO_RESIDUAL, FAULT_PROTOCOL = 8, 16, 32
HARD_FAULTS = FAULT_BAD_DRAFT_ID | FAULT_NONFINITE | FAULT_EMPTY_ROW | FAULT_PROTOCOL


def version() -> str:
    return _lib.load().sd_version().decode()


def _dtype_code(t: torch.Tensor) -> int:
    if t.dtype == torch.float32:
        return _lib.SD_DTYPE_F32
    if t.dtype == torch.bfloat16:
        return _lib.SD_DTYPE_BF16
    raise TypeError(f"logits must be float32 or bfloat16, got {t.dtype}")


def _shape(batch, k, vocab, ld_p, ld_q, dtype_code) -> _lib.Shape:
    return _lib.Shape(batch, k, vocab, ld_p, ld_q, dtype_code)


def workspace_size(batch: int, k: int, vocab: int, temperature: float,
                   dtype: torch.dtype = torch.float32) -> int:
    code = _lib.SD_DTYPE_F32 if dtype == torch.float32 else _lib.SD_DTYPE_BF16
    n = ctypes.c_size_t()
    per16 = 4 if code == _lib.SD_DTYPE_F32 else 8          # elements per 16 bytes
    ld = (vocab + per16 - 1) // per16 * per16              # the size does not depend on ld
    sh = _shape(batch, k, vocab, ld, ld, code)
    check(_lib.load().sd_verify_workspace_size(ctypes.byref(sh), float(temperature),
                                               ctypes.byref(n)), "sd_verify_workspace_size")
    return n.value


def plan(batch: int, k: int, vocab: int, temperature: float,
         dtype: torch.dtype = torch.float32) -> dict:
    """How sd_verify runs this shape (sd_verify_plan): kernel variant, launches per call,
    cluster size, logits per CTA slice, CTAs per launch."""
    code = _lib.SD_DTYPE_F32 if dtype == torch.float32 else _lib.SD_DTYPE_BF16
    per16 = 4 if code == _lib.SD_DTYPE_F32 else 8
    ld = (vocab + per16 - 1) // per16 * per16
    sh = _shape(batch, k, vocab, ld, ld, code)
    out = _lib.Plan()
    check(_lib.load().sd_verify_plan(ctypes.byref(sh), float(temperature), ctypes.byref(out)),
          "sd_verify_plan")
    return {"variant": _lib.VARIANT_NAMES.get(out.variant, str(out.variant)),
            "launches": out.launches, "cluster": out.cluster, "slice": out.slice,
            "ctas": out.ctas, "tail_ctas": out.tail_ctas, "tagged": bool(out.tagged),
            "options": [n for bit, n in _lib.PLAN_OPTIONS.items() if out.options & bit]}


class Workspace:
    """A zero-filled device workspace (zero-filled on `stream`, default: the current stream, so
    the fill is ordered before the calls that use it there); sd_verify leaves it zero-filled after
    every call and re-zeroes what it needs when the shape changes (include/starsd.h)."""

    def __init__(self, batch, k, vocab, temperature, dtype=torch.float32, device=None,
                 stream: torch.cuda.Stream | None = None):
        self.nbytes = workspace_size(batch, k, vocab, temperature, dtype)
        with torch.cuda.stream(stream) if stream is not None else _nullctx():
            self.buf = torch.zeros(max(self.nbytes, 16), dtype=torch.uint8, device=device)


class _nullctx:
    def __enter__(self):
        return self

    def __exit__(self, *a):
        return False


_ws_cache: dict = {}


def _workspace_for(device, stream, batch, k, vocab, temperature, dtype) -> Workspace:
    """One cached workspace per (device, stream, shape): calls on different streams never share
    one (a workspace must not serve two calls that may run concurrently)."""
    key = (str(device), stream.cuda_stream, batch, k, vocab, temperature == 0.0, dtype)
    ws = _ws_cache.get(key)
    if ws is None:
        ws = Workspace(batch, k, vocab, temperature, dtype, device, stream)
        _ws_cache[key] = ws
    return ws


def verify(p: torch.Tensor, q: torch.Tensor | None, ids: torch.Tensor, temperature: float,
           seed: int = 0, round: int = 0, request_id_base: int = 0, vocab: int | None = None,
           out: tuple | None = None, workspace: Workspace | None = None,
           stream: torch.cuda.Stream | None = None):
    """One batched verify step (sd_verify).  p: [B, k+1, ld] and q: [B, k, ld] CUDA tensors
    (float32 or bfloat16, rows contiguous), ids: [B, k] int32.  Returns (accept_len [B],
    tokens [B, k+1], status [B]) int32 CUDA tensors, ordered on `stream` (default: current)."""
    if not p.is_cuda:
        raise StarsdError("verify(): tensors must be CUDA tensors (use verify_host for host data)")
    B, k1, ld_p = p.shape
    k = k1 - 1
    if ids.shape != (B, k) or ids.dtype != torch.int32 or not ids.is_contiguous():
        raise StarsdError("ids must be a contiguous int32 [B, k] tensor")
    if p.stride(-1) != 1 or p.stride(-2) != ld_p or p.stride(0) != k1 * ld_p:
        raise StarsdError("p must be contiguous [B, k+1, ld]")
    code = _dtype_code(p)
    ld_q = 0
    qptr = None
    if q is not None:
        if q.dtype != p.dtype or q.shape[:2] != (B, k) or q.stride(-1) != 1:
            raise StarsdError("q must be [B, k, ld] with the dtype of p")
        ld_q = q.shape[-1]
        if q.stride(-2) != ld_q or q.stride(0) != k * ld_q:
            raise StarsdError("q must be contiguous [B, k, ld]")
        qptr = q.data_ptr()
    V = ld_p if vocab is None else vocab
    if out is None:
        L = torch.empty(B, dtype=torch.int32, device=p.device)
        tok = torch.empty(B, k + 1, dtype=torch.int32, device=p.device)
        st = torch.empty(B, dtype=torch.int32, device=p.device)
    else:
        L, tok, st = out
    s = stream if stream is not None else torch.cuda.current_stream(p.device)
    ws = workspace or _workspace_for(p.device, s, B, k, V, float(temperature), p.dtype)
    sh = _shape(B, k, V, ld_p, ld_q, code)
    check(_lib.load().sd_verify(p.data_ptr(), qptr, ids.data_ptr(), ctypes.byref(sh),
                                float(temperature), seed & (2**64 - 1), round & (2**64 - 1),
                                request_id_base & (2**64 - 1), L.data_ptr(), tok.data_ptr(),
                                st.data_ptr() if st is not None else None, ws.buf.data_ptr(),
                                ws.nbytes, s.cuda_stream), "sd_verify")
    return L, tok, st


def _check_q(q: torch.Tensor):
    if q.dim() != 3 or q.stride(-1) != 1 or q.stride(-2) != q.shape[-1] or \
            q.stride(0) != q.shape[1] * q.shape[-1]:
        raise StarsdError("q must be a contiguous [B, k, ld] tensor")
    return _dtype_code(q)


def draft_workspace_size(batch: int, k: int, vocab: int, temperature: float,
                         dtype: torch.dtype = torch.float32) -> int:
    code = _lib.SD_DTYPE_F32 if dtype == torch.float32 else _lib.SD_DTYPE_BF16
    per16 = 4 if code == _lib.SD_DTYPE_F32 else 8
    ld = (vocab + per16 - 1) // per16 * per16
    n = ctypes.c_size_t()
    check(_lib.load().sd_draft_workspace_size(ctypes.byref(_shape(batch, k, vocab, ld, ld, code)),
                                              float(temperature), ctypes.byref(n)),
          "sd_draft_workspace_size")
    return n.value


class DraftWorkspace(Workspace):
    def __init__(self, batch, k, vocab, temperature, dtype=torch.float32, device=None, stream=None):
        self.nbytes = draft_workspace_size(batch, k, vocab, temperature, dtype)
        with torch.cuda.stream(stream) if stream is not None else _nullctx():
            self.buf = torch.zeros(max(self.nbytes, 16), dtype=torch.uint8, device=device)


_dws_cache: dict = {}


def _draft_ws(q, stream, T):
    B, k, V = q.shape
    key = (str(q.device), stream.cuda_stream, B, k, V, T == 0.0, q.dtype)
    ws = _dws_cache.get(key)
    if ws is None:
        ws = DraftWorkspace(B, k, V, T, q.dtype, q.device, stream)
        _dws_cache[key] = ws
    return ws


def draft_sample(q: torch.Tensor, temperature: float, seed: int = 0, round: int = 0,
                 request_id_base: int = 0, vocab: int | None = None, want_qmeta: bool = True,
                 workspace=None, stream: torch.cuda.Stream | None = None):
    """sd_draft_sample (NEXT-2): x_j ~ softmax(q[b, j] / T) for every (b, j).  q: [B, k, ld] CUDA
    float32/bfloat16.  Returns (ids [B, k] int32, qmeta [B, k, 3] int64 holding sd_qmeta or None,
    status [B, k] int32)."""
    code = _check_q(q)
    B, k, ld = q.shape
    V = ld if vocab is None else vocab
    ids = torch.empty(B, k, dtype=torch.int32, device=q.device)
    qm = torch.empty(B, k, 3, dtype=torch.int64, device=q.device) if want_qmeta else None
    st = torch.empty(B, k, dtype=torch.int32, device=q.device)
    s = stream if stream is not None else torch.cuda.current_stream(q.device)
    ws = workspace or _draft_ws(q, s, float(temperature))
    sh = _shape(B, k, V, ld, ld, code)
    check(_lib.load().sd_draft_sample(q.data_ptr(), ctypes.byref(sh), float(temperature),
                                      seed & (2**64 - 1), round & (2**64 - 1),
                                      request_id_base & (2**64 - 1), ids.data_ptr(),
                                      qm.data_ptr() if qm is not None else None, st.data_ptr(),
                                      ws.buf.data_ptr(), ws.nbytes, s.cuda_stream), "sd_draft_sample")
    return ids, qm, st


def draft_qmeta(q: torch.Tensor, ids: torch.Tensor, temperature: float, vocab: int | None = None,
                workspace=None, stream: torch.cuda.Stream | None = None) -> torch.Tensor:
    """sd_draft_qmeta: the sd_qmeta [B, k] (as int64 [B, k, 3]) of given draft tokens."""
    code = _check_q(q)
    B, k, ld = q.shape
    V = ld if vocab is None else vocab
    if ids.shape != (B, k) or ids.dtype != torch.int32 or not ids.is_contiguous():
        raise StarsdError("ids must be a contiguous int32 [B, k] tensor")
    qm = torch.empty(B, k, 3, dtype=torch.int64, device=q.device)
    s = stream if stream is not None else torch.cuda.current_stream(q.device)
    ws = workspace or _draft_ws(q, s, float(temperature))
    sh = _shape(B, k, V, ld, ld, code)
    check(_lib.load().sd_draft_qmeta(q.data_ptr(), ids.data_ptr(), ctypes.byref(sh),
                                     float(temperature), qm.data_ptr(), ws.buf.data_ptr(),
                                     ws.nbytes, s.cuda_stream), "sd_draft_qmeta")
    return qm


def qmeta_fields(qm: torch.Tensor) -> dict:
    """Decode sd_qmeta records (int64 [..., 3]) into S (float64), D, zx (float32), status."""
    flat = qm.reshape(-1, 3).contiguous()
    S = flat[:, 0].view(torch.float64)
    DZ = flat[:, 1].contiguous().view(torch.float32).reshape(-1, 2)
    st = flat[:, 2].contiguous().view(torch.int32).reshape(-1, 2)[:, 0]
    shp = qm.shape[:-1]
    return {"S": S.reshape(shp), "D": DZ[:, 0].reshape(shp), "zx": DZ[:, 1].reshape(shp),
            "status": st.reshape(shp)}


def verify_qmeta(p: torch.Tensor, q: torch.Tensor, qmeta: torch.Tensor, ids: torch.Tensor,
                 temperature: float, seed: int = 0, round: int = 0, request_id_base: int = 0,
                 vocab: int | None = None, out: tuple | None = None,
                 workspace: Workspace | None = None, stream: torch.cuda.Stream | None = None):
    """sd_verify_qmeta (NEXT-1): verify with the draft rows as metadata; q [B, k, ld] is read only
    at each request's stop position.  Same results as verify() on the same rows."""
    B, k1, ld_p = p.shape
    k = k1 - 1
    if ids.shape != (B, k) or ids.dtype != torch.int32 or not ids.is_contiguous():
        raise StarsdError("ids must be a contiguous int32 [B, k] tensor")
    if p.stride(-1) != 1 or p.stride(-2) != ld_p or p.stride(0) != k1 * ld_p:
        raise StarsdError("p must be contiguous [B, k+1, ld]")
    code = _dtype_code(p)
    _check_q(q)
    if qmeta.shape != (B, k, 3) or qmeta.dtype != torch.int64 or not qmeta.is_contiguous():
        raise StarsdError("qmeta must be int64 [B, k, 3] (sd_qmeta records)")
    V = ld_p if vocab is None else vocab
    if out is None:
        out = (torch.empty(B, dtype=torch.int32, device=p.device),
               torch.empty(B, k + 1, dtype=torch.int32, device=p.device),
               torch.empty(B, dtype=torch.int32, device=p.device))
    L, tok, st = out
    s = stream if stream is not None else torch.cuda.current_stream(p.device)
    ws = workspace or _workspace_for(p.device, s, B, k, V, float(temperature), p.dtype)
    sh = _shape(B, k, V, ld_p, q.shape[-1], code)
    check(_lib.load().sd_verify_qmeta(p.data_ptr(), q.data_ptr(), qmeta.data_ptr(), ids.data_ptr(),
                                      ctypes.byref(sh), float(temperature), seed & (2**64 - 1),
                                      round & (2**64 - 1), request_id_base & (2**64 - 1),
                                      L.data_ptr(), tok.data_ptr(), st.data_ptr(),
                                      ws.buf.data_ptr(), ws.nbytes, s.cuda_stream),
          "sd_verify_qmeta")
    return L, tok, st


def tree_verify(p: torch.Tensor, q: torch.Tensor | None, tree_tokens: torch.Tensor, branching: int,
                temperature: float, seed: int = 0, round: int = 0, request_id_base: int = 0,
                vocab: int | None = None, stream: torch.cuda.Stream | None = None):
    """sd_tree_verify (NEXT-3): p [B, N, ld], q [B, N_int, ld] (None at T = 0), tree_tokens
    [B, N] int32 for full `branching`-ary trees of depth d in level order.  Returns (accept_len
    [B], tokens [B, d+1], status [B], stop node [B])."""
    B, N, ld_p = p.shape
    m = branching
    d, n, w = 0, 1, 1
    while n < N:
        w *= m
        n += w
        d += 1
    if n != N or d < 1:
        raise StarsdError(f"p holds {N} nodes: not a full {m}-ary tree")
    if tree_tokens.shape != (B, N) or tree_tokens.dtype != torch.int32 or not tree_tokens.is_contiguous():
        raise StarsdError("tree_tokens must be a contiguous int32 [B, N] tensor")
    code = _dtype_code(p)
    ld_q = q.shape[-1] if q is not None else ld_p
    V = ld_p if vocab is None else vocab
    L = torch.empty(B, dtype=torch.int32, device=p.device)
    tok = torch.empty(B, d + 1, dtype=torch.int32, device=p.device)
    st = torch.empty(B, dtype=torch.int32, device=p.device)
    node = torch.empty(B, dtype=torch.int32, device=p.device)
    s = stream if stream is not None else torch.cuda.current_stream(p.device)
    sh = _shape(B, d, V, ld_p, ld_q, code)
    check(_lib.load().sd_tree_verify(p.data_ptr(), q.data_ptr() if q is not None else None,
                                     tree_tokens.data_ptr(), ctypes.byref(sh), m, float(temperature),
                                     seed & (2**64 - 1), round & (2**64 - 1),
                                     request_id_base & (2**64 - 1), L.data_ptr(), tok.data_ptr(),
                                     st.data_ptr(), node.data_ptr(), s.cuda_stream), "sd_tree_verify")
    return L, tok, st, node


def verify_host(p: torch.Tensor, q: torch.Tensor | None, ids: torch.Tensor, temperature: float,
                seed: int = 0, round: int = 0, request_id_base: int = 0,
                device: torch.device | str = "cuda", staging: dict | None = None,
                zero_copy: bool = True):
    """End-to-end call on HOST tensors.  Pinned logits (zero_copy, the default) are read by the
    kernels in place: pinned memory is mapped into the device's address space, so sd_verify's bulk
    copies pull over PCIe only the rows the lazy path needs (include/starsd.h).  Otherwise (or
    unpinned logits) the logits are copied to the device first.  The draft ids go to the device,
    the results come back, then a stream synchronize.  `staging` (optional dict) caches the device
    buffers between calls."""
    dev = torch.device(device)
    st = staging if staging is not None else {}
    zc = zero_copy and p.is_pinned() and (q is None or q.is_pinned())
    sig = (tuple(p.shape), p.dtype, None if q is None else (tuple(q.shape), q.dtype), tuple(ids.shape), zc)
    if st.get("sig") != sig:
        st["sig"] = sig
        st["p"] = None if zc else torch.empty(p.shape, dtype=p.dtype, device=dev)
        st["q"] = torch.empty(q.shape, dtype=q.dtype, device=dev) if q is not None and not zc else None
        # zero copy, sampled: device stages the statistics pass fills with the rows it reads, so
        # the sampler's stop rows do not cross PCIe twice (sd_verify_staged)
        st["p_stage"] = torch.empty(p.shape, dtype=p.dtype, device=dev) if zc and q is not None else None
        st["q_stage"] = torch.empty(q.shape, dtype=q.dtype, device=dev) if zc and q is not None else None
        st["ids"] = torch.empty(ids.shape, dtype=torch.int32, device=dev)
        B, k = ids.shape
        st["out"] = (torch.empty(B, dtype=torch.int32, device=dev),
                     torch.empty(B, k + 1, dtype=torch.int32, device=dev),
                     torch.empty(B, dtype=torch.int32, device=dev))
        st["host_out"] = tuple(torch.empty(t.shape, dtype=t.dtype, pin_memory=True)
                               for t in st["out"])
    st["ids"].copy_(ids, non_blocking=True)
    if zc:
        _verify_ptrs(p, q, st["ids"], temperature, seed, round, request_id_base, st["out"], dev,
                     st["p_stage"], st["q_stage"])
    else:
        st["p"].copy_(p, non_blocking=True)
        if q is not None:
            st["q"].copy_(q, non_blocking=True)
        verify(st["p"], st["q"], st["ids"], temperature, seed, round, request_id_base,
               out=st["out"])
    for h, d in zip(st["host_out"], st["out"]):
        h.copy_(d, non_blocking=True)
    torch.cuda.current_stream(dev).synchronize()
    return st["host_out"]


def _verify_ptrs(p, q, ids, temperature, seed, round, request_id_base, out, dev, p_stage=None,
                 q_stage=None):
    """sd_verify / sd_verify_staged on pinned host logits (zero copy): the same marshalling as
    verify()."""
    B, k1, ld_p = p.shape
    k = k1 - 1
    if p.stride(-1) != 1 or p.stride(-2) != ld_p or p.stride(0) != k1 * ld_p:
        raise StarsdError("p must be contiguous [B, k+1, ld]")
    ld_q = q.shape[-1] if q is not None else 0
    if q is not None and (q.stride(-1) != 1 or q.stride(-2) != ld_q or q.stride(0) != k * ld_q):
        raise StarsdError("q must be contiguous [B, k, ld]")
    s = torch.cuda.current_stream(dev)
    ws = _workspace_for(dev, s, B, k, ld_p, float(temperature), p.dtype)
    sh = _shape(B, k, ld_p, ld_p, ld_q, _dtype_code(p))
    L, tok, status = out
    args = (p.data_ptr(), q.data_ptr() if q is not None else None, ids.data_ptr(), ctypes.byref(sh),
            float(temperature), seed & (2**64 - 1), round & (2**64 - 1),
            request_id_base & (2**64 - 1), L.data_ptr(), tok.data_ptr(), status.data_ptr(),
            ws.buf.data_ptr(), ws.nbytes)
    if p_stage is not None and temperature != 0.0:
        check(_lib.load().sd_verify_staged(*args, p_stage.data_ptr(), q_stage.data_ptr(),
                                           s.cuda_stream), "sd_verify_staged")
    else:
        check(_lib.load().sd_verify(*args, s.cuda_stream), "sd_verify (zero copy)")


def verify_trace(p: torch.Tensor, accept_len: torch.Tensor, temperature: float,
                 workspace: Workspace, vocab: int | None = None, ld_q: int | None = None,
                 stream: torch.cuda.Stream | None = None) -> dict:
    """sd_verify_trace: the fp64 statistics the last sampled sd_verify call on `workspace`
    decided with (lam_p [B, k+1], lam_q [B, k], a [B, k], R [B]; NaN where not reached)."""
    B, k1, ld_p = p.shape
    k = k1 - 1
    V = ld_p if vocab is None else vocab
    sh = _shape(B, k, V, ld_p, ld_q if ld_q is not None else ld_p, _dtype_code(p))
    dev = p.device
    out = {"lam_p": torch.empty(B, k + 1, dtype=torch.float64, device=dev),
           "lam_q": torch.empty(B, k, dtype=torch.float64, device=dev),
           "a": torch.empty(B, k, dtype=torch.float64, device=dev),
           "R": torch.empty(B, dtype=torch.float64, device=dev)}
    s = stream if stream is not None else torch.cuda.current_stream(dev)
    check(_lib.load().sd_verify_trace(ctypes.byref(sh), float(temperature), workspace.buf.data_ptr(),
                                      accept_len.data_ptr(), out["lam_p"].data_ptr(),
                                      out["lam_q"].data_ptr(), out["a"].data_ptr(),
                                      out["R"].data_ptr(), s.cuda_stream), "sd_verify_trace")
    return out


def philox_words(seed: int, round: int, pos: torch.Tensor, rid: torch.Tensor) -> torch.Tensor:
    """The four Philox4x32-10 words per (pos, rid) the verify step draws from (CUDA tensors:
    pos int32/uint32 [n], rid int64 [n]).  Returns int64 [n, 4] holding the uint32 words."""
    n = pos.numel()
    out = torch.empty(n, 4, dtype=torch.int32, device=pos.device)
    s = torch.cuda.current_stream(pos.device)
    check(_lib.load().sd_philox_uniforms(seed & (2**64 - 1), round & (2**64 - 1),
                                         pos.contiguous().data_ptr(), rid.contiguous().data_ptr(),
                                         n, out.data_ptr(), s.cuda_stream), "sd_philox_uniforms")
    return out.to(torch.int64) & 0xFFFFFFFF
