"""C-ABI boundary checks that need no GPU: the library builds, loads, exports every symbol
include/starsd.h declares, and rejects host-checkable bad arguments before touching CUDA."""
import ctypes
import os
import re
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def lib():
    from paper_2601_21622_b200 import build, _lib
    build.build()
    return _lib.load()


def header_functions():
    src = open(os.path.join(ROOT, "include", "starsd.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(sd_[a-z_0-9]+)\s*\(", src)))


def test_header_declares_the_north_star_entry_points():
    fns = header_functions()
    for name in ("sd_verify", "sd_star_round", "sd_verify_workspace_size", "sd_star_create",
                 "sd_star_poll", "sd_star_stats", "sd_star_destroy", "sd_status_string",
                 "sd_last_error"):
        assert name in fns


def test_library_exports_every_declared_symbol(lib):
    from paper_2601_21622_b200 import _lib
    out = subprocess.check_output(["nm", "-D", "--defined-only", _lib.LIB_PATH], text=True)
    exported = set(re.findall(r" T (sd_\w+)", out))
    declared = set(header_functions())
    assert declared <= exported, declared - exported
    assert set(_lib.EXPORTS) == declared


def test_library_is_sm100a_and_uses_bulk_copies(lib):
    from paper_2601_21622_b200 import _lib
    out = subprocess.check_output(["cuobjdump", "--list-elf", _lib.LIB_PATH], text=True)
    assert "sm_100a" in out
    sass = subprocess.check_output(["cuobjdump", "-sass", _lib.LIB_PATH], text=True)
    assert "UBLKCP" in sass          # TMA bulk copy global -> shared
    assert "SYNCS" in sass           # mbarrier transaction waits


def shape(B=4, k=3, V=1000, ld_p=0, ld_q=0, dtype=0):
    from paper_2601_21622_b200._lib import Shape
    return Shape(B, k, V, ld_p, ld_q, dtype)


@pytest.mark.parametrize("sh,T", [
    (dict(k=0), 1.0), (dict(k=32), 1.0), (dict(V=1), 1.0), (dict(B=-1), 1.0),
    (dict(dtype=7), 1.0), (dict(ld_p=999), 1.0), (dict(V=1001, ld_p=1001), 1.0),
    ({}, -1.0), ({}, float("nan")), ({}, float("inf")), ({}, 1e-4),
])
def test_invalid_shapes_rejected_on_host(lib, sh, T):
    n = ctypes.c_size_t()
    s = shape(**sh)
    assert lib.sd_verify_workspace_size(ctypes.byref(s), T, ctypes.byref(n)) == 1
    assert lib.sd_last_error()


def test_workspace_size_is_host_only(lib):
    n = ctypes.c_size_t()
    s = shape(B=128, k=7, V=128256)
    assert lib.sd_verify_workspace_size(ctypes.byref(s), 1.0, ctypes.byref(n)) == 0
    assert 0 < n.value < 64 * 1024 * 1024
    assert n.value % 16 == 0


def test_verify_null_arguments_rejected_before_cuda(lib):
    s = shape()
    ws = ctypes.create_string_buffer(1 << 20)
    # NULL p / q(T>0) / ids / outputs / workspace
    assert lib.sd_verify(None, 16, 16, ctypes.byref(s), 1.0, 0, 0, 0, 16, 16, None, 16, 1 << 20,
                         None) == 1
    assert lib.sd_verify(16, None, 16, ctypes.byref(s), 1.0, 0, 0, 0, 16, 16, None, 16, 1 << 20,
                         None) == 1
    assert lib.sd_verify(16, 16, None, ctypes.byref(s), 1.0, 0, 0, 0, 16, 16, None, 16, 1 << 20,
                         None) == 1
    assert lib.sd_verify(16, 16, 16, ctypes.byref(s), 1.0, 0, 0, 0, None, 16, None, 16, 1 << 20,
                         None) == 1
    assert lib.sd_verify(16, 16, 16, ctypes.byref(s), 1.0, 0, 0, 0, 16, 16, None, None, 1 << 20,
                         None) == 1
    # misaligned p, too-small workspace
    assert lib.sd_verify(17, 16, 16, ctypes.byref(s), 1.0, 0, 0, 0, 16, 16, None, 16, 1 << 20,
                         None) == 1
    assert lib.sd_verify(16, 16, 16, ctypes.byref(s), 1.0, 0, 0, 0, 16, 16, None, 16, 8,
                         None) == 1
    assert b"workspace" in lib.sd_last_error()
    # empty batch is a valid no-op
    s0 = shape(B=0)
    assert lib.sd_verify(16, 16, 16, ctypes.byref(s0), 1.0, 0, 0, 0, 16, 16, None, 16, 0,
                         None) == 0


def test_status_strings(lib):
    assert lib.sd_status_string(0) == b"SD_OK"
    assert lib.sd_status_string(1) == b"SD_ERR_INVALID_ARGUMENT"
    assert lib.sd_status_string(6) == b"SD_ERR_NOT_READY"
    assert b"sm_100a" in lib.sd_version()


def test_product_package_never_imports_the_oracle():
    """The product path must not reference oracle/ (it shares no code with it)."""
    pkg = os.path.join(ROOT, "paper_2601_21622_b200")
    for dirpath, _, files in os.walk(pkg):
        for f in files:
            if f.endswith((".py", ".cu", ".cuh", ".cpp", ".h")):
                src = open(os.path.join(dirpath, f)).read()
                assert "import oracle" not in src and "from oracle" not in src, f
                assert "starsd_ref" not in src, f
    for f in os.listdir(os.path.join(ROOT, "oracle")):
        if f.endswith((".py", ".c", ".h")):
            src = open(os.path.join(ROOT, "oracle", f)).read()
            assert "import paper_2601" not in src and "from paper_2601" not in src, f
            assert not re.search(r'#include\s*[<"][^>"]*starsd\.h', src), f


def test_verify_plan_default_is_two_launch_with_16kb_chunks(lib):
    """sd_verify_plan on the host: the default variant, its launch count and chunking (Llama-3
    shape: V=128256 fp32 -> 32 chunks of 4096 logits = 16 KB, grid (k+1)*B*nch CTAs)."""
    import torch
    import paper_2601_21622_b200 as sd
    pl = sd.plan(128, 7, 128256, 1.0)
    assert pl["variant"] == "two_launch" and pl["launches"] == 2
    assert pl["slice"] == 4096 and pl["ctas"] == 8 * 128 * 32
    assert pl["cluster"] == 0                                  # nch = 32 > 8: cluster-free rows
    # start-ticket deciders; k_sample_req (one CTA per request) launched during the last position
    # wave, plus its completion probe
    assert pl["tagged"] and pl["tail_ctas"] == 129 and pl["options"] == ["early"]
    pg = sd.plan(128, 7, 128256, 0.0)
    assert pg["tail_ctas"] == 1                                # greedy finalize: 128 threads/CTA
    assert pg["slice"] == 8192 and pg["ctas"] == 8 * 128 * 16  # greedy fp32 rows: 32 KB slices
    plb = sd.plan(64, 5, 32000, 0.0, torch.bfloat16)          # bf16: 8192 logits per 16 KB chunk
    assert plb["slice"] == 8192 and plb["ctas"] == 6 * 64 * 4 and plb["cluster"] == 4
    # a cluster covers a whole row of nch <= 8 chunks (power of two, padded with empty chunks)
    assert sd.plan(64, 5, 32000, 1.0)["cluster"] == 8          # nch = 8
    p5 = sd.plan(16, 3, 20000, 1.0)                            # nch = 5 -> 8 (3 empty chunks)
    assert p5["cluster"] == 8 and p5["ctas"] == 4 * 16 * 8
    assert sd.plan(16, 3, 3000, 1.0)["cluster"] == 0           # one chunk per row
    with pytest.raises(sd.StarsdError):
        sd.plan(4, 40, 1000, 1.0)                               # k > 31 rejected on the host


def test_verify_staged_rejects_missing_or_misaligned_stages_on_host(lib):
    """sd_verify_staged validates its stage buffers before any GPU work (T > 0 needs both)."""
    import ctypes
    SD_ERR_INVALID_ARGUMENT = 1
    sh = shape()
    fake = ctypes.c_void_p(0x10000)
    for ps, qs in ((None, None), (fake, None), (None, fake), (ctypes.c_void_p(0x10008), fake)):
        rc = lib.sd_verify_staged(fake, fake, fake, ctypes.byref(sh), 1.0, 0, 0, 0, fake, fake, None,
                                  fake, 1 << 20, ps, qs, None)
        assert rc == SD_ERR_INVALID_ARGUMENT
        assert b"stage" in lib.sd_last_error()
