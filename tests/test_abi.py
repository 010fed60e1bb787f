"""CPU-side checks of the C ABI: the library loads, exports every symbol include/mosaicbert.h
declares, and the host-only entry points behave (no GPU needed: nothing here launches a kernel)."""
import ctypes
import os
import re
import subprocess

import numpy as np
import pytest

import oracle as O

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "mosaicbert.h")
LIB = os.path.join(ROOT, "paper_2312_17482_b200", "libmosaicbert.so")


@pytest.fixture(scope="module")
def lib():
    if not os.path.exists(LIB):
        from paper_2312_17482_b200 import build
        build.build(verbose=False)
    from paper_2312_17482_b200 import _lib
    return _lib.lib()


def declared_symbols():
    txt = open(HEADER).read()
    return sorted(set(re.findall(r"MB_API\s+[\w\s\*]*?\b(mb_\w+)\s*\(", txt)))


def test_header_declares_abi():
    syms = declared_symbols()
    for s in ("mb_unpad_index", "mb_encoder_forward", "mb_encoder_backward", "mb_mlm_loss", "mb_alibi_slopes",
              "mb_dropout_mask",
              "mb_gather_rows", "mb_scatter_rows", "mb_embed_forward", "mb_embed_backward"):
        assert s in syms


def test_library_exports_every_declared_symbol(lib):
    out = subprocess.run(["nm", "-D", "--defined-only", LIB], capture_output=True, text=True).stdout
    exported = set(re.findall(r"\sT\s(mb_\w+)", out))
    missing = [s for s in declared_symbols() if s not in exported]
    assert not missing, missing
    from paper_2312_17482_b200 import _lib
    assert set(_lib.exported_symbols()) <= exported


def test_sass_is_sm100a_tcgen05(lib):
    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "-sass", LIB], capture_output=True, text=True).stdout
    assert "sm_100a" in out
    for mnemonic in ("UTCHMMA", "UTMALDG", "LDTM"):  # tcgen05.mma, TMA loads, tcgen05.ld
        assert mnemonic in out, mnemonic


@pytest.mark.parametrize("n", [1, 2, 8, 12, 16, 24])
def test_alibi_slopes_bitexact_vs_oracle(lib, n):
    from paper_2312_17482_b200 import _lib
    got = _lib.alibi_slopes(n)
    want = O.alibi_slopes(n).astype(np.float32)  # correctly rounded fp32 of the closed form
    assert got.dtype == np.float32 and np.array_equal(got, want)


def test_host_argument_errors(lib):
    out = np.zeros(4, np.float32)
    assert lib.mb_alibi_slopes(0, out.ctypes.data) == 2  # MB_ERR_CONFIG
    assert lib.mb_alibi_slopes(4, None) == 1
    assert lib.mb_unpad_index(None, None, 0, 1, 1, None, None, None, None, 0, None) == 1
    assert lib.mb_unpad_index(1, 1, 0, 1, 1, 1, 1, 1, None, 0, None) == 2  # ids given, vocab < 1
    assert lib.mb_mlm_select(None, None, 0, 1, None, None, None, None, None, 0, None) == 1
    assert lib.mb_loss_normalize(None, None, 1.0, None, None, None) == 1
    assert lib.mb_gemm(4, 4, 4, None, 8, 0, None, 8, 0, None, 8, 0, None, None, 0, None, 0, None) == 1
    from paper_2312_17482_b200 import _lib
    d = _lib.dims(96, 5, 256, 128)  # hidden % heads != 0
    lp = _lib.LayerPtrs()
    pk = _lib.Packed(1, 1, 1, 1)
    assert lib.mb_encoder_forward(ctypes.byref(d), ctypes.byref(lp), ctypes.byref(pk), 1, 1, 1, 1, None, None) == 2
    d = _lib.dims(64, 1, 256, 128)  # head_dim 64 ok, but I=256 ok -> null ptrs -> invalid arg
    assert lib.mb_encoder_forward(ctypes.byref(d), ctypes.byref(lp), ctypes.byref(pk), None, None, None, None,
                                  None, None) == 1
    bad = _lib.Dropout(1.5, 0, 0)  # p outside [0, 1)
    assert lib.mb_dropout_mask(ctypes.byref(bad), 0, 4, 8, 1, None) == 1
    ok = _lib.Dropout(0.1, 0, 0)
    assert lib.mb_dropout_mask(ctypes.byref(ok), 0, 4, 12, 1, None) == 2  # cols % 8 != 0
    # mb_mlm_loss: dy_top and g must be both given (training) or both NULL (forward-only evaluation)
    hd = _lib.dims(64, 2, 256, 128)
    hp, hg = _lib.HeadPtrs(), _lib.HeadPtrs()
    assert lib.mb_mlm_loss(ctypes.byref(hd), ctypes.byref(hp), 8, 4, 8, 8, 2, ctypes.c_float(1.0), 8, 8, None,
                           ctypes.byref(hg), 8, 1 << 20, None) == 1
    assert lib.mb_mlm_loss(ctypes.byref(hd), ctypes.byref(hp), 8, 4, 8, 8, 2, ctypes.c_float(1.0), 8, 8, 8, None, 8,
                           1 << 20, None) == 1
    assert lib.mb_status_string(4) == b"MB_ERR_MASK_LAYOUT"
    assert lib.mb_status_string(9) == b"MB_ERR_TOKEN_RANGE"


def test_arch_error_without_b200(lib):
    """Well-formed calls on a machine whose current device is not sm_100 (here: no device at all)
    return MB_ERR_ARCH and launch nothing (the library carries sm_100a SASS only)."""
    import torch
    if torch.cuda.is_available() and torch.cuda.get_device_capability() == (10, 0):
        pytest.skip("running on a B200")
    n0 = lib.mb_launch_count()
    assert lib.mb_layernorm_forward(8, 8, 8, 4, 64, ctypes.c_float(1e-5), 8, 8, None) == 7
    assert lib.mb_unpad_index(8, None, 0, 2, 4, 8, 8, 8, None, 0, None) == 7
    assert lib.mb_loss_normalize(8, None, ctypes.c_float(1.0), 8, None, None) == 7
    assert lib.mb_launch_count() == n0


def test_library_holds_no_device_allocation():
    """The header's contract: the library allocates nothing (every scratch is a caller workspace)."""
    csrc = os.path.join(ROOT, "paper_2312_17482_b200", "csrc")
    for f in os.listdir(csrc):
        txt = open(os.path.join(csrc, f)).read()
        for call in ("cudaMalloc", "cudaFree", "cudaHostAlloc", "malloc("):
            assert call not in txt, (f, call)


def test_workspace_queries(lib):
    from paper_2312_17482_b200 import _lib
    assert _lib.unpad_workspace_bytes(512) == 2 * 512 * 4 and _lib.unpad_workspace_bytes(0) == 0
    assert _lib.select_workspace_bytes(65536) == 64 * 4 and _lib.select_workspace_bytes(1) == 4
    d = _lib.dims(768, 12, 3072, 30528)
    sb = _lib.layer_saved_bytes(d, 65536)
    # QKV 3H + O H + S1 H + Y1 H + U 2I + Z I + S2 H (bf16) + LSE heads + 2x stats (fp32) per token
    per_tok = 2 * (3 * 768 + 768 + 768 + 768 + 2 * 3072 + 3072 + 768) + 4 * 12 + 16
    assert per_tok * 65536 <= sb <= per_tok * 65536 + 16 * 256
    assert _lib.layer_workspace_bytes(d, 65536, 128) > 0
    # fused softmax-CE: no fp32 logits; the bf16 dz [n, V] (input of the two backward GEMMs) is the
    # largest buffer, and the workspace stays below the unfused logits + dz (6 B per logit)
    assert 100 * 30528 * 2 <= _lib.mlm_workspace_bytes(d, 100) < 100 * 30528 * 6


def test_lr_schedule_matches_oracle():
    """mb_lr_schedule (F1, a host function: callable without a GPU) vs the pinned oracle schedule."""
    import oracle as O
    from paper_2312_17482_b200 import _lib
    pk = 5e-4
    for T in (1, 7, 100, 70000):
        for step in sorted({0, 1, T // 20, int(0.06 * T), int(0.06 * T) + 1, T // 2, T - 1, T}):
            assert _lib.lr_schedule(step, T, pk) == pytest.approx(O.lr_at(step, T, pk), rel=2e-6, abs=1e-12), (T, step)
        # past the end the library clamps to the final value (the oracle rejects the step)
        assert _lib.lr_schedule(T + 5, T, pk) == pytest.approx(O.lr_at(T, T, pk), rel=2e-6)
    assert _lib.lr_schedule(123, None, pk) == pytest.approx(pk, rel=1e-7)


def test_header_is_plain_c():
    """include/mosaicbert.h is a C header (extern "C" ABI): it compiles as C99 with -Wall -Werror."""
    import shutil
    import tempfile
    cc = shutil.which("gcc") or shutil.which("cc")
    if cc is None:
        pytest.skip("no C compiler")
    with tempfile.TemporaryDirectory() as d:
        src = os.path.join(d, "t.c")
        with open(src, "w") as f:
            f.write('#include "mosaicbert.h"\nint main(void) { return 0; }\n')
        r = subprocess.run([cc, "-std=c99", "-Wall", "-Werror", "-I", os.path.join(ROOT, "include"), "-c", src, "-o",
                            os.path.join(d, "t.o")], capture_output=True, text=True)
        assert r.returncode == 0, r.stderr
