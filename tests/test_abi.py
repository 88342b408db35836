"""CPU-side checks of the C-ABI boundary (include/lpy.h): the library loads,
exports every declared symbol, and validates arguments BEFORE any CUDA call
(so these run without a GPU; nothing here launches work)."""
import ctypes
import os
import re

import pytest

import paper_1405_7470_b200 as lpy

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "lpy.h")


@pytest.fixture(scope="module", autouse=True)
def built():
    import __graft_entry__
    __graft_entry__.build_library()


def declared_functions():
    src = open(HEADER).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(lpy_[a-z0-9_]+)\s*\(", src)))


def test_header_declares_the_boundary():
    assert declared_functions() == sorted([
        "lpy_gemm_f32", "lpy_gemm_f32_ex", "lpy_gemm_f32_host", "lpy_select_path",
        "lpy_status_string", "lpy_last_cuda_error", "lpy_version", "lpy_saxpy_f32",
        "lpy_saxpy_f32_host", "lpy_coulomb_f32", "lpy_coulomb_f32_host", "lpy_gemm_f32_gated",
        "lpy_kgate_signal"])


def test_library_exports_every_declared_symbol():
    lib = ctypes.CDLL(lpy.library_path())
    for name in declared_functions():
        assert hasattr(lib, name), name
        assert hasattr(lpy, name), f"binding lacks {name}"


def test_version_and_status_strings():
    assert lpy.lpy_version() == 5
    for code in range(10):
        s = lpy.lpy_status_string(code)
        assert s.startswith("LPY_")
    assert lpy.lpy_status_string(0) == "LPY_OK"
    assert "UNKNOWN" in lpy.lpy_status_string(99)
    assert lpy.lpy_last_cuda_error() == 0


def test_select_path_is_host_only():
    assert lpy.lpy_select_path(128, 128, 128, lpy.PATH_AUTO) == (0, lpy.PATH_FFMA)
    assert lpy.lpy_select_path(8192, 8192, 8192, lpy.PATH_FFMA) == (0, lpy.PATH_FFMA)
    assert lpy.lpy_select_path(8192, 8192, 8192, lpy.PATH_3XTF32) == (0, lpy.PATH_3XTF32)
    assert lpy.lpy_select_path(-1, 8, 8)[0] == 1
    assert lpy.lpy_select_path(8, 8, 8, 7)[0] == 1


FAKE = 1 << 40      # never dereferenced: validation fails first


def call(M=4, N=4, K=4, A=FAKE, lda=4, la=0, B=FAKE + (1 << 20), ldb=4, lb=0,
         C=FAKE + (2 << 20), ldc=4, lc=0, path=0, opts=None):
    return lpy.lpy_gemm_f32_ex(M, N, K, A, lda, la, B, ldb, lb, C, ldc, lc, None, path, opts)


@pytest.mark.parametrize("kw,code", [
    (dict(M=-1), 1), (dict(K=-3), 1), (dict(N=1 << 31), 1), (dict(K=(1 << 31) - 1023), 1),
    (dict(N=(1 << 31) - 1023, ldb=(1 << 31) - 1023, ldc=(1 << 31) - 1023), 1),
    # a footprint past 2^62 elements: (lines-1)*ld would overflow int64
    (dict(M=(1 << 31) - 1024, lda=(1 << 38) - 1, K=4), 1),
    (dict(la=2), 1), (dict(lc=-1), 1), (dict(path=3), 1),
    (dict(lda=3), 2), (dict(ldb=0), 2), (dict(ldc=3), 2), (dict(la=1, lda=3), 2),
    (dict(M=5, la=1, lda=4), 2), (dict(lda=1 << 40), 2),
    (dict(A=0), 3), (dict(B=0), 3), (dict(C=0), 3),
    (dict(A=FAKE + 2), 4), (dict(C=FAKE + (2 << 20) + 1), 4),
    (dict(C=FAKE + 8), 5), (dict(C=FAKE + (1 << 20) - 4), 5),
])
def test_validation_errors_precede_cuda(kw, code):
    assert call(**kw) == code


def test_bad_opts_rejected():
    o = lpy.GemmOpts()
    o.reserved[2] = 1
    assert call(opts=o) == 1
    o = lpy.GemmOpts()
    o.tile_n = 100
    assert call(opts=o) == 1
    o = lpy.GemmOpts()
    o.num_ctas = -2
    assert call(opts=o) == 1
    # promotion intervals beyond 16 k-blocks break the 1e-5 contract (lpy.h)
    o = lpy.GemmOpts()
    o.promote_kblocks = 17
    assert call(opts=o) == 1
    o.promote_kblocks = 16                 # accepted: fails later, in the device query
    import torch
    if not torch.cuda.is_available():
        assert call(opts=o) in (6, 8)


def test_plan_sms_field_replaces_a_reserved_word():
    import ctypes as ct
    assert ct.sizeof(lpy.GemmOpts) == 32          # layout unchanged since version 4
    assert lpy.GemmOpts.plan_sms.offset == 16
    o = lpy.GemmOpts()
    o.plan_sms = -1
    assert call(opts=o) == 1


def gated_call(gate, **kw):
    args = dict(M=4, N=4, K=64, A=FAKE, lda=64, la=0, B=FAKE + (1 << 20), ldb=4, lb=0,
                C=FAKE + (2 << 20), ldc=4, lc=0)
    args.update(kw)
    return lpy.lpy_gemm_f32_gated(args["M"], args["N"], args["K"], args["A"], args["lda"], args["la"],
                                  args["B"], args["ldb"], args["lb"], args["C"], args["ldc"], args["lc"],
                                  None, 0, None, gate)


def test_gated_validation_precedes_cuda():
    flags = FAKE + (3 << 20)
    assert gated_call(None) == 3                                        # the gate is mandatory
    assert gated_call(lpy.KGate(0, 32, 1, 0)) == 3                      # NULL flags
    assert gated_call(lpy.KGate(flags + 2, 32, 1, 0)) == 4              # misaligned flags
    assert gated_call(lpy.KGate(flags, 16, 1, 0)) == 1                  # chunk_k below 32
    assert gated_call(lpy.KGate(flags, 1 << 31, 1, 0)) == 1             # chunk_k beyond the dims bound
    assert gated_call(lpy.KGate(flags, 32, 1, 0), M=-1) == 1            # the operand checks still apply
    assert gated_call(lpy.KGate(flags, 32, 1, 0), C=FAKE + 8) == 5
    assert gated_call(lpy.KGate(flags, 32, 1, 0), M=0, A=0, C=0) == 0   # empty domain: no-op
    assert lpy.lpy_kgate_signal(0, 1, None) == 3
    assert lpy.lpy_kgate_signal(flags + 1, 1, None) == 4


def test_empty_domain_is_noop_without_cuda():
    # M == 0 or N == 0 returns before any CUDA call; NULL is fine then
    assert call(M=0, A=0, C=0) == 0
    assert call(N=0, B=0, C=0) == 0
    # column-major C with an empty extent
    assert call(M=0, A=0, C=0, lc=1) == 0


def test_null_allowed_for_zero_extent_operand():
    # K == 0: A and B have no footprint, NULL allowed; C must still be valid.
    # Without a GPU the call then fails in the device query, never before.
    st = call(K=0, A=0, B=0)
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present: covered by the gpu tests")
    assert st in (6, 8)


def test_binding_fails_loudly_without_library(tmp_path, monkeypatch):
    monkeypatch.setattr(lpy, "_lib", None)
    monkeypatch.setattr(lpy, "library_path", lambda: str(tmp_path / "missing.so"))
    with pytest.raises(RuntimeError, match="not built"):
        lpy.load_library()


def test_operand_layout_inference():
    import torch
    x = torch.empty(5, 7)
    assert lpy.operand_layout(x) == (lpy.ROW_MAJOR, 7)
    assert lpy.operand_layout(x.t()) == (lpy.COL_MAJOR, 7)
    y = torch.empty(5, 12)[:, :7]
    assert lpy.operand_layout(y) == (lpy.ROW_MAJOR, 12)
    assert lpy.operand_layout(torch.empty(6, 8)[::2, ::2]) is None


def saxpy_call(n=4, alpha=1.0, x=FAKE, incx=1, y=FAKE + (1 << 20), incy=1, host=False):
    fn = lpy.lpy_saxpy_f32_host if host else lpy.lpy_saxpy_f32
    return fn(n, alpha, x, incx, y, incy, None)


@pytest.mark.parametrize("host", [False, True])
@pytest.mark.parametrize("kw,code", [
    (dict(n=-1), 1), (dict(incx=0), 1), (dict(incy=-2), 1), (dict(n=1 << 40, incx=1 << 30), 1),
    (dict(x=0), 3), (dict(y=0), 3),
    (dict(x=FAKE + 2), 4), (dict(y=FAKE + (1 << 20) + 1), 4),
    (dict(y=FAKE + 8), 5), (dict(y=FAKE, incy=2), 5), (dict(x=FAKE + (1 << 20) - 4), 5),
    (dict(n=3, incx=4, y=FAKE + 4), 5),
])
def test_saxpy_validation_errors_precede_cuda(kw, code, host):
    assert saxpy_call(host=host, **kw) == code


@pytest.mark.parametrize("host", [False, True])
def test_saxpy_empty_is_a_noop(host):
    assert saxpy_call(n=0, x=0, y=0, host=host) == 0


def coulomb_call(nt=4, t=FAKE, ldt=3, ns=4, s=FAKE + (1 << 20), lds=3, q=FAKE + (2 << 20),
                 phi=FAKE + (3 << 20), host=False):
    fn = lpy.lpy_coulomb_f32_host if host else lpy.lpy_coulomb_f32
    return fn(nt, t, ldt, ns, s, lds, q, phi, None)


@pytest.mark.parametrize("host", [False, True])
@pytest.mark.parametrize("kw,code", [
    (dict(nt=-1), 1), (dict(ns=-2), 1), (dict(ldt=2), 2), (dict(lds=0), 2),
    (dict(t=0), 3), (dict(s=0), 3), (dict(q=0), 3), (dict(phi=0), 3),
    (dict(t=FAKE + 2), 4), (dict(q=FAKE + (2 << 20) + 1), 4), (dict(phi=FAKE + (3 << 20) + 3), 4),
    (dict(phi=FAKE + 4), 5), (dict(phi=FAKE + (1 << 20) + 40), 5), (dict(phi=FAKE + (2 << 20) - 4), 5),
])
def test_coulomb_validation_errors_precede_cuda(kw, code, host):
    assert coulomb_call(host=host, **kw) == code


@pytest.mark.parametrize("host", [False, True])
def test_coulomb_empty_targets_is_a_noop(host):
    assert coulomb_call(nt=0, t=0, phi=0, host=host) == 0


def test_coulomb_binding_checks_arguments_before_the_library():
    """out / charges / point arrays are checked in the binding (a short,
    strided or float64 `out` would otherwise be overrun or silently garbage)."""
    import torch
    P = torch.zeros(4, 3)
    q = torch.zeros(4)
    # a (1, 3) view whose column stride is not 1 (X.T[:1] of a (3, n) tensor)
    with pytest.raises(TypeError, match="unit column stride"):
        lpy.coulomb_host(torch.zeros(3, 5).T[:1], P, q, torch.zeros(1))
    with pytest.raises(TypeError, match="out"):
        lpy.coulomb_host(P, P, q, torch.zeros(3))                       # short out
    with pytest.raises(TypeError, match="out"):
        lpy.coulomb_host(P, P, q, torch.zeros(4, dtype=torch.float64))  # wrong dtype
    with pytest.raises(TypeError, match="out"):
        lpy.coulomb_host(P, P, q, torch.zeros(8)[::2])                  # strided
    with pytest.raises(TypeError, match="charges"):
        lpy.coulomb_host(P, P, torch.zeros(3), torch.zeros(4))          # short charges
    with pytest.raises(ValueError, match="cuda"):
        lpy.coulomb(P, P, q)                                            # host tensors to the device entry
    with pytest.raises(ValueError, match="overlap"):
        lpy.coulomb_host(torch.zeros(12).as_strided((4, 3), (2, 1)), P, q, torch.zeros(4))
