"""GPU parity for saxpy (y := alpha*x + y, Table 1's saxpy row)
through the C-ABI (lpy_saxpy_f32 / lpy_saxpy_f32_host) against the float64
oracle on the same seeded inputs.  Bar (reading S1): every element is
the round-to-nearest fp32 of the exact alpha*x_i + y_i (at most half an fp32
ulp from the oracle's value), exact on integer inputs; elements outside the
strided vector (the gaps, and a guard zone after the end) are never written."""
import numpy as np
import pytest
import torch

import oracle
import paper_1405_7470_b200 as lpy
import synth

pytestmark = pytest.mark.gpu

GUARD = 64
SENTINEL = np.float32(-31337.0)


def run_saxpy(n, alpha, x, y, incx=1, incy=1, offx=0, offy=0, host=False, same=False):
    """saxpy through the C ABI on strided device (or host) buffers placed
    `off` floats after a 16-byte boundary; returns (y logical, gaps intact)."""
    xb = synth.strided(x, incx)
    yb = synth.strided(y, incy, pad_value=SENTINEL)
    dev = "cpu" if host else "cuda"
    ty = torch.full((offy + yb.size + GUARD,), float(SENTINEL), dtype=torch.float32, device=dev)
    if host:
        ty = ty.pin_memory()
    ty[offy:offy + yb.size].copy_(torch.from_numpy(yb))
    if same:
        tx, px = ty, ty.data_ptr() + 4 * offy
    else:
        tx = torch.zeros(offx + xb.size + GUARD, dtype=torch.float32, device=dev)
        if host:
            tx = tx.pin_memory()
        tx[offx:offx + xb.size].copy_(torch.from_numpy(xb))
        px = tx.data_ptr() + 4 * offx
    fn = lpy.lpy_saxpy_f32_host if host else lpy.lpy_saxpy_f32
    stream = None if host else torch.cuda.current_stream().cuda_stream
    st = fn(n, alpha, px if n else 0, incx, ty.data_ptr() + 4 * offy if n else 0, incy, stream)
    if st != 0:
        raise lpy.LpyError(st, "saxpy")
    torch.cuda.synchronize()
    out = ty.cpu().numpy()
    got = out[offy:offy + yb.size][::incy].copy() if n else np.zeros(0, np.float32)
    mask = np.ones(out.size, dtype=bool)
    mask[offy + np.arange(n) * incy] = False
    untouched = bool(np.all(out[mask] == SENTINEL))
    return got, untouched


def check(got, n, alpha, x, y, incx=1, incy=1):
    ref = oracle.saxpy(n, alpha, synth.strided(x, incx), incx, synth.strided(y, incy), incy)
    err = oracle.saxpy_error_ulps(got, ref)
    assert err <= 1.0, f"max error {err:.3f} half-ulps"
    return ref


@pytest.mark.parametrize("n", [0, 1, 2, 3, 4, 5, 7, 8, 63, 64, 65, 1023, 4097, 100003, (1 << 20) + 3])
def test_sizes(n):
    x = synth.vector(n, 1, synth.VECTOR_X)
    y = synth.vector(n, 1, synth.VECTOR_Y)
    got, untouched = run_saxpy(n, 1.75, x, y)
    check(got, n, 1.75, x, y)
    assert untouched


@pytest.mark.parametrize("offx,offy", [(0, 0), (1, 0), (0, 1), (2, 3), (3, 3), (1, 1), (2, 1)])
def test_alignments(offx, offy):
    """Head/tail around y's 16-byte boundaries; x aligned with y (vector
    loads) and not (scalar loads)."""
    n = 10007
    x = synth.vector(n, 2, synth.VECTOR_X)
    y = synth.vector(n, 2, synth.VECTOR_Y)
    got, untouched = run_saxpy(n, -0.375, x, y, offx=offx, offy=offy)
    check(got, n, -0.375, x, y)
    assert untouched


@pytest.mark.parametrize("incx,incy", [(2, 1), (1, 3), (7, 5), (4, 4)])
def test_increments(incx, incy):
    n = 5001
    x = synth.vector(n, 3, synth.VECTOR_X)
    y = synth.vector(n, 3, synth.VECTOR_Y)
    got, untouched = run_saxpy(n, 2.5, x, y, incx=incx, incy=incy)
    check(got, n, 2.5, x, y, incx, incy)
    assert untouched


@pytest.mark.parametrize("dist", synth.DISTS)
def test_distributions(dist):
    n = 1 << 16
    x = synth.vector(n, 4, synth.VECTOR_X, dist)
    y = synth.vector(n, 4, synth.VECTOR_Y, dist)
    for alpha in (float(np.float32(1 / 3)), -1e3, 2.0 ** -10):
        got, _ = run_saxpy(n, alpha, x, y)
        ref = check(got, n, alpha, x, y)
        if dist == "int" and alpha == 2.0 ** -10:
            assert np.array_equal(got.astype(np.float64), ref)   # exact in fp32


def test_closed_forms():
    n = 30001
    x = synth.vector(n, 5, synth.VECTOR_X)
    y = synth.vector(n, 5, synth.VECTOR_Y)
    got, _ = run_saxpy(n, 0.0, x, y)
    assert np.array_equal(got, y)                                # alpha = 0
    got, _ = run_saxpy(n, 1.0, x, np.zeros(n, np.float32))
    assert np.array_equal(got, x)                                # y = 0
    got, _ = run_saxpy(n, -1.0, x, x)
    assert np.array_equal(got, np.zeros(n, np.float32))          # x - x
    got, _ = run_saxpy(n, 2.0, x, x, same=True)                  # x == y: y := 3y
    check(got, n, 2.0, x, x)


def test_same_vector_strided():
    n = 2000
    y = synth.vector(n, 6, synth.VECTOR_Y)
    got, untouched = run_saxpy(n, -0.5, y, y, incx=3, incy=3, same=True)
    check(got, n, -0.5, y, y, 3, 3)
    assert untouched


@pytest.mark.parametrize("n,incx,incy,offx,offy", [(0, 1, 1, 0, 0), (5, 1, 1, 1, 2), (1 << 20, 1, 1, 0, 0),
                                                   ((1 << 21) + 5, 1, 1, 3, 1), (3001, 2, 3, 0, 0)])
def test_host_entry(n, incx, incy, offx, offy):
    x = synth.vector(n, 7, synth.VECTOR_X)
    y = synth.vector(n, 7, synth.VECTOR_Y)
    got, untouched = run_saxpy(n, 1.25, x, y, incx, incy, offx, offy, host=True)
    check(got, n, 1.25, x, y, incx, incy)
    assert untouched


def test_torch_binding_and_determinism():
    n = 1 << 20
    x = torch.from_numpy(synth.vector(n, 8, synth.VECTOR_X)).cuda()
    y0 = torch.from_numpy(synth.vector(n, 8, synth.VECTOR_Y)).cuda()
    outs = []
    for _ in range(3):
        y = y0.clone()
        lpy.saxpy(0.625, x, y)
        outs.append(y.cpu().numpy())
    assert all(np.array_equal(outs[0], o) for o in outs[1:])
    check(outs[0], n, 0.625, x.cpu().numpy(), y0.cpu().numpy())
    ys = y0.clone()
    lpy.saxpy(0.625, x[::2], ys[::2])                            # strided views
    assert np.array_equal(ys[::2].cpu().numpy(), outs[0][::2])
    assert np.array_equal(ys[1::2].cpu().numpy(), y0[1::2].cpu().numpy())


@pytest.mark.slow
def test_full_size_bench_config_sampled():
    """The bench workload (n = 2^28, the launch configuration bench.py times):
    every element against the oracle."""
    n = 1 << 28
    x = synth.vector(n, 0, synth.VECTOR_X)
    y = synth.vector(n, 0, synth.VECTOR_Y)
    got, untouched = run_saxpy(n, 1.5, x, y)
    check(got, n, 1.5, x, y)
    assert untouched
