"""GPU parity for the 3D Coulomb potential (Table 1's third row)
through the C-ABI (lpy_coulomb_f32 / lpy_coulomb_f32_host) against the float64
oracle on the same seeded particles.  Bar (reading C2):
|phi - phi_ref| <= 5e-6 * sum_j |q_j| / r_ij for every target; exact zeros where
the oracle is exactly zero; phi's neighbours never written."""
import numpy as np
import pytest
import torch

import oracle
import paper_1405_7470_b200 as lpy
import synth

pytestmark = pytest.mark.gpu

TOL = 5e-6
SENTINEL = np.float32(-31337.0)


def lay(p, ld):
    if p.shape[0] == 0:
        return np.zeros(0, np.float32)
    buf = np.full((p.shape[0], ld), np.nan, np.float32)
    buf[:, :3] = p
    return buf.reshape(-1)[: (p.shape[0] - 1) * ld + 3].copy()


def run_coulomb(tgt, src, q, ldt=3, lds=3, host=False):
    """(phi as np.float32, neighbours of phi untouched)."""
    nt, ns = tgt.shape[0], src.shape[0]
    tb, sb = lay(tgt, ldt), lay(src, lds)
    dev = "cpu" if host else "cuda"

    def put(a):
        x = torch.from_numpy(np.ascontiguousarray(a)) if a.size else torch.zeros(1)
        return x.pin_memory() if host else x.cuda()
    dt, ds, dq = put(tb), put(sb), put(q.astype(np.float32))
    out = torch.full((nt + 8,), float(SENTINEL), dtype=torch.float32, device=dev)
    if host:
        out = out.pin_memory()
    fn = lpy.lpy_coulomb_f32_host if host else lpy.lpy_coulomb_f32
    st = fn(nt, dt.data_ptr() if nt else 0, ldt, ns, ds.data_ptr() if ns else 0, lds,
            dq.data_ptr() if ns else 0, out.data_ptr() + 16 if nt else 0,
            None if host else torch.cuda.current_stream().cuda_stream)
    if st != 0:
        raise lpy.LpyError(st, "coulomb")
    torch.cuda.synchronize()
    o = out.cpu().numpy()
    return o[4:4 + nt], bool(np.all(o[:4] == SENTINEL) and np.all(o[4 + nt:] == SENTINEL))


def check(phi, tgt, src, q):
    ref, D = oracle.coulomb(tgt.shape[0], lay(tgt, 3), 3, src.shape[0], lay(src, 3), 3, q.astype(np.float32))
    assert np.all(np.isfinite(phi))
    zero = D == 0
    assert np.all(phi[zero] == 0)
    err = np.abs(phi.astype(np.float64) - ref)[~zero] / D[~zero]
    assert err.size == 0 or err.max() <= TOL, f"max normalised error {err.max():.3e}"
    return float(err.max()) if err.size else 0.0


def cloud(n, seed, charges="uniform"):
    pos, q = synth.particles(n, seed, charges)
    return pos.reshape(n, 3), q


@pytest.mark.parametrize("n", [1, 2, 3, 255, 256, 257, 1000, 1024, 1025, 4099])
def test_self_potential_sizes(n):
    """targets == sources (every target's own charge excluded): ragged tiles and
    target blocks, split and unsplit grids."""
    p, q = cloud(n, 1)
    phi, untouched = run_coulomb(p, p, q)
    check(phi, p, p, q)
    assert untouched


@pytest.mark.parametrize("nt,ns", [(5, 100000), (3000, 7), (1, 1), (777, 1), (2048, 300001 // 7)])
def test_separate_targets_and_sources(nt, ns):
    t, _ = cloud(nt, 2)
    s, q = cloud(ns, 3)
    phi, untouched = run_coulomb(t, s, q)
    check(phi, t, s, q)
    assert untouched


@pytest.mark.parametrize("charges", ["uniform", "uniform01", "int"])
def test_charge_distributions(charges):
    p, q = cloud(6000, 4, charges)
    phi, _ = run_coulomb(p, p, q)
    check(phi, p, p, q)


@pytest.mark.parametrize("ldt,lds", [(3, 4), (4, 3), (7, 5)])
def test_strided_points(ldt, lds):
    t, _ = cloud(1500, 5)
    s, q = cloud(2500, 6)
    phi, _ = run_coulomb(t, s, q, ldt, lds)
    ref, _ = run_coulomb(t, s, q)
    np.testing.assert_array_equal(phi, ref)      # layout changes where points live, not the sum
    check(phi, t, s, q)


def test_closed_forms_and_exclusion():
    src = np.array([[-1, -1, -1], [-1, -1, 1], [-1, 1, -1], [-1, 1, 1], [1, -1, -1], [1, -1, 1],
                    [1, 1, -1], [1, 1, 1]], np.float32)
    q = np.ones(8, np.float32)
    tgt = np.array([[0, 0, 0], [1, 1, 1]], np.float32)
    phi, _ = run_coulomb(tgt, src, q)
    np.testing.assert_allclose(phi, [8 / np.sqrt(3), 1.5 + 3 / (2 * np.sqrt(2)) + 1 / (2 * np.sqrt(3))],
                               rtol=2e-6)
    p, q = cloud(3000, 7)
    zero, _ = run_coulomb(p, p, np.zeros_like(q))
    assert np.all(zero == 0)
    empty, _ = run_coulomb(p[:10], p[:0], q[:0])
    assert np.all(empty == 0)
    # a target on a source sees the set without it (bitwise: the excluded term is an exact 0)
    k = 1234
    keep = np.arange(3000) != k
    on, _ = run_coulomb(p[k:k + 1], p, q)
    q_wo = q.copy()
    q_wo[k] = 0
    off, _ = run_coulomb(p[k:k + 1], p, q_wo)
    np.testing.assert_array_equal(on, off)
    check(on, p[k:k + 1], p[keep], q[keep])


def test_duplicate_positions_far_apart():
    """Two particles at the same position with distant indices (different
    source tiles, outside the masked diagonal tiles of a self-potential): each
    excludes the other -- the non-finite fallback path -- and the other targets
    are unaffected."""
    p, q = cloud(5000, 11)
    p[4321] = p[17]
    phi, _ = run_coulomb(p, p, q)
    check(phi, p, p, q)
    t = np.concatenate([p[17:18], p[:3]])       # separate target set, first target on two sources
    phi2, _ = run_coulomb(t, p, q)
    check(phi2, t, p, q)


def test_determinism_and_scaling():
    p, q = cloud(20000, 8)
    a, _ = run_coulomb(p, p, q)
    b, _ = run_coulomb(p, p, q)
    np.testing.assert_array_equal(a, b)
    s4, _ = run_coulomb(p * np.float32(4), p * np.float32(4), q)   # every fp32 step scales exactly...
    np.testing.assert_allclose(s4, a / 4, rtol=0, atol=4 * TOL * np.abs(a).max())  # ...except rsqrt's approx


def test_host_entry_and_torch_binding():
    p, q = cloud(5000, 9)
    phi_h, untouched = run_coulomb(p, p, q, host=True)
    check(phi_h, p, p, q)
    assert untouched
    dp, dq = torch.from_numpy(p).cuda(), torch.from_numpy(q).cuda()
    phi_t = lpy.coulomb(dp, dp, dq).cpu().numpy()
    np.testing.assert_array_equal(phi_t, phi_h)


@pytest.mark.slow
def test_bench_config_sampled():
    """The bench workload (N = 2^16 particles, self-potential, the launch
    configuration bench.py times): 2048 sampled targets against the oracle."""
    n = 1 << 16
    p, q = cloud(n, 0)
    phi, _ = run_coulomb(p, p, q)
    idx = np.random.default_rng(0).choice(n, 2048, replace=False)
    ref, D = oracle.coulomb(idx.size, lay(p[idx], 3), 3, n, lay(p, 3), 3, q)
    assert np.max(np.abs(phi[idx] - ref) / D) <= TOL
