"""tcgen05 kind::tf32 characterisation (liblpy_probe.so): descriptor
encodings for every operand orientation the GEMM uses, how fp32 operand bits
enter the tensor core (truncation vs rounding to tf32), and how the TMEM
accumulation rounds -- the facts DESIGN.md readings A9/A10 rest on.  Results
are also written to gpurun_out/tmem_numerics.json for DESIGN.md."""
import ctypes
import json
import os

import numpy as np
import pytest
import torch

import paper_1405_7470_b200 as lpy

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
RESULTS = {}


@pytest.fixture(scope="module")
def probe():
    lib = ctypes.CDLL(os.path.join(os.path.dirname(lpy.library_path()), "liblpy_probe.so"))
    lib.lpy_probe_umma_tf32.argtypes = [ctypes.c_void_p] * 3 + [ctypes.c_int] * 5 + [ctypes.c_void_p]
    lib.lpy_probe_umma_tf32.restype = ctypes.c_int
    lib.lpy_probe_umma_rate.argtypes = [ctypes.c_int] * 3 + [ctypes.c_void_p, ctypes.c_void_p]
    lib.lpy_probe_umma_rate.restype = ctypes.c_int
    yield lib
    os.makedirs(os.path.join(ROOT, "gpurun_out"), exist_ok=True)
    with open(os.path.join(ROOT, "gpurun_out", "tmem_numerics.json"), "w") as f:
        json.dump(RESULTS, f, indent=1)


def tile(probe, A, B, a_mn=0, b_mn=0, acc_first=0):
    """D = A B^T for A: 128 x Kp, B: N x Kp through one tcgen05 tile."""
    N, Kp = B.shape
    dA = torch.from_numpy(np.ascontiguousarray(A, np.float32)).cuda()
    dB = torch.from_numpy(np.ascontiguousarray(B, np.float32)).cuda()
    dD = torch.full((128, N), -7.0, device="cuda")
    rc = probe.lpy_probe_umma_tf32(dA.data_ptr(), dB.data_ptr(), dD.data_ptr(), N, Kp, a_mn, b_mn,
                                   acc_first, None)
    assert rc == 0
    torch.cuda.synchronize()
    return dD.cpu().numpy()


@pytest.mark.parametrize("a_mn", [0, 1, 2, 3])
@pytest.mark.parametrize("b_mn", [0, 1, 2, 3])
@pytest.mark.parametrize("N,Kp", [(64, 32), (256, 32), (128, 64), (224, 64)])
def test_descriptors_exact_on_tf32_values(probe, a_mn, b_mn, N, Kp):
    """Operand formats: 0 K-major SW128, 1 MN-major 128B_BASE32B (32-k panels),
    2 K-major SW64, 3 MN-major 128B_BASE32B (16-k panels)."""
    rng = np.random.default_rng(N + Kp)
    A = rng.integers(-8, 9, (128, Kp)).astype(np.float32) * np.float32(0.25)
    B = rng.integers(-8, 9, (N, Kp)).astype(np.float32)
    D = tile(probe, A, B, a_mn, b_mn)
    np.testing.assert_array_equal(D, A.astype(np.float64) @ B.astype(np.float64).T)


def one_dot(probe, a, b):
    """sum_k a[k] b[k] (k < len(a) <= 32) as computed by one or more MMAs."""
    A = np.zeros((128, 32), np.float32)
    B = np.zeros((16, 32), np.float32)
    A[0, :len(a)] = a
    B[0, :len(b)] = b
    return float(tile(probe, A, B)[0, 0])


def test_operand_conversion(probe):
    ulp10 = 2.0 ** -10
    x_trunc_vs_round = np.float32(1 + 2.0 ** -11 + 2.0 ** -20)   # RN -> 1+2^-10, trunc -> 1
    got = one_dot(probe, [x_trunc_vs_round], [1.0])
    RESULTS["operand_1+2^-11+2^-20"] = got
    assert got in (1.0, 1.0 + ulp10)
    tie = np.float32(1 + 2.0 ** -11)                              # RNA -> 1+2^-10; RNE/trunc -> 1
    RESULTS["operand_tie_1+2^-11"] = one_dot(probe, [tie], [1.0])
    RESULTS["operand_mode"] = "truncate" if got == 1.0 else "round"


def test_accumulation_rounding(probe):
    u = 2.0 ** -23
    # within one instruction (k < 8): 1 + 0.75 ulp
    RESULTS["in_mma_1+0.75ulp"] = (one_dot(probe, [1.0, 2.0 ** -12], [1.0, 1.5 * 2.0 ** -12]) - 1) / u
    RESULTS["in_mma_-1-0.75ulp"] = (one_dot(probe, [-1.0, 2.0 ** -12], [1.0, -1.5 * 2.0 ** -12]) + 1) / u
    # four quarter-ulp products in one instruction: exact sum 1 + 1 ulp
    RESULTS["in_mma_1+4x0.25ulp"] = (one_dot(probe, [1.0] + [2.0 ** -12] * 4,
                                             [1.0] + [2.0 ** -13] * 4) - 1) / u
    # across instructions (k = 0 in MMA 0, k = 8 in MMA 1): 1 + 0.75 ulp
    a = [1.0] + [0.0] * 7 + [2.0 ** -12]
    b = [1.0] + [0.0] * 7 + [1.5 * 2.0 ** -12]
    RESULTS["across_mma_1+0.75ulp"] = (one_dot(probe, a, b) - 1) / u
    a = [1.0] + [0.0] * 7 + [2.0 ** -12]
    b = [1.0] + [0.0] * 7 + [0.5 * 2.0 ** -12]
    RESULTS["across_mma_1+0.25ulp"] = (one_dot(probe, a, b) - 1) / u
    a = [-1.0] + [0.0] * 7 + [2.0 ** -12]
    b = [1.0] + [0.0] * 7 + [-1.5 * 2.0 ** -12]
    RESULTS["across_mma_-1-0.75ulp"] = (one_dot(probe, a, b) + 1) / u
    # 1 + (-0.25 ulp): RZ/RD give 1 - 0.5ulp(below 1), RN gives 1
    a = [1.0] + [0.0] * 7 + [2.0 ** -12]
    b = [1.0] + [0.0] * 7 + [-0.5 * 2.0 ** -12]
    RESULTS["across_mma_1-0.25ulp"] = (one_dot(probe, a, b) - 1) / u
    for k, v in RESULTS.items():
        print(k, v)


def test_uniform_accumulation_error(probe):
    """Error growth of long TMEM accumulation on [0,1) tf32-exact data:
    Kp=64 per tile -> 8 MMAs; measured against exact float64."""
    rng = np.random.default_rng(0)
    A = (rng.integers(0, 2 ** 10, (128, 64)) * 2.0 ** -10).astype(np.float32)
    B = (rng.integers(0, 2 ** 10, (256, 64)) * 2.0 ** -10).astype(np.float32)
    D = tile(probe, A, B)
    ref = A.astype(np.float64) @ B.astype(np.float64).T
    rel = (D - ref) / ref
    RESULTS["uniform_k64_mean_rel_err"] = float(rel.mean())
    RESULTS["uniform_k64_max_abs_rel_err"] = float(np.abs(rel).max())
    assert np.abs(rel).max() < 1e-5


def test_mma_rate(probe):
    cyc = torch.zeros(1, dtype=torch.int64, device="cuda")
    for n in (128, 160, 192, 224, 256):
        for ctas in (1, 148):
            probe.lpy_probe_umma_rate(n, 2000, ctas, cyc.data_ptr(), None)
            torch.cuda.synchronize()
            RESULTS[f"cycles_per_mma_M128_N{n}_K8_ctas{ctas}"] = cyc.item() / 2000
    print(RESULTS)


def test_ffma_rate(probe):
    """FP32 FMA pipe throughput (FFMA and packed FFMA2), for the FFMA roofline."""
    probe.lpy_probe_ffma_rate.argtypes = [ctypes.c_void_p] + [ctypes.c_int] * 4 + [ctypes.c_void_p]
    out = torch.zeros(1, device="cuda")
    sms = torch.cuda.get_device_properties(0).multi_processor_count
    for pair in (0, 1):
        iters, blocks, threads = 20000, sms * 4, 256
        probe.lpy_probe_ffma_rate(out.data_ptr(), 100, blocks, threads, pair, None)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        probe.lpy_probe_ffma_rate(out.data_ptr(), iters, blocks, threads, pair, None)
        e1.record()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1)
        flops = 2.0 * 16 * iters * blocks * threads
        RESULTS[f"ffma_tflops_pair{pair}"] = flops / ms / 1e9
    print(RESULTS)


def test_mma_rate_per_operand_format(probe):
    """Cycles per kind::tf32 MMA (N=256, K=8) for each smem operand format, single
    CTA (M=128) and CTA pair (M=256).  Full rate is 128 cycles."""
    probe.lpy_probe_umma_rate_fmt.argtypes = [ctypes.c_int] * 6 + [ctypes.c_void_p, ctypes.c_void_p]
    cyc = torch.zeros(1, dtype=torch.int64, device="cuda")
    iters = 4000
    for cg in (1, 2):
        for fa in range(4):
            for fb in range(4):
                for same in (False, True):
                    rc = probe.lpy_probe_umma_rate_fmt(256, fa, fb, -iters if same else iters, 148, cg,
                                                       cyc.data_ptr(), None)
                    torch.cuda.synchronize()
                    assert rc == 0
                    key = f"cycles_per_mma_cg{cg}_fa{fa}_fb{fb}" + ("_same" if same else "")
                    RESULTS[key] = cyc.item() / iters
    print({k: v for k, v in RESULTS.items() if k.startswith("cycles_per_mma_cg")})


def test_rsqrt_rate(probe):
    """MUFU.RSQ throughput (rsqrt.approx.ftz.f32), the Coulomb kernel's bound:
    per-SM results per clock at the measured SM clock."""
    probe.lpy_probe_rsqrt_rate.argtypes = [ctypes.c_void_p] + [ctypes.c_int] * 3 + [ctypes.c_void_p]
    out = torch.zeros(1, device="cuda")
    sms = torch.cuda.get_device_properties(0).multi_processor_count
    iters, blocks, threads = 4000, sms * 4, 256
    probe.lpy_probe_rsqrt_rate(out.data_ptr(), 100, blocks, threads, None)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    probe.lpy_probe_rsqrt_rate(out.data_ptr(), iters, blocks, threads, None)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1)
    per_s = 16.0 * iters * blocks * threads / (ms * 1e-3)
    RESULTS["rsqrt_per_s"] = per_s
    RESULTS["rsqrt_per_clk_per_sm_at_1965MHz"] = per_s / sms / 1.965e9
    print(RESULTS)
    assert per_s > 0


def test_rsqrt_accuracy(probe):
    """Max relative error of rsqrt.approx.ftz.f32 over every fp32 mantissa in
    [1, 4) (two binades cover all exponent parities), against float64: the
    per-term error in DESIGN.md reading C2's bound."""
    probe.lpy_probe_rsqrt_eval.argtypes = [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int, ctypes.c_void_p]
    bits = np.arange(0x3F800000, 0x40800000, dtype=np.uint32)
    x = bits.view(np.float32)
    dx = torch.from_numpy(x).cuda()
    dy = torch.empty_like(dx)
    assert probe.lpy_probe_rsqrt_eval(dx.data_ptr(), dy.data_ptr(), x.size, None) == 0
    torch.cuda.synchronize()
    y = dy.cpu().numpy().astype(np.float64)
    rel = np.abs(y * np.sqrt(x.astype(np.float64)) - 1.0)
    RESULTS["rsqrt_max_rel_err"] = float(rel.max())
    RESULTS["rsqrt_max_rel_err_log2"] = float(np.log2(rel.max()))
    print(RESULTS)
    assert rel.max() < 2.0 ** -21


def test_f32x2_rates(probe):
    """Per-SM lane-op throughput of packed fp32 (FFMA2 / FADD2 / FMUL2) and of
    scalar FADD / FFMA at the 1.965 GHz max clock: which FMA-pipe half the
    packed forms use (the Coulomb kernel's r^2 arithmetic)."""
    probe.lpy_probe_x2_rate.argtypes = [ctypes.c_int, ctypes.c_void_p] + [ctypes.c_int] * 3 + [ctypes.c_void_p]
    out = torch.zeros(1, device="cuda")
    sms = torch.cuda.get_device_properties(0).multi_processor_count
    iters, blocks, threads = 20000, sms * 4, 256
    for kind, name in enumerate(["ffma2", "fadd2", "fmul2", "fadd", "ffma"]):
        probe.lpy_probe_x2_rate(kind, out.data_ptr(), 100, blocks, threads, None)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        probe.lpy_probe_x2_rate(kind, out.data_ptr(), iters, blocks, threads, None)
        e1.record()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1)
        lane_ops = 16.0 * iters * blocks * threads
        RESULTS[f"{name}_lane_ops_per_clk_per_sm"] = lane_ops / (ms * 1e-3) / sms / 1.965e9
    print(RESULTS)
