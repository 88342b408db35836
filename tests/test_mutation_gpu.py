"""The race detector can fail (SPEC.md acceptance criterion 6).

liblpy_mutant.so is the product library compiled with -DLPY_MUTATE_STAGE_RACE
(paper_1405_7470_b200/_build.py): the FFMA consumers release a shared-memory
stage to the TMA producer BEFORE reading it, and the 3xTF32 split-transform
warps mark a stage ready for the MMA BEFORE writing its small parts.  Every
barrier still receives its arrivals once per phase, so nothing hangs (a first
3xTF32 mutant that skipped the MMA's wait instead let barrier phases overrun
and hung) -- the kernels just read stages that are being refilled or not yet
written.

The detector is the check of tests/test_parity_gpu.py::test_repeatable_every_element
(repeated runs bitwise equal, every element within the 1e-5 bound of a float64
reference), run in a child process per library: on the product library it must
pass, on the mutant it must fail, on both paths."""
import os
import subprocess
import sys
import textwrap

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

DETECTOR = textwrap.dedent("""
    import sys, torch
    sys.path.insert(0, {root!r})
    import paper_1405_7470_b200 as lpy
    lib = sys.argv[1]
    if lib != "product":
        lpy.library_path = lambda: lib
    path = sys.argv[2]
    M, N, K = (int(x) for x in sys.argv[3:6])
    g = torch.Generator(device="cuda")
    g.manual_seed(M + K)
    A = torch.rand(M, K, device="cuda", generator=g) * 2 - 1
    B = torch.rand(K, N, device="cuda", generator=g) * 2 - 1
    ref = A.double() @ B.double()
    D = A.abs().double() @ B.abs().double()
    first, worst, same = None, 0.0, True
    for _ in range(6):
        C = lpy.gemm(A, B, path=path)
        worst = max(worst, ((C.double() - ref).abs() / D).max().item())
        if first is None:
            first = C.clone()
        else:
            same = same and torch.equal(C, first)
    ok = worst <= 1e-5 and same
    print("DETECTOR", "PASS" if ok else "FAIL", f"max_err={{worst:.3e}} repeatable={{same}}")
""").format(root=ROOT)


def _run(lib, path, shape):
    r = subprocess.run([sys.executable, "-c", DETECTOR, lib, path, *map(str, shape)], capture_output=True,
                       text=True, timeout=120, cwd=ROOT)
    line = [x for x in r.stdout.splitlines() if x.startswith("DETECTOR")]
    assert line, (r.stdout[-2000:], r.stderr[-2000:])
    return line[0]


@pytest.mark.parametrize("path", ["ffma", "3xtf32"])
@pytest.mark.parametrize("shape", [(4096, 4096, 1024), (1024, 1024, 1024)])
def test_race_detector_passes_product_and_fails_mutant(path, shape):
    """(4096 x 4096 x 1024: full-width tiles; 1024^3: the FFMA cluster split and
    the 3xTF32 narrow tiles whose A_small goes through TMEM)"""
    import paper_1405_7470_b200._build as b
    assert os.path.exists(b.MUTANT_LIB), "liblpy_mutant.so not built (__graft_entry__.build())"
    good = _run("product", path, shape)
    assert "PASS" in good, good
    bad = _run(b.MUTANT_LIB, path, shape)
    assert "FAIL" in bad, f"the race detector did not catch the stage race on {path}: {bad}"
