#!/usr/bin/env python
"""Mutation check of the oracle's pins ("Oracle pins").

Each mutation below is a plausible slip in oracle/oracle.c -- a dropped term,
a wrong sign or index, a transposed operand, a wrong layout accessor, a
missing |.| or a scaled normaliser.  For each one the script copies tests/,
oracle/ and synth/ into a scratch directory, applies the mutation to the copy
of oracle.c, rebuilds it there and runs the CPU pin suites against it.  A
mutation must make at least one pin fail ("caught"); the script exits 1 if any
survives.  The product package is not involved.

    python scripts/oracle_mutations.py [--keep]      # log: profiles/r02_oracle_mutations.txt
"""
from __future__ import annotations

import os
import shutil
import subprocess
import sys
import tempfile

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
PIN_SUITES = ["tests/test_oracle.py", "tests/test_coulomb_oracle.py", "tests/test_saxpy_oracle.py"]

# (name, exact source text, replacement, occurrence index or None for all)
MUTATIONS = [
    # GEMM
    ("gemm: dropped first k term", "for (int64_t k = 0; k < K; ++k) {     /* k ascending */",
     "for (int64_t k = 1; k < K; ++k) {     /* k ascending */", None),
    ("gemm: B transposed (B(j,k))", "const double b = at(B, ldb, lb, k, j);",
     "const double b = at(B, ldb, lb, j % K, k % (N ? N : 1));", None),
    ("gemm: col-major accessor uses row-major",
     "layout == ORACLE_ROW_MAJOR ? X[r * ld + c] : X[r + c * ld]",
     "layout == ORACLE_ROW_MAJOR ? X[r * ld + c] : X[c + r * ld]", None),
    ("gemm: |a| in the product", "c[j] += a * b;                /* a*b exact in float64 */",
     "c[j] += fabs(a) * b;", None),
    ("gemm: subtract instead of add", "c[j] += a * b;                /* a*b exact in float64 */",
     "c[j] -= a * b;", None),
    ("gemm: D missing |a|", "if (d) d[j] += fabs(a) * fabs(b);", "if (d) d[j] += a * fabs(b);", None),
    ("gemm: D scaled by 2", "if (d) d[j] += fabs(a) * fabs(b);", "if (d) d[j] += 2.0 * fabs(a) * fabs(b);",
     None),
    ("gemm: nonzero initial value", "c[j] = 0.0;                       /* sum identity (S:583) */",
     "c[j] = 1e-3;", None),
    ("gemm elems: wrong row index", "const double a = at(A, lda, la, ii[e], k);",
     "const double a = at(A, lda, la, jj[e] % M, k);", None),
    ("gemm elems: D scaled", "d += fabs(a) * fabs(b);", "d += 0.5 * fabs(a) * fabs(b);", None),
    # saxpy
    ("saxpy: alpha dropped", "out[i] = (double)alpha * (double)x[i * incx] + (double)y[i * incy];",
     "out[i] = (double)x[i * incx] + (double)y[i * incy];", None),
    ("saxpy: ignores incx", "out[i] = (double)alpha * (double)x[i * incx] + (double)y[i * incy];",
     "out[i] = (double)alpha * (double)x[i] + (double)y[i * incy];", None),
    ("saxpy: fp32 rounding of the product",
     "out[i] = (double)alpha * (double)x[i * incx] + (double)y[i * incy];",
     "out[i] = (double)(float)(alpha * x[i * incx]) + (double)y[i * incy];", None),
    # Coulomb
    ("coulomb: D missing |q|", "dacc += fabs((double)q[j]) / r;", "dacc += (double)q[j] / r;", None),
    ("coulomb: D scaled", "dacc += fabs((double)q[j]) / r;", "dacc += fabs((double)q[j]) / (2.0 * r);", None),
    ("coulomb: D from r^2", "dacc += fabs((double)q[j]) / r;", "dacc += fabs((double)q[j]) / (r * r);", None),
    ("coulomb: 1/r^2", "acc += (double)q[j] / r;", "acc += (double)q[j] / (r * r);", None),
    ("coulomb: dropped z", "const double r = sqrt(dx * dx + dy * dy + dz * dz);",
     "const double r = sqrt(dx * dx + dy * dy);", None),
    ("coulomb: sign of a difference", "const double dy = y - (double)s[j * lds + 1];",
     "const double dy = y + (double)s[j * lds + 1];", None),
    ("coulomb: no coincident exclusion", "if (r == 0.0) continue;          /* coincident: excluded (reading C1) */",
     "", None),
    ("coulomb: source/target stride mixed", "const double dx = x - (double)s[j * lds];",
     "const double dx = x - (double)s[j * ldt];", None),
]


def run_one(name, old, new, scratch):
    for d in ("tests", "oracle", "synth"):
        dst = os.path.join(scratch, d)
        if os.path.exists(dst):
            shutil.rmtree(dst)
        shutil.copytree(os.path.join(ROOT, d), dst,
                        ignore=shutil.ignore_patterns("__pycache__", "*.so"))
    shutil.copy(os.path.join(ROOT, "pytest.ini"), scratch)
    src = os.path.join(scratch, "oracle", "oracle.c")
    text = open(src).read()
    if old not in text:
        return "MUTATION NOT APPLICABLE (source text not found)", None
    open(src, "w").write(text.replace(old, new))
    env = dict(os.environ, PYTHONDONTWRITEBYTECODE="1")
    r = subprocess.run([sys.executable, "-m", "pytest", "-q", "-x", "-p", "no:cacheprovider", "-m", "not gpu",
                        *PIN_SUITES], cwd=scratch, env=env, capture_output=True, text=True, timeout=900)
    tail = [ln for ln in r.stdout.splitlines() if ln.strip()][-1:] or ["(no output)"]
    failed = [ln.split(" - ")[0] for ln in r.stdout.splitlines() if ln.startswith("FAILED")]
    return ("caught" if r.returncode != 0 else "SURVIVED"), (failed[0] if failed else tail[0])


def main():
    keep = "--keep" in sys.argv
    scratch = tempfile.mkdtemp(prefix="oracle_mut_")
    survived = 0
    lines = []
    try:
        base, _ = run_one("baseline", "", "", scratch)
        lines.append(f"unmutated oracle: {'pins pass' if base == 'SURVIVED' else 'PINS FAIL'}")
        for name, old, new, _ in MUTATIONS:
            verdict, detail = run_one(name, old, new, scratch)
            survived += verdict != "caught"
            lines.append(f"{verdict:8s}  {name:45s}  {detail or ''}")
            print(lines[-1], flush=True)
    finally:
        if not keep:
            shutil.rmtree(scratch, ignore_errors=True)
    lines.append(f"{len(MUTATIONS) - survived}/{len(MUTATIONS)} mutations caught")
    print(lines[-1])
    out = os.path.join(ROOT, "profiles", "r02_oracle_mutations.txt")
    with open(out, "w") as f:
        f.write("# scripts/oracle_mutations.py: each mutation of oracle/oracle.c must fail a pin in\n")
        f.write(f"# {', '.join(PIN_SUITES)} (run with -x: the first failing test is named)\n")
        f.write("\n".join(lines) + "\n")
    sys.exit(1 if survived else 0)


if __name__ == "__main__":
    main()
