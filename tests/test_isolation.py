"""The oracle and the CUDA path share nothing, and the product has no fallback
(task rules):
  * nothing under paper_1405_7470_b200/ (Python or CUDA) names, imports, links
    or includes oracle/; importing the product package does not load it;
  * oracle/ never includes or imports the product (its C source includes only
    libc headers);
  * synth/ (the one module both sides use) holds no arithmetic of the methods;
  * a missing liblpy.so is an error, not a silent CPU path.
CPU only."""
import glob
import os
import re
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
PKG = os.path.join(ROOT, "paper_1405_7470_b200")


def product_sources():
    pats = ["*.py", "csrc/*.cu", "csrc/*.cuh", "csrc/*.h"]
    files = [f for p in pats for f in glob.glob(os.path.join(PKG, p))]
    return files + glob.glob(os.path.join(ROOT, "include", "*.h"))


def code_only(path):
    """Source text without comments / docstrings (prose may name the oracle)."""
    src = open(path).read()
    if path.endswith(".py"):
        src = re.sub(r'("""|\'\'\').*?\1', "", src, flags=re.S)
        return "\n".join(line.split("#", 1)[0] for line in src.splitlines())
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return "\n".join(line.split("//", 1)[0] for line in src.splitlines())


def test_product_never_references_the_oracle():
    files = product_sources()
    assert len(files) >= 10
    for f in files:
        src = code_only(f)
        assert not re.search(r"\boracle\b", src), f"{f} refers to the oracle"
        assert "lpy_oracle" not in src, f


def test_importing_the_product_does_not_load_the_oracle():
    code = ("import sys; sys.path.insert(0, %r); import paper_1405_7470_b200, paper_1405_7470_b200.dist; "
            "print('oracle' in sys.modules, any(m.startswith('oracle') for m in sys.modules))" % ROOT)
    out = subprocess.run([sys.executable, "-c", code], capture_output=True, text=True, check=True).stdout
    assert out.strip() == "False False"


def test_oracle_includes_only_libc():
    src = open(os.path.join(ROOT, "oracle", "oracle.c")).read()
    includes = re.findall(r'#include\s*[<"]([^>"]+)[>"]', src)
    assert set(includes) <= {"stdint.h", "stddef.h", "math.h", "omp.h"}, includes
    py = code_only(os.path.join(ROOT, "oracle", "__init__.py"))
    imports = re.findall(r"^\s*(?:import|from)\s+([\w.]+)", py, flags=re.M)
    assert not any(m.split(".")[0] in ("paper_1405_7470_b200", "synth") for m in imports), imports


def test_synth_holds_no_method_arithmetic():
    src = open(os.path.join(ROOT, "synth", "__init__.py")).read()
    code = re.sub(r'""".*?"""', "", src, flags=re.S)
    for forbidden in ("@", "matmul", "dot(", "einsum", "rsqrt", "sqrt(", "fma"):
        assert forbidden not in code, forbidden


def test_missing_library_fails_loudly(monkeypatch):
    import paper_1405_7470_b200 as lpy
    monkeypatch.setattr(lpy, "_lib", None)
    monkeypatch.setattr(lpy, "library_path", lambda: os.path.join(PKG, "no_such_liblpy.so"))
    with pytest.raises(RuntimeError, match="not built"):
        lpy.load_library()
    with pytest.raises(RuntimeError):
        lpy.lpy_version()
