"""CPU-side checks of the product library: it builds for sm_100a, loads without
a GPU, exports every entry point include/lp.h declares, and contains no
oracle code.  No compute calls (those need a GPU)."""
import os
import re
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _declared():
    hdr = open(os.path.join(ROOT, "include", "lp.h")).read()
    hdr = re.sub(r"/\*.*?\*/", "", hdr, flags=re.S)
    return sorted(set(re.findall(r"\b(lp_[a-z_]+)\s*\(", hdr)))


def test_build_and_exports():
    from paper_2412_09734_b200 import _build
    lib = _build.build()
    out = subprocess.run(["nm", "-D", "--defined-only", lib], capture_output=True, text=True, check=True).stdout
    syms = set(re.findall(r"\bT (\w+)", out))
    declared = _declared()
    assert len(declared) >= 15
    missing = [s for s in declared if s not in syms]
    assert not missing, missing
    assert not [s for s in syms if s.startswith("ora_")]          # no oracle code in the product
    import paper_2412_09734_b200 as mp
    L = mp.lib()
    for s in declared:
        assert hasattr(L, s)
    assert sorted(mp.EXPORTED_SYMBOLS) == declared


def test_sm100a_cubin():
    from paper_2412_09734_b200 import _build
    lib = _build.build()
    out = subprocess.run(["cuobjdump", "--list-elf", lib], capture_output=True, text=True).stdout
    assert "sm_100a" in out


def test_default_options_and_errors_without_gpu():
    import paper_2412_09734_b200 as mp
    o = mp.default_options()
    assert (o.eps_abs, o.eps_rel, o.eps_primal_infeasible, o.eps_dual_infeasible, o.eps_feas_polish) == \
        (1e-4, 1e-4, 1e-8, 1e-8, 1e-6)                                      # Appendix
    assert o.iteration_limit == 2**63 - 1 and o.check_frequency == 64 and o.display_frequency == 10
    assert o.algorithm == mp.R2HPDHG and o.path == mp.PATH_AUTO
    L = mp.lib()
    assert L.lp_error_string(-4) == b"crossed bounds"
    # argument errors are reported before any device work
    with pytest.raises(mp.LpError) as e:
        mp.Solver(mp.Problem(0, 0, 0, [0], [], [], [], [], [], []))
    assert e.value.code == -2


def test_no_oracle_import_in_product():
    pkg = os.path.join(ROOT, "paper_2412_09734_b200")
    for dirpath, _, files in os.walk(pkg):
        for f in files:
            if f.endswith((".py", ".cu", ".cuh", ".h", ".cpp")):
                src = open(os.path.join(dirpath, f)).read()
                assert "oracle" not in re.sub(r"#.*|//.*", "", src).replace("oracle/", ""), f
