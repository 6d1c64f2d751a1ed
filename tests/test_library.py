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


def test_abi_struct_layouts(tmp_path):
    """The binding's ctypes structs match include/lp.h byte for byte (sizes and every field
    offset, from a C program compiled against the header)."""
    import ctypes as C

    import paper_2412_09734_b200 as mp
    from paper_2412_09734_b200 import lp as mlp
    structs = {"lp_options": mlp.Options, "lp_result": mlp.Result, "lp_problem_desc": mlp.ProblemDesc}
    lines = ["#include <stdio.h>", "#include <stddef.h>", '#include "lp.h"', "int main(void) {"]
    for cname, py in structs.items():
        lines.append(f'  printf("{cname} %zu\\n", sizeof({cname}));')
        for f, _ in py._fields_:
            lines.append(f'  printf("{cname}.{f} %zu\\n", offsetof({cname}, {f}));')
    lines += ["  return 0;", "}"]
    src = tmp_path / "abi.c"
    src.write_text("\n".join(lines))
    exe = tmp_path / "abi"
    subprocess.run(["gcc", "-std=c11", "-I", os.path.join(ROOT, "include"), str(src), "-o", str(exe)], check=True)
    got = dict(line.split() for line in subprocess.run([str(exe)], capture_output=True, text=True,
                                                        check=True).stdout.splitlines())
    for cname, py in structs.items():
        assert int(got[cname]) == C.sizeof(py), cname
        for f, _ in py._fields_:
            assert int(got[f"{cname}.{f}"]) == getattr(py, f).offset, (cname, f)
    o = mp.default_options()
    assert o.precision == mp.FP64 and o.reflection == 1.0 and o.step_rule == mp.STEP_ADAPTIVE
    assert mp.default_options(precision="fp32").precision == mp.FP32
