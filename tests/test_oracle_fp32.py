"""Pins of the fp32 build of the oracle (liboracle_f32.so, reading 39: the same C file
compiled with -DORA_FP32 -fsingle-precision-constant, MPAX's default precision).

Held to what the mathematics fixes, not to the fp64 build's digits: it is really a single-
precision program (every output is an IEEE single), it reaches the known optimum of the generated
LPs at the paper's 1e-4 tolerance (checked by the fp64 oracle's independent KKT evaluation), and
on an LP whose data and iterates are exact in both precisions it reproduces the fp64 trajectory."""
import numpy as np
import pytest

import lpgen
import oracle

CASES = [("C1", lpgen.g_rand(50, 100, 10, seed=1)), ("ragged", lpgen.g_rand(37, 61, 5, seed=7)),
         ("powerlaw", lpgen.g_powerlaw(300, 600, 12, seed=9))]


@pytest.mark.parametrize("alg", ["ra", "r2"])
def test_outputs_are_single_precision(alg):
    lp = CASES[0][1]
    r32 = oracle.solve(lp, alg, precision="fp32")
    r64 = oracle.solve(lp, alg)
    for v in ("x", "y", "lam"):
        a = r32[v]
        assert np.array_equal(a, a.astype(np.float32).astype(np.float64)), v   # every value a float32
    assert not np.array_equal(r32["x"], r64["x"])                                # and not the fp64 program
    for f in ("primal_objective", "rel_kkt", "omega", "eta"):
        assert r32[f] == float(np.float32(r32[f]))


@pytest.mark.parametrize("alg", ["ra", "r2"])
@pytest.mark.parametrize("name,lp", CASES)
def test_reaches_the_known_optimum(alg, name, lp):
    r = oracle.solve(lp, alg, precision="fp32")
    assert r["status"] == oracle.OPTIMAL and r["rel_kkt"] <= 1e-4
    # the fp64 oracle's independent KKT evaluation of the fp32 point: the termination test holds
    # up to the fp32 rounding of the point itself (a few ulps of single relative to the norms)
    k = oracle.kkt_original(lp, r["x"], r["y"])
    slack = 1.05
    assert k["pres"] <= slack * (1e-4 + 1e-4 * np.linalg.norm(lp.q))
    assert k["dres"] <= slack * (1e-4 + 1e-4 * np.linalg.norm(lp.c))
    assert abs(r["primal_objective"] - lp.obj_star) <= 1e-3 * (1 + abs(lp.obj_star))


def test_exact_data_gives_the_fp64_trajectory():
    """The SPEC example LP (tiny_spec): small integers, so the scaling, the iterates and the step
    sizes of the first attempts are exact or rounded identically in both precisions -- the fp32
    program takes the fp64 program's decisions and lands on the same optimum."""
    lp = lpgen.tiny_spec()
    for alg in ("ra", "r2"):
        r32 = oracle.solve(lp, alg, precision="fp32", log_capacity=4096)
        r64 = oracle.solve(lp, alg, log_capacity=4096)
        assert r32["status"] == r64["status"] == oracle.OPTIMAL
        assert abs(r32["primal_objective"] - r64["primal_objective"]) <= 1e-5 * (1 + abs(r64["primal_objective"]))
        n = min(len(r32.get("att_log", [])), len(r64["att_log"]))
        if n:
            assert np.array_equal(r32["att_log"][:min(n, 8), 1], r64["att_log"][:min(n, 8), 1])
