"""Mutation check of the oracle's pins (pins "chosen so that a
plausible mistake anywhere ... fails one of them").  Each case below edits ONE line of
oracle/mpax_oracle.c into a plausible slip (a swapped weight, a dropped term, a wrong
comparison, a wrong constant), builds the edited copy into a temporary library, and runs
the oracle pin suites against it (oracle.py loads MPAX_ORACLE_LIB when set).  The case
passes only if some pin FAILS.  The unmutated oracle passing the same suites is the rest
of the CPU suite.  CPU only; the cases run in parallel."""
import concurrent.futures as cf
import os
import subprocess
import sys
import tempfile

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SRC = os.path.join(ROOT, "oracle", "mpax_oracle.c")
PIN_SUITES = ["tests/test_oracle_readings.py", "tests/test_oracle_pins.py", "tests/test_oracle_solve.py",
              "tests/test_oracle_infeasibility.py", "tests/test_oracle_polish.py"]

# (name, [(exact source text, replacement)], contract step / reading it breaks)
MUTATIONS = [
    ("kkt_omega weights swapped", [("sqrt(omega * r.pres * r.pres + r.dres * r.dres * inv_omega",
                                    "sqrt(r.pres * r.pres * inv_omega + omega * r.dres * r.dres")], "step 5"),
    ("omega0 from the unscaled ||q||", [("nq = m ? norm2(S->q, m) : 0.0;", "nq = m ? norm2(S->q0, m) : 0.0;")],
     "c.3 #7"),
    ("omega0 inverted", [("*omega = nc / nq;", "*omega = nq / nc;")], "c.3 #7"),
    ("eta0 from the unscaled K", [("mx = dmax(mx, fabs(S->K.v[k]));", "mx = dmax(mx, fabs(S->K.v[k] / S->Dr[0]));")],
     "c.3 #5"),
    ("candidate tie goes to the average", [("return kkt_omega_avg < kkt_omega_cur ? 1 : 0;",
                                           "return kkt_omega_avg <= kkt_omega_cur ? 1 : 0;")], "c.3 #10"),
    ("r2 reference never reset", [("if (k_in == 0) { ref = rP; ref_set = 1; }",
                                   "if (!ref_set) { ref = rP; ref_set = 1; }"),
                                  ("      else ref_set = 0;\n", "      else {}\n")], "c.3 #12"),
    ("primal step uses eta * omega", [("double tau = eta * (1.0 / omega), sigma", "double tau = eta * omega, sigma")],
     "step 3"),
    ("dual step drops +K~x", [("(S->q[i] - 2.0 * Kxp[i] + Kx[i])", "(S->q[i] - 2.0 * Kxp[i])")], "step 3"),
    ("dual objective upper-bound sign", [("if (u[j] < ORA_INF) dobj -= u[j] * lm;",
                                          "if (u[j] < ORA_INF) dobj += u[j] * lm;")], "step 5"),
    ("Halpern drops the anchor", [("rho * z[i]) + b * z0[i];", "rho * z[i]);")], "step 4 (P:64)"),
    ("restart artificial 0.63", [("k_in >= 0.36 * (double)k", "k_in >= 0.63 * (double)k")], "c.3 #12"),
    ("restart sufficient 0.25", [("metric <= 0.2 * ref", "metric <= 0.25 * ref")], "c.3 #12"),
    ("scaled lower bound l*Dc", [("S->l[j] = p->l[j] / Dc[j];", "S->l[j] = p->l[j] * Dc[j];")], "step 1"),
    ("average weight eta/W_old", [("double theta = eta / W1;", "double theta = eta / (W > 0.0 ? W : W1);")],
     "c.3 #16"),
    ("dual projection misses a row", [("for (int64_t i = 0; i < m1; ++i) y[i] = dmax(y[i], 0.0);",
                                       "for (int64_t i = 0; i + 1 < m1; ++i) y[i] = dmax(y[i], 0.0);")], "step 3"),
    ("primal weight ratio inverted", [("sqrt(omega * (dy / dx))", "sqrt(omega * (dx / dy))")], "c.3 #9"),
    ("termination strict", [("return r->pres <= eps_abs", "return r->pres < eps_abs")], "c.3 #21"),
    ("line-search exponents swapped", [("(1.0 - pow(jp1, -0.3)) * eb, (1.0 + pow(jp1, -0.6)) * eta",
                                        "(1.0 - pow(jp1, -0.6)) * eb, (1.0 + pow(jp1, -0.3)) * eta")], "c.3 #4"),
    ("Pock-Chambolle uses max", [("if (use_sum) { rho[i] += a; gam[j] += a; }",
                                  "if (0) { rho[i] += a; gam[j] += a; }")], "c.3 #3"),
    (">= rows clipped as = rows in pres", [("if (i < m1) ri = dmax(ri, 0.0);", "if (i < 0) ri = dmax(ri, 0.0);")],
     "step 5"),
]


def _run(case, tmp):
    name, edits, _ = case
    src = open(SRC).read()
    for old, new in edits:
        assert src.count(old) == 1, f"{name}: mutation anchor not unique/found: {old!r}"
        src = src.replace(old, new)
    tag = "".join(ch if ch.isalnum() else "_" for ch in name)
    cfile, so = os.path.join(tmp, tag + ".c"), os.path.join(tmp, tag + ".so")
    open(cfile, "w").write(src)
    subprocess.check_call(["gcc", "-O2", "-std=c11", "-fopenmp", "-ffp-contract=off", "-fno-fast-math", "-fPIC",
                           "-shared", cfile, "-o", so, "-lm"])
    env = dict(os.environ, MPAX_ORACLE_LIB=so, OMP_NUM_THREADS="2")
    p = subprocess.run([sys.executable, "-m", "pytest", "-x", "-q", "-p", "no:cacheprovider", "-m", "not gpu",
                        "--timeout", "30", "--timeout-method", "thread", *PIN_SUITES],
                       cwd=ROOT, env=env, capture_output=True, text=True, timeout=900)
    return p.returncode, p.stdout[-600:]


def test_every_mutation_fails_a_pin():
    # a pin that hangs under a mutation (a solve that no longer converges) fails by
    # pytest-timeout's 30 s limit, which exits the run with status 1 like any failure
    with tempfile.TemporaryDirectory() as tmp:
        with cf.ThreadPoolExecutor(max_workers=max(2, min(8, os.cpu_count() or 2))) as ex:
            futs = {case[0]: ex.submit(_run, case, tmp) for case in MUTATIONS}
            survivors = []
            for name, f in futs.items():
                rc, tail = f.result()
                if rc == 0:
                    survivors.append(name)
                else:
                    assert rc == 1, f"{name}: pytest exited {rc} (not a test failure):\n{tail}"
    assert not survivors, f"mutations no pin catches: {survivors}"


@pytest.mark.parametrize("case", MUTATIONS, ids=[c[0] for c in MUTATIONS])
def test_mutation_anchor_present(case):
    """Each mutation edits text that exists exactly once (so the check above is real)."""
    src = open(SRC).read()
    for old, _ in case[1]:
        assert src.count(old) == 1, old
