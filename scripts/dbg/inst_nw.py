import sys, os, subprocess, json
sys.path.insert(0, '.')
if len(sys.argv) > 1:
    import numpy as np, lpgen, torch
    import paper_2412_09734_b200 as mp
    out = {}
    for k in (12, 30):
        lp = lpgen.warcraft_lp(k); C = lpgen.warcraft_costs(k, 70, seed=k)
        dev = torch.device("cuda", 0)
        bs = mp.BatchSolver(mp.Problem.from_lp(lp).to(dev), torch.as_tensor(C, device=dev))
        for alg in ("ra",):
            bs.solve(algorithm=alg, iteration_limit=512, eps_abs=0.0, eps_rel=0.0)
            r = bs.solve(algorithm=alg, iteration_limit=512, eps_abs=0.0, eps_rel=0.0)
            t = r[0]["solve_seconds"]; a = r["attempts"].max()
            out[f"k{k}"] = round(1e6 * t / a, 2)
        bs.close()
    print(json.dumps(out))
else:
    for nw in ("4", "8", "16", "32"):
        env = dict(os.environ, MPAX_INST_NW=nw)
        r = subprocess.run([sys.executable, __file__, "x"], env=env, capture_output=True, text=True)
        print("NW", nw, "us/attempt", r.stdout.strip(), r.stderr[-300:])
