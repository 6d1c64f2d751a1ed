import sys, os, subprocess, json
sys.path.insert(0, '.')
if len(sys.argv) > 1:
    import numpy as np, lpgen, torch
    import paper_2412_09734_b200 as mp
    lp, C = lpgen.g_grid(batch=1024, seed=2)
    dev = torch.device("cuda", 0)
    prob = mp.Problem.from_lp(lp).to(dev); Cd = torch.as_tensor(C, device=dev)
    out = {}
    for alg in ("ra", "r2"):
        bs = mp.BatchSolver(prob, Cd)
        bs.solve(algorithm=alg, iteration_limit=1024, eps_abs=0.0, eps_rel=0.0)
        ts = [bs.solve(algorithm=alg, iteration_limit=1024, eps_abs=0.0, eps_rel=0.0)[0]["solve_seconds"] for _ in range(5)]
        r = bs.solve(algorithm=alg)
        out[alg] = (round(min(ts) * 1e3, 4), round(r[0]["solve_seconds"] * 1e3, 4))
        bs.close()
    print(json.dumps(out))
else:
    for v in sys.argv[1:] or ["0", "1"]:
        pass
    for v in ("0", "2", "0", "2"):
        env = dict(os.environ, MPAX_TINY_VARIANT=v)
        r = subprocess.run([sys.executable, __file__, "x"], env=env, capture_output=True, text=True)
        print("variant", v, "ms (1024 attempts, full solve)", r.stdout.strip(), r.stderr[-300:])
