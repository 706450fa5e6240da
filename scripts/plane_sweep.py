"""KP (plane-fused y.z.y) vs the K2/K3/K4 pencil path on thin-film grids: ms/step
of the graph-replayed Euler step (CUDA events, 50 steps after 10 warm-up), each
configuration in a fresh process so GRACE_PLANE is read at context creation.

    python scripts/plane_sweep.py [--out gpurun_out/plane_sweep.json]
"""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
GRIDS = [(512, 512, 8), (256, 256, 8), (1024, 512, 8), (512, 512, 4), (1024, 1024, 4), (1024, 1024, 2),
         (256, 256, 4), (2048, 1024, 2), (512, 512, 2)]


def one(n):
    sys.path.insert(0, ROOT)
    import torch

    import paper_1411_2565_b200 as pb
    from workloads import GAMMA0, random_m
    g = pb.Grace(n, (5e-9, 5e-9, 3e-9), 8e5, 1.3e-11, 0.0, 0.5, GAMMA0)
    s = torch.cuda.Stream()
    pb.grace_set_stream(g.h, s.cuda_stream)
    g.set_m(random_m(n, 8e5))
    g.step(10, 1e-14)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    e0.record(s)
    g.step(50, 1e-14)
    e1.record(s)
    torch.cuda.synchronize()
    k = g.geometry["kernels"]
    g.close()
    return e0.elapsed_time(e1) / 50, k


if __name__ == "__main__":
    if len(sys.argv) > 1 and sys.argv[1] == "--one":
        n = tuple(int(v) for v in sys.argv[2].split("x"))
        ms, k = one(n)
        print(json.dumps({"ms": ms, "kernels": k}))
        sys.exit(0)
    out = sys.argv[sys.argv.index("--out") + 1] if "--out" in sys.argv else None
    res = []
    for n in GRIDS:
        row = {"grid": list(n)}
        for tag, env in (("plane", {"GRACE_PLANE": "1"}), ("pencil", {})):
            r = subprocess.run([sys.executable, __file__, "--one", "x".join(map(str, n))], env=dict(os.environ, **env),
                               capture_output=True, text=True, timeout=300)
            try:
                d = json.loads(r.stdout.strip().splitlines()[-1])
                row[tag] = d["ms"]
                row[tag + "_kernels"] = d["kernels"]
            except Exception:
                row[tag] = None
                row[tag + "_err"] = r.stderr[-300:]
        res.append(row)
        print(json.dumps(row), flush=True)
    if out:
        json.dump(res, open(out, "w"), indent=1)
