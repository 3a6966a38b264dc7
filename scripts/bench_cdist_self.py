"""Self all-pairs matrix: ffd_cdist_self(A) vs ffd_cdist(A, A) on the
config-4 set A (20k curves, L = 128, 2-D fp32, L2).  Reports the time of both, the DP
cells actually evaluated by each, and checks the two matrices are identical."""
import json, os, sys
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2404_05708_b200 as ffd
import workload

cfg = workload.CONFIGS[4]
n = int(sys.argv[1]) if len(sys.argv) > 1 else cfg.nA
A = torch.from_numpy(workload.gen_set(cfg.scaled(nA=n), "A")).cuda()
out_full = torch.empty((n, n), dtype=torch.float32, device="cuda")
out_self = torch.empty((n, n), dtype=torch.float32, device="cuda")
res = {}
for name, fn in (("full", lambda: ffd.cdist(A, A, "l2", out=out_full)),
                 ("self", lambda: ffd.cdist_self(A, "l2", out=out_self))):
    fn(); torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(); fn(); e1.record(); torch.cuda.synchronize()
    res[name] = e0.elapsed_time(e1)
L = cfg.length
print(json.dumps({"n": n, "L": L, "full_ms": res["full"], "self_ms": res["self"],
                  "speedup": res["full"] / res["self"],
                  "full_cells_per_s": n * n * L * L / (res["full"] * 1e-3),
                  "self_evaluated_cells_per_s_approx": (n * (n + 1) / 2) * L * L / (res["self"] * 1e-3),
                  "identical": bool(torch.equal(out_full, out_self))}))
