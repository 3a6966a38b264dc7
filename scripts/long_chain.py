"""Per-step time of the long-pair chain against its length and link types:
one pair (n, m) with n = G·8 bands·32·7 rows (R = 7 for every G), run on G CTAs
(FFD_LONG_CTAS), with and without cluster DSMEM links (FFD_LONG_CLUSTER=1).
ns/step = kernel time / (m/2 two-column steps + bands × 47 fill steps)."""
import json, os, sys, subprocess

if len(sys.argv) > 1 and sys.argv[1] == "child":
    import numpy as np, torch
    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    import paper_2404_05708_b200 as ffd
    G, m = int(sys.argv[2]), int(sys.argv[3])
    n = G * 8 * 32 * 7
    rng = np.random.default_rng(1)
    p = torch.from_numpy(np.cumsum(rng.normal(size=(n, 2)), 0).astype(np.float32)).cuda()
    q = torch.from_numpy(np.cumsum(rng.normal(size=(m, 2)), 0).astype(np.float32)).cuda()
    off = torch.tensor([0, 0], dtype=torch.int64, device="cuda")
    lens = torch.tensor([n, m], dtype=torch.int32, device="cuda")
    for _ in range(2):
        ffd.batch(p, q, off, lens, norm="l2")
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    reps = 3
    for _ in range(reps):
        ffd.batch(p, q, off, lens, norm="l2")
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / reps
    bands = G * 8
    steps = m / 2 + bands * 47
    print(json.dumps({"G": G, "n": n, "m": m, "cluster": os.environ.get("FFD_LONG_CLUSTER", "auto"),
                      "ms": round(ms, 3), "ns_per_step": round(ms * 1e6 / steps, 1),
                      "gcells": round(n * m / ms / 1e6, 1)}), flush=True)
    sys.exit(0)

m = 131072
for G in (1, 2, 4, 8, 16, 32, 64, 147):
    for cl in ("auto", "1"):
        env = dict(os.environ, FFD_LONG_CTAS=str(G))
        if cl == "1":
            env["FFD_LONG_CLUSTER"] = "1"
        subprocess.run([sys.executable, __file__, "child", str(G), str(m)], env=env, timeout=300)
