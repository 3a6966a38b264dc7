"""End-time lag between consecutive bands of the long-pair kernel (FFD_LONG_TRACE=1),
grouped by the consumer band's warp index and by CTA: where the fill time goes."""
import os, re, subprocess, sys, json
import numpy as np
n = int(sys.argv[1]) if len(sys.argv) > 1 else 262144
env = dict(os.environ, FFD_LONG_TRACE="1")
r = subprocess.run([sys.executable, os.path.join(os.path.dirname(__file__), "one_long.py"), str(n)],
                   capture_output=True, text=True, env=env)
rows = [tuple(map(int, m.groups())) for m in re.finditer(r"ffdtrace band (\d+) cta (\d+) warp (\d+) start (\d+) end (\d+)", r.stdout)]
last = {}
for b, c, w, s, e in rows:
    last[b] = (s, e, c, w)
bands = sorted(last)
en = np.array([last[b][1] for b in bands], np.float64)
st = np.array([last[b][0] for b in bands], np.float64)
en -= st.min()
lag = np.diff(en) / 1e3  # us, lag of band i+1 behind band i
warp = np.array([last[b][3] for b in bands[1:]])
cta = np.array([last[b][2] for b in bands[1:]])
out = {"n": n, "env_cluster": os.environ.get("FFD_LONG_CLUSTER", "auto"), "bands": len(bands),
       "total_ms": en.max() / 1e6, "first_end_ms": en[0] / 1e6, "sum_lag_ms": float(lag.sum()) / 1e3,
       "lag_us_by_consumer_warp": {int(w): round(float(lag[warp == w].mean()), 2) for w in range(8)},
       "lag_us_p50": round(float(np.median(lag)), 2), "lag_us_p90": round(float(np.percentile(lag, 90)), 2),
       "lag_us_max": round(float(lag.max()), 2)}
# cumulative lag by CTA decile (is the fill uniform along the chain?)
dec = np.array_split(lag, 10)
out["lag_us_mean_by_decile"] = [round(float(d.mean()), 2) for d in dec]
print(json.dumps(out))
