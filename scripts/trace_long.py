"""Band start/end times of the long-pair kernel (FFD_LONG_TRACE=1) for one pair."""
import os, re, subprocess, sys, json
import numpy as np
n = int(sys.argv[1]) if len(sys.argv) > 1 else 131072
env = dict(os.environ, FFD_LONG_TRACE="1")
r = subprocess.run([sys.executable, os.path.join(os.path.dirname(__file__), "one_long.py"), str(n)],
                   capture_output=True, text=True, env=env)
rows = [tuple(map(int, m.groups())) for m in re.finditer(r"ffdtrace band (\d+) cta (\d+) warp (\d+) start (\d+) end (\d+)", r.stdout)]
last = {}
for b, c, w, s, e in rows:   # keep the last call's trace (one_long runs 3 calls)
    last[b] = (s, e, c, w)
bands = sorted(last)
st = np.array([last[b][0] for b in bands], np.float64); en = np.array([last[b][1] for b in bands], np.float64)
t0 = st.min()
st -= t0; en -= t0
print(json.dumps({"n": n, "bands": len(bands), "total_ms": (en.max()) / 1e6,
                  "last_band_start_ms": st[-1] / 1e6, "first_band_end_ms": en[0] / 1e6,
                  "median_band_duration_ms": float(np.median(en - st)) / 1e6,
                  "start_lag_us_per_band_p50": float(np.median(np.diff(st))) / 1e3,
                  "start_lag_us_cta_boundary": float(np.mean([st[i + 1] - st[i] for i in range(len(bands) - 1) if (i + 1) % 8 == 0])) / 1e3 if len(bands) > 8 else None,
                  "start_lag_us_in_cta": float(np.mean([st[i + 1] - st[i] for i in range(len(bands) - 1) if (i + 1) % 8 != 0])) / 1e3,
                  "end_lag_us_per_band_p50": float(np.median(np.diff(en))) / 1e3}))
print("start(us) first 20:", [round(x / 1e3, 1) for x in st[:20]])
print("end(us) first 20:", [round(x / 1e3, 1) for x in en[:20]])
