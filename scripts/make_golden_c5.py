"""Write tests/golden/c5_expected.json: the CPU oracle's δ for BASELINE config 5.

Config 5 is one pair of n = m = 262,144 points (2-D fp32 Gaussian walks); its
full (n+1)×(m+1) table would need 550 GB, so the oracle's linear-memory form
(Alg. 5; pinned bit-exact to the table form in
tests/test_oracle_pins.py) is used, in fp64, once per norm (L1, L2, L∞).
Calls only oracle/ and workload/ (the seeded generator).  ~4 min per norm.

    python scripts/make_golden_c5.py
"""
import hashlib
import json
import os
import sys
import time
from concurrent.futures import ThreadPoolExecutor

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def one(norm):
    import oracle
    import workload
    p, q = workload.gen_long_pair(workload.CONFIGS[5])
    t0 = time.time()
    v = oracle.pair(p, q, norm, form="linear")
    return norm, v, time.time() - t0


def main():
    import workload
    p, q = workload.gen_long_pair(workload.CONFIGS[5])
    digest = hashlib.sha256(p.tobytes() + q.tobytes()).hexdigest()
    out = {"_about": "oracle (fp64, Alg. 5 linear form) δ_dF of BASELINE config 5's pair; written by "
                     "scripts/make_golden_c5.py (calls only oracle/ and workload/)",
           "config": workload.CONFIGS[5].name, "n": int(p.shape[0]), "m": int(q.shape[0]),
           "input_sha256": digest, "expected": {}, "seconds": {}}
    with ThreadPoolExecutor(3) as ex:  # ctypes releases the GIL
        for norm, v, dt in ex.map(one, ["l1", "l2", "linf"]):
            out["expected"][norm] = v
            out["seconds"][norm] = round(dt, 1)
    path = os.path.join(ROOT, "tests", "golden", "c5_expected.json")
    with open(path, "w") as f:
        json.dump(out, f, indent=2)
    print(json.dumps(out))


if __name__ == "__main__":
    main()
