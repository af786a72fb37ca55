"""A/B timing of libh2 build variants selected by environment variables (one process per
variant so static choices re-read the environment).  Prints the mean phase times of K timed
builds after W warm-ups:  python tools/ab_phases.py WORKLOAD K W 'ENV=1 ENV2=0' 'ENV=0' ..."""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CHILD = r'''
import json, os, sys, time
sys.path.insert(0, os.environ["ROOT"])
import numpy as np, torch
import paper_2506_16759_b200 as g
from synth import WORKLOADS
w = WORKLOADS[sys.argv[1]]; K, W = int(sys.argv[2]), int(sys.argv[3])
X = w["points"](); T = g.Tree(X, w["leaf"], 0.7)
opts = dict(adaptive=True, d_init=32, d_blk=32, d_max=512)
for _ in range(W): g.build(T, (w["kernel"], w["param"]), w["tol"], **opts)
torch.cuda.synchronize()
st, ms = [], []
for _ in range(K):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(); H = g.build(T, (w["kernel"], w["param"]), w["tol"], **opts); e1.record(); e1.synchronize()
    ms.append(e0.elapsed_time(e1)); st.append(H.stats)
ph = {k: round(float(np.mean([s["t_phase_ms"][k] for s in st])), 2) for k in st[0]["t_phase_ms"]}
dep = {t: round(float(np.mean([s["t_depth_ms"][t] for s in st])), 2) for t in st[0]["t_depth_ms"]}
print(json.dumps({"ms": round(float(np.mean(ms)), 2), "samples": st[-1]["samples"], "phase_ms": ph,
                  "depth_ms": dep, "cpqr_variants": st[-1]["cpqr_variants"]}))
'''

if __name__ == "__main__":
    wl, K, W = sys.argv[1], sys.argv[2], sys.argv[3]
    for spec in sys.argv[4:]:
        env = dict(os.environ, ROOT=ROOT)
        for kv in spec.split():
            k, v = kv.split("=")
            env[k] = v
        out = subprocess.run([sys.executable, "-c", CHILD, wl, K, W], env=env, capture_output=True, text=True)
        line = out.stdout.strip().splitlines()[-1] if out.stdout.strip() else out.stderr[-800:]
        print(f"[{spec}] {line}", flush=True)
