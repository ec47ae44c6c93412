"""Max relative moment / Sigma error of windows = 2 against the whole-grid
solve for clip factors K (DGDIFF_WINK), per element type, on c3 sources."""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

CODE = r'''
import sys, json, numpy as np
sys.path.insert(0, "%s")
from paper_1907_06191_b200 import configs, dgdiff as dg
p, el, w = int(sys.argv[1]), int(sys.argv[2]), int(sys.argv[3])
m = configs.mask("c3"); src = configs.sources("c3")[:128]
dt = ({1: 1/32, 2: 1/128, 3: 1/256} if el == 0 else {1: 1/16, 2: 1/64})[p]
with dg.Solver(m, 1.0, 1.0, p, element=el, windows=w) as s:
    s.solve(src, dt, 300); S, mu = s.covariance(); mom = s.moments()
print(json.dumps(dict(mom=mom.tolist(), S=S.tolist())))
''' % ROOT


def run(p, el, w, k=None):
    env = dict(os.environ)
    if k is not None:
        env["DGDIFF_WINK"] = str(k)
        env["DGDIFF_TUNING_LIB"] = "1"   # knobs are read by the tuning build only
    out = subprocess.run([sys.executable, "-c", CODE, str(p), str(el), str(w)], capture_output=True, text=True, env=env)
    return json.loads(out.stdout.strip().splitlines()[-1])


import numpy as np
for p, el in ((1, 0), (2, 0), (3, 0), (1, 1), (2, 1)):
    ref = run(p, el, 0)
    M0 = np.array(ref["mom"])
    for k in (15, 20, 25, 30, 40, 50):
        r = run(p, el, 2, k)
        e = np.abs(np.array(r["mom"]) - M0).max() / np.abs(M0).max()
        print(json.dumps(dict(p=p, element=el, K=k, max_rel_mom_err=e)), flush=True)
