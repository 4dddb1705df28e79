"""Errors of each LU schedule against numpy's inverse (tests/_lu_schedules.py under env variants)."""
import os, subprocess, sys, numpy as np
here = os.path.dirname(os.path.abspath(__file__)); root = os.path.dirname(here)
for i, env in enumerate([{"BRI_LU_EXTEND": "0"}, {"BRI_LU_EXTEND": "1"}, {"BRI_LOOKAHEAD": "0"}]):
    path = f"/tmp/v{i}.npz"
    subprocess.run([sys.executable, os.path.join(root, "tests", "_lu_schedules.py"), path],
                   env=dict(os.environ, PYTHONPATH=root, **env), check=True, timeout=300)
    got = np.load(path)
    print(env, {k: float(got[k]) for k in got.files if k.startswith("err_")}, flush=True)
