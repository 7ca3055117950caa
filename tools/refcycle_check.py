import sys, time, json
sys.path.insert(0, '.')
from oracle.oracle import RefCycleOracle
import numpy as np
R = RefCycleOracle()
t = time.time()
snaps = R.nature_run(16, 16, 2*np.pi*10/4, 2*np.pi*10/4, 24.0, 24.0, 12.0, 3)
print("nature", snaps.shape, np.abs(snaps).max(), time.time()-t)
cfg = {"grid": {"nx": 16, "ny": 16, "lx": 2*np.pi*10/4, "ly": 2*np.pi*10/4}, "cycles": 3,
       "ensemble_size": 4, "spinup_hours": 24.0, "clim_hours": 48.0, "variant": "ensf",
       "ensf": {"n_steps": 20}}
t = time.time()
print(R.run_experiment(cfg), time.time()-t)
