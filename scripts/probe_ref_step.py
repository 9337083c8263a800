# time one reference-mode run_step of the reference CPU build at a given latent
import sys, time, os, dataclasses
sys.path.insert(0, os.getcwd())
import numpy as np
from oracle import ref as R
from oracle import patchsim_np as O
hw = int(sys.argv[1]) if len(sys.argv) > 1 else 128
cfg = (4, 320, 3, 32, 2048, -1)
cond = O.random_condition(2048, 7)
x = O.random_normal(1, 4, hw, hw, 1234)
t0 = time.time(); m = R.Model(cfg, 42); print("build", time.time() - t0, flush=True)
rr = R.PatchRunner(m, cond, hw, hw, mode="reference")
t0 = time.time(); e = rr.step("run_step", x, 980, 0); print(f"step {hw}: {time.time()-t0:.2f}s", flush=True)
