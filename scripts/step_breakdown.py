"""Per-launch device time of ONE UNet step in the pipelined (graph-replayed) generation.

usage: python scripts/step_breakdown.py [LATENT] [DTYPE] [BANDS] [PDL(0|1)]
CUPTI kernel records (torch.profiler) of one generation; prints the launches between the
21st and 22nd DDIM update (one displaced step) with grid and duration, and per-kernel
totals over the whole generation.  PDL off (default) so a kernel's span does not include
its griddepcontrol.wait on the predecessor.
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402
from torch.profiler import ProfilerActivity, profile  # noqa: E402

from paper_2402_19481_b200 import _native as NAT  # noqa: E402
from paper_2402_19481_b200 import patchsim as P  # noqa: E402

hw = int(sys.argv[1]) if len(sys.argv) > 1 else 128
dtype = sys.argv[2] if len(sys.argv) > 2 else "bf16"
bands = int(sys.argv[3]) if len(sys.argv) > 3 else 1
pdl = int(sys.argv[4]) if len(sys.argv) > 4 else 0
NAT.lib().pp_set_pdl(pdl)
m = P.build_model(P.SDXL_SHAPE, 42)
cond = P.random_condition(2048, 7)
r = P.PatchRunner(m, cond, hw, hw, mode="displaced", n_devices=bands, warmup_steps=4, dtype=dtype)
x = P.random_normal(1, 4, hw, hw, 1234)
plan, abar = P.make_plan(1000, 50), P.make_schedule(1000)
r.sample(x, plan, abar)
r.sample(x, plan, abar)
torch.cuda.synchronize()
with profile(activities=[ProfilerActivity.CUDA]) as prof:
    r.sample(x, plan, abar)
    torch.cuda.synchronize()
ev = [e for e in prof.events() if str(getattr(e, "device_type", "")).endswith("CUDA")
      and "Memcpy" not in e.name and "Memset" not in e.name]
ev.sort(key=lambda e: e.time_range.start)
dd = [i for i, e in enumerate(ev) if "ddim" in e.name]
print(f"latent {hw} {dtype} bands {bands} pdl {pdl}: {len(ev)} kernels, generation "
      f"{r.last_device_ms():.3f} ms")
if len(dd) > 22:
    a, b = dd[20], dd[21]
    tot = 0.0
    t_first = ev[a].time_range.end
    for e in ev[a + 1:b + 1]:
        us = e.time_range.elapsed_us()
        tot += us
        gap = e.time_range.start - t_first
        name = e.name.replace("void pp::(anonymous namespace)::", "").split("(")[0]
        print(f"{us:8.2f} us  start+{gap:8.1f}  {name[:70]}")
    print(f"sum {tot:.1f} us, span {ev[b].time_range.end - t_first:.1f} us")
agg = {}
for e in ev:
    name = e.name.replace("void pp::(anonymous namespace)::", "").split("(")[0]
    s, c = agg.get(name, (0.0, 0))
    agg[name] = (s + e.time_range.elapsed_us(), c + 1)
for k, (s, c) in sorted(agg.items(), key=lambda kv: -kv[1][0]):
    print(f"{s / 1e3:9.3f} ms {c:6d} x {s / c:8.2f} us  {k[:70]}")
