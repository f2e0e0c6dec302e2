"""SM clock, power and throttle reasons sampled (NVML) while a workload's plan runs back to back
for a few seconds: are FP64-heavy passes power-capped?"""
import os
import sys
import threading
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import pynvml
import torch

import paper_2009_01845_b200 as q
from paper_2009_01845_b200 import engine

n = 30
name = sys.argv[1] if len(sys.argv) > 1 else "trotter4"
if name == "trotter4":
    step = q.trotter_step_circuit(q.combine(q.build_x(n), 0.5, q.build_tfim(n, 1.0), 0.5), 0.05)
    circ = q.Circuit(n).add([g for _ in range(4) for g in step.queue])
elif name == "var":
    import math

    import numpy as np

    circ = q.variational_circuit(n, 5, np.random.default_rng(42).uniform(0, 2 * math.pi, n * 11), fused=True)
elif name == "grid":
    circ = q.random_grid_circuit(3, 10, 20, 42)
else:
    circ = q.qft_circuit(n)
st = q.uniform_state(n, q.Precision.F64)
plan = engine.plan_for_state(st, circ.queue)
holder: dict = {}
engine.run_plan(st, plan, holder)
torch.cuda.synchronize()
pynvml.nvmlInit()
h = pynvml.nvmlDeviceGetHandleByIndex(0)
samples = []
stop = threading.Event()


def poll():
    while not stop.is_set():
        samples.append((pynvml.nvmlDeviceGetClockInfo(h, pynvml.NVML_CLOCK_SM),
                        pynvml.nvmlDeviceGetPowerUsage(h) / 1000.0,
                        pynvml.nvmlDeviceGetCurrentClocksEventReasons(h)))
        time.sleep(0.05)


th = threading.Thread(target=poll)
th.start()
a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
times = []
t_end = time.time() + 6
while time.time() < t_end:
    a.record()
    engine.run_plan(st, plan, holder)
    b.record()
    b.synchronize()
    times.append(a.elapsed_time(b))
stop.set()
th.join()
clk = sorted(s[0] for s in samples)
pw = sorted(s[1] for s in samples)
reasons = {}
for s in samples:
    reasons[s[2]] = reasons.get(s[2], 0) + 1
print(f"{name}: {len(times)} runs, ms min {min(times):.2f} median {sorted(times)[len(times) // 2]:.2f} max {max(times):.2f}")
print(f"sm clock MHz min {clk[0]} median {clk[len(clk) // 2]} max {clk[-1]}; power W median {pw[len(pw) // 2]:.0f} max {pw[-1]:.0f}")
print("reason bitmasks (count):", {hex(k): v for k, v in reasons.items()})
