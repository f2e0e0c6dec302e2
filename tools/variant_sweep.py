"""Per-pass geometry sweep: every pass of a workload's plan compiled for each specialised-kernel
geometry (256 x 16 one CTA, 128 x 32 two CTAs, 128 x 32 split transposes, 256 x 16 two CTAs) and
timed alone (CUDA events, warm, state >> L2), against the planner's choice."""
import math
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import paper_2009_01845_b200 as q
from paper_2009_01845_b200 import _native as nat
from paper_2009_01845_b200 import fusion, jit

n = int(os.environ.get("N", "30"))
dt = nat.QSB_C128 if os.environ.get("DT", "c128") == "c128" else nat.QSB_C64
prec = q.Precision.F64 if dt == nat.QSB_C128 else q.Precision.F32
which = sys.argv[1:] or ["trotter4", "variational", "grid"]


def workload(name):
    if name.startswith("trotter"):
        w = int(name[7:] or "1")
        step = q.trotter_step_circuit(q.combine(q.build_x(n), 0.5, q.build_tfim(n, 1.0), 0.5), 0.05)
        return q.Circuit(n).add([g for _ in range(w) for g in step.queue])
    if name == "variational":
        params = np.random.default_rng(42).uniform(0, 2 * math.pi, n * 11)
        return q.variational_circuit(n, 5, params, fused=True)
    return q.random_grid_circuit(3, n // 3, 20, 42)


geos = {"jit": fusion.GEOMETRY_JIT[dt], "2q": fusion.GEOMETRY_JIT_2Q[dt]}
if dt in fusion.GEOMETRY_JIT_2Q_SPLIT:
    geos["split"] = fusion.GEOMETRY_JIT_2Q_SPLIT[dt]
if dt in fusion.GEOMETRY_JIT_2Q_X2:
    geos["x2"] = fusion.GEOMETRY_JIT_2Q_X2[dt]

amp = 16 if dt == nat.QSB_C128 else 8
src = torch.empty((1 << n) * amp // 8, dtype=torch.float64, device="cuda").normal_()
dst = torch.empty_like(src)
stream = torch.cuda.current_stream().cuda_stream


def time_words(words, reps=4):
    c, co = jit.compile_words(words, dt)
    for _ in range(2):
        jit.run(words, dt, src.data_ptr(), dst.data_ptr(), n, stream, c, co)
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(reps):
        jit.run(words, dt, src.data_ptr(), dst.data_ptr(), n, stream, c, co)
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / reps


for name in which:
    circ = workload(name)
    plan = fusion.plan_circuit(list(circ.queue), n, dt, True, True, fusion.GEOMETRY_JIT[dt])
    tot_chosen = tot_best = 0.0
    print(f"== {name} n={n} {'c128' if dt else 'c64'}: {plan.n_passes} passes", flush=True)
    for i, st in enumerate(s for s in plan.steps if isinstance(s, fusion.PassStep)):
        cost = sum(fusion.matrix_cost(g.matrix) for g in st.gates if g.kind in ("g1", "g2"))
        chosen = time_words(st.words)
        row = {}
        for gname, geo in geos.items():
            try:
                w, info = fusion.compile_pass(st.gates, set(st.tile_pos), n, dt, geo)
                row[gname] = (time_words(w), info["transposes"])
            except Exception as e:  # noqa: BLE001
                row[gname] = (float("nan"), str(e)[:40])
        best = min(v[0] for v in row.values() if v[0] == v[0])
        tot_chosen += chosen
        tot_best += min(best, chosen)
        print(f"  pass {i:2d} gates {len(st.gates):3d} cost {cost:6.1f} flags {int(st.words[7]):2d} trans {st.n_transposes:2d} "
              f"chosen {chosen:6.3f} | " + "  ".join(f"{k} {v[0]:6.3f}/{v[1]}" for k, v in row.items()), flush=True)
    print(f"  total chosen {tot_chosen:.2f} ms, best-per-pass {tot_best:.2f} ms", flush=True)
