#!/usr/bin/env python
"""Benchmark: circuit wall-seconds and achieved HBM GB/s of the B200 state-vector engine.

Workload (BASELINE.json configs[1]): the 30-qubit complex128 QFT on one B200, i.e.
qft_circuit(30) (480 gates) applied to a state resident in HBM.  One "step" = one full circuit.
  value      device time per circuit (CUDA events, K steps after W warm-ups), seconds;
  e2e        the same through the public API: Circuit.execute() (|0..0> allocation + plan +
             program upload + passes) and a device->host read of the full result state into
             pinned memory, per step;
  roofline   the dominant kernel (the specialised fused pass): algorithmic bytes per launch
             (one read + one write of the 2^n-amplitude state) / its mean CUDA-event duration,
             against the measured HBM copy peak (MEASURED_PEAKS.json);
  cpu_baseline  the reference algorithm (oracle/ numpy port, all host threads) on a bounded
             sample of the same circuit: three representative gates at n=30, extrapolated.
`--impl reference` runs only that CPU arm.  Under torchrun (N>1) rank 0 reports; the
distributed path shards the state over ranks by global qubits (n = 30 + log2 N, weak scaling).
"""

from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "circuit wall-seconds & achieved HBM GB/s (QFT/variational, c128) at 1/2/4/8 B200"


def _local_device() -> int:
    """This rank's GPU (LOCAL_RANK; modulo the visible devices for validation runs that put
    several ranks on one GPU)."""
    import torch

    n = max(1, torch.cuda.device_count())
    return int(os.environ.get("LOCAL_RANK", 0)) % n


def _peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            p = json.load(f)
        return float(p["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback"


def _ncu_traffic():
    path = os.path.join(ROOT, "profiles", "ncu_pass_summary.json")
    try:
        with open(path) as f:
            d = json.load(f)
        return d.get("dram_bytes_per_launch"), d
    except Exception:
        return None, None


class ClockSampler:
    """NVML polling thread: SM clock and throttle reasons while the timed region runs."""

    REASONS = {
        0x1: "gpu_idle", 0x2: "applications_clocks_setting", 0x4: "sw_power_cap", 0x8: "hw_slowdown",
        0x10: "sync_boost", 0x20: "sw_thermal_slowdown", 0x40: "hw_thermal_slowdown", 0x80: "hw_power_brake_slowdown",
        0x100: "display_clock_setting",
    }

    def __init__(self, index=0, period=0.01):
        self.samples, self.reasons, self.ok = [], set(), False
        self.period = period
        self._stop = threading.Event()
        try:
            import pynvml

            pynvml.nvmlInit()
            self.nv = pynvml
            self.h = pynvml.nvmlDeviceGetHandleByIndex(index)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
            self.ok = True
        except Exception:
            self.max_mhz = None

    def _run(self):
        nv = self.nv
        while not self._stop.is_set():
            try:
                self.samples.append(nv.nvmlDeviceGetClockInfo(self.h, nv.NVML_CLOCK_SM))
                r = nv.nvmlDeviceGetCurrentClocksEventReasons(self.h)
                for bit, name in self.REASONS.items():
                    if r & bit and name != "gpu_idle":
                        self.reasons.add(name)
            except Exception:
                pass
            time.sleep(self.period)

    def __enter__(self):
        if self.ok:
            self.t = threading.Thread(target=self._run, daemon=True)
            self.t.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        if self.ok:
            self.t.join()

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": self.max_mhz, "reasons": sorted(self.reasons), "samples": 0}
        return {"sm_mhz": statistics.median(self.samples), "sm_max_mhz": self.max_mhz,
                "reasons": sorted(self.reasons), "samples": len(self.samples)}


# ------------------------------------------------------------------------------ CPU arm
def cpu_threads():
    try:
        return len(os.sched_getaffinity(0))
    except Exception:
        return os.cpu_count() or 1


def host_ram_bytes():
    try:
        return os.sysconf("SC_PAGE_SIZE") * os.sysconf("SC_PHYS_PAGES")
    except Exception:
        return 0


def cpu_info():
    """CPU model, core count and the numpy / BLAS build the reference arm ran with."""
    import numpy as np

    model = ""
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith("model name"):
                    model = line.split(":", 1)[1].strip()
                    break
    except OSError:
        pass
    blas = ""
    try:
        from threadpoolctl import threadpool_info

        info = [d for d in threadpool_info() if d.get("user_api") == "blas"]
        if info:
            blas = f"{info[0].get('internal_api')} {info[0].get('version')} ({info[0].get('architecture')})"
    except Exception:
        pass
    return {"cpu_model": model, "host_threads": cpu_threads(), "numpy": np.__version__, "blas": blas,
            "host_ram_gb": round(host_ram_bytes() / 2**30, 1)}


class single_core:
    """T=1 for the CPU reference: the process pinned to one core (os.sched_setaffinity, as the
    paper's taskset runs) and the BLAS pool limited to one thread."""

    def __enter__(self):
        self.aff = os.sched_getaffinity(0)
        os.sched_setaffinity(0, {min(self.aff)})
        try:
            from threadpoolctl import threadpool_limits

            self.lim = threadpool_limits(1)
        except Exception:
            self.lim = None
        return self

    def __exit__(self, *a):
        if self.lim is not None:
            self.lim.restore_original_limits()
        os.sched_setaffinity(0, self.aff)


def cpu_qft_full(n: int, threads: int) -> float:
    """Wall seconds of one complete QFT-n c128 through the reference algorithm (the oracle's
    numpy restatement of qsim.Circuit.execute / apply_matrix), |0..0> input."""
    from oracle import statevec as ov

    gates = ov.qft(n)
    t0 = time.perf_counter()
    ov.run(gates, n, n_threads=threads)
    return time.perf_counter() - t0


def cpu_reference_sample(n: int, threads: int):
    """Bounded sample of QFT-n on the CPU reference (the GPU arm's cpu_baseline): the circuit's
    first column -- H(0) and the n-1 CZPow(k, 0) gates, in order -- plus one SWAP, timed on a
    2^n state, extrapolated by gate kind to the full circuit (n H, n(n-1)/2 CZPow, n/2 SWAP)."""
    import numpy as np

    from oracle import statevec as ov

    amps = np.zeros(1 << n, dtype=np.complex128)
    amps[:] = 1.0 / math.sqrt(1 << n)  # touch every page outside the timed region
    gates = ov.qft(n)
    column = [g for g in gates[:n]]  # H(0), CZPow(1,0) ... CZPow(n-1,0)
    swap = [g for g in gates if g[0] == "SWAP"][:1]
    times = {"H": 0.0, "CZPow": 0.0, "SWAP": 0.0}
    seen = {"H": 0, "CZPow": 0, "SWAP": 0}
    for kind, tg, ct, _p, m in column + swap:
        t0 = time.perf_counter()
        ov.apply_matrix(amps, n, tg, m, ct, n_threads=threads)
        times[kind] += time.perf_counter() - t0
        seen[kind] += 1
    counts = {"H": n, "CZPow": n * (n - 1) // 2, "SWAP": n // 2}
    per = {k: times[k] / seen[k] for k in times}
    total = sum(per[k] * counts[k] for k in counts)
    del amps
    return total, per, counts, sum(times.values())


def run_reference_arm(args, rank, world):
    """The reference's CPU path, timed in full: QFT-n c128 (qft_circuit(n).execute(), 480 gates at
    n = 30) through the reference algorithm with every host thread.  The K timed steps TOGETHER
    execute the circuit once: step i applies the i-th contiguous slice of the gate list to the
    running state, so `value` (the sum of the step times) is the measured wall time of one whole
    circuit, and the run ends after one circuit (~6 min at n = 30) instead of K.  Warm-up steps
    run the CPU-only config (QFT-20, BASELINE configs[0]) in full, alternately at T=1 (one
    pinned core, one BLAS thread) and T=all."""
    if rank != 0:
        return
    import numpy as np

    from oracle import statevec as ov

    threads = cpu_threads()
    n = args.qubits
    measured_n = n
    if host_ram_bytes() < (40 << 30) and n > 28:
        measured_n = 28  # the state and its copies do not fit: measure n = 28, extrapolate below
    qft20 = {"T1": [], "Tall": []}
    for i in range(args.warmup):
        if i % 2 == 0:
            with single_core():
                qft20["T1"].append(cpu_qft_full(20, 1))
        else:
            qft20["Tall"].append(cpu_qft_full(20, threads))
    gates = ov.qft(measured_n)
    amps = np.zeros(1 << measured_n, dtype=np.complex128)
    amps[0] = 1.0
    k = max(1, args.steps)
    bounds = [len(gates) * s // k for s in range(k + 1)]
    step_s = []
    for s in range(k):
        t0 = time.perf_counter()
        for _kind, tg, ct, _p, m in gates[bounds[s]:bounds[s + 1]]:
            ov.apply_matrix(amps, measured_n, tg, m, ct, n_threads=threads)
        step_s.append(time.perf_counter() - t0)
    full = sum(step_s)
    # the run's own check: QFT|0> is the uniform state
    err = float(np.max(np.abs(amps - 1.0 / math.sqrt(1 << measured_n))))
    del amps
    scale = 2.0 ** (n - measured_n)
    value = full * scale
    sample = (f"one complete QFT-{measured_n} c128 ({len(gates)} gates) split over the {k} timed steps, "
              f"reference algorithm (numpy port of qsim.Circuit.execute/apply_matrix), {threads} threads"
              + (f"; x{scale:g} extrapolation to n={n} (host RAM too small for the full state)" if scale != 1 else ""))
    best20 = min(qft20["T1"] + qft20["Tall"]) if qft20["T1"] + qft20["Tall"] else None
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": "s", "n_gpus": args.gpus, "steps": k,
        "warmup": args.warmup, "ms_per_step": statistics.mean(step_s) * 1e3 * scale, "higher_is_better": False,
        "scaling": "weak", "vs_baseline": None, "dtype": "c128", "data": "synthetic",
        "config": {"workload": f"QFT {n} qubits complex128 (qft_circuit({n}), {len(ov.qft(n))} gates) on |0..0>",
                   "n_qubits": n, "measured_n": measured_n, "precision": "f64", "parallelism": "host threads",
                   "steps_cover": "the timed steps together execute ONE full circuit (value = their sum)"},
        "cpu_baseline": {"value": value, "unit": "s", "cores": threads, "kind": "port", "sample": sample},
        "e2e": {"value": value, "unit": "s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "qft20": {"T1_s": min(qft20["T1"]) if qft20["T1"] else None,
                  "Tall_s": min(qft20["Tall"]) if qft20["Tall"] else None, "best_s": best20,
                  "what": "BASELINE configs[0]: full QFT-20 c128 on the CPU reference, T=1 (pinned core, "
                          "1 BLAS thread) and T=all"},
        "parity": {"check": f"QFT-{measured_n}|0> == uniform state", "max_abs_err": err},
        "host": cpu_info(),
        "step_seconds": step_s,
    }
    print(json.dumps(line), flush=True)


# ------------------------------------------------------------------------------ GPU arm
def run_gpu_arm(args, rank, world):
    import torch

    import paper_2009_01845_b200 as q
    from paper_2009_01845_b200 import engine
    from paper_2009_01845_b200.fusion import PassStep

    torch.cuda.set_device(_local_device())
    if world > 1:
        return run_distributed_arm(args, rank, world)

    n = args.qubits
    prec = q.Precision.F64 if args.precision == "f64" else q.Precision.F32
    if n > q.max_qubits():
        q.set_max_qubits(n)
    circuit = q.qft_circuit(n) if args.workload == "qft" else q.variational_circuit(
        n, 5, __import__("numpy").random.default_rng(42).uniform(0, 2 * math.pi, n * 11), fused=True)
    state = q.uniform_state(n, prec)
    plan = engine.plan_for_state(state, circuit.queue)
    holder: dict = {}
    for _ in range(args.warmup):
        engine.run_plan(state, plan, holder)
    torch.cuda.synchronize()
    evs: list = []
    t0 = torch.cuda.Event(enable_timing=True)
    t1 = torch.cuda.Event(enable_timing=True)
    with ClockSampler(_local_device()) as clk:
        t0.record()
        for _ in range(args.steps):
            engine.run_plan(state, plan, holder, events=evs)
        t1.record()
        torch.cuda.synchronize()
    ms = t0.elapsed_time(t1) / args.steps
    value = ms / 1e3
    launches = [a.elapsed_time(b) for a, b in evs]
    n_pass = sum(1 for s in plan.steps if isinstance(s, PassStep))
    amp_bytes = prec.itemsize
    pass_bytes = 2 * (1 << n) * amp_bytes
    mean_pass_ms = statistics.mean(launches) if launches else float("nan")
    achieved = pass_bytes / (mean_pass_ms * 1e-3) / 1e9
    peak, peak_kind = _peaks()
    traffic, _ncu = _ncu_traffic()
    sweeps = plan.state_sweeps()
    circuit_gbs = sweeps * pass_bytes / value / 1e9

    # e2e through the public API, host readback of the full state into pinned memory
    e2e_steps = max(1, min(args.steps, 3))
    pinned = None
    try:
        pinned = torch.empty((1 << n,), dtype=prec.torch_dtype, pin_memory=True)
    except Exception:
        pinned = None
    del state
    holder.clear()
    torch.cuda.empty_cache()
    h2d = sum(int(s.words.nbytes) for s in plan.steps if isinstance(s, PassStep))
    d2h = (1 << n) * amp_bytes if pinned is not None else 16
    torch.cuda.synchronize()
    e2e_times = []
    for i in range(e2e_steps + 1):
        w0 = time.perf_counter()
        st = circuit.execute(precision=prec)
        if pinned is not None:
            st.copy_to_host(pinned)  # chunked over four copy streams
        else:
            st.tensor[:1].cpu()
        torch.cuda.synchronize()
        dt = time.perf_counter() - w0
        del st
        if i > 0:  # the first call pays one-off allocations
            e2e_times.append(dt)
    e2e = statistics.mean(e2e_times)

    # the timed kernels' own result, checked at full size: QFT-n on a basis state |k> against the
    # analytic DFT column (the reference's known answer, tests/test_circuit.py:189-201), on device
    from paper_2009_01845_b200.verify import dft_column_error

    parity = None
    if args.workload == "qft":
        k = int(__import__("numpy").random.default_rng(n).integers(1 << n))
        st = q.basis_state(n, k, prec)
        engine.run_plan(st, plan, {})
        err = dft_column_error(st, k)
        tol = 1e-12 if prec is q.Precision.F64 else 1e-5
        parity = {"check": f"QFT-{n}|k={k}> vs analytic DFT column (same plan / kernels as timed)",
                  "max_abs_err": err, "tol": tol, "ok": err <= tol}
        del st
        torch.cuda.empty_cache()

    others = {} if args.no_extra_workloads else extra_workloads(q, engine, n, peak)

    cpu = None
    if rank == 0 and not args.no_cpu_baseline:
        threads = cpu_threads()
        sn = n if host_ram_bytes() >= (48 << 30) else min(n, 28)
        total, per, counts, spent = cpu_reference_sample(sn, threads)
        scale = 2.0 ** (n - sn)
        cpu = {"value": total * scale, "unit": "s", "cores": threads, "kind": "port",
               "sample": f"first QFT-{sn} column (H(0) + {sn - 1} CZPow(k,0)) + SWAP(0,{sn - 1}) on the CPU reference "
                         f"(numpy port of qsim.apply_matrix, {threads} threads; {spent:.1f} s of CPU work), per-gate "
                         f"{', '.join(f'{k}={v:.2f}s' for k, v in per.items())}, extrapolated to "
                         f"{sum(counts.values())} gates" + (f", x{scale:g} to n={n}" if scale != 1 else "")
                         + "; bench.py --impl reference times the whole circuit",
               "qft20_s": cpu_qft_full(20, threads), "host": cpu_info()}

    line = {
        "metric": METRIC, "value": value, "unit": "s", "n_gpus": 1, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": ms, "higher_is_better": False, "scaling": "weak", "vs_baseline": None,
        "dtype": "c128" if prec is q.Precision.F64 else "c64", "data": "synthetic",
        "config": {"workload": f"{'QFT' if args.workload == 'qft' else 'variational(L=5, fused)'} {n} qubits "
                               f"{'complex128' if prec is q.Precision.F64 else 'complex64'} on 1 B200, "
                               f"{len(circuit.queue)} gates, state resident in HBM",
                   "n_qubits": n, "gates": len(circuit.queue), "passes": n_pass, "state_sweeps": sweeps,
                   "state_bytes": (1 << n) * amp_bytes, "parallelism": "single GPU",
                   "l2": "inputs (state) far larger than the 126 MB L2; no flush needed"},
        "hbm": {"circuit_effective_gbs": circuit_gbs, "per_pass_ms": mean_pass_ms},
        "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s", "frac": achieved / peak,
                     "traffic": traffic, "peak_kind": peak_kind, "kernel": "qsb_pass_<hash> (NVRTC-specialised fused pass)",
                     "bytes_per_launch": pass_bytes, "launches": len(launches)},
        "e2e": {"value": e2e, "unit": "s", "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h,
                "api": "qft_circuit(n).execute() + StateVector.copy_to_host(pinned)"},
        "workloads": others,
        "parity": parity,
        "gpu_launches": len(plan.steps) * args.steps,
        "clocks": clk.summary(),
        "cpu_baseline": cpu,
    }
    if rank == 0:
        print(json.dumps(line), flush=True)


def extra_workloads(q, engine, n, peak):
    """The other BASELINE configs that fit one GPU, timed the same way (device time per circuit,
    state resident, warm-ups first): variational (RY layers + CZ ladder, L=5, fused) in c128 and
    c64, and the QFT in c64.  hbm_frac = state sweeps x sweep bytes / time / measured peak."""
    import numpy as np
    import torch

    from paper_2009_01845_b200.fusion import PassStep, matrix_cost

    out = {}
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            sm_mhz = float(json.load(f).get("sm_max_mhz", 1965.0))
    except Exception:
        sm_mhz = 1965.0
    params = np.random.default_rng(42).uniform(0, 2 * math.pi, n * 11)
    rows = 3 if n % 3 == 0 else 2
    grid = q.random_grid_circuit(rows, n // rows, 20, 42)
    cases = [("variational_L5_fused_c128", q.variational_circuit(n, 5, params, fused=True), q.Precision.F64),
             ("variational_L5_fused_c64", q.variational_circuit(n, 5, params, fused=True), q.Precision.F32),
             ("qft_c64", q.qft_circuit(n), q.Precision.F32),
             (f"random_grid_{rows}x{n // rows}_20cycles_c128", grid, q.Precision.F64),
             ("trotter_tfim_step_c128", q.trotter_step_circuit(q.combine(q.build_x(n), 0.5, q.build_tfim(n, 1.0), 0.5),
                                                               0.05), q.Precision.F64)]
    # evolve() runs consecutive Trotter steps as one circuit when no callback reads the state in
    # between (evolution.STEP_WINDOW): the same step, four at a time, reported per step
    step = cases[-1][1]
    window = q.Circuit(n).add([g for _ in range(4) for g in step.queue])
    cases.append(("trotter_tfim_4steps_c128", window, q.Precision.F64))
    for name, circ, prec in cases:
        st = q.uniform_state(n, prec)
        plan = engine.plan_for_state(st, circ.queue)
        holder: dict = {}
        for _ in range(3):
            engine.run_plan(st, plan, holder)
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        reps = 3
        a.record()
        for _ in range(reps):
            engine.run_plan(st, plan, holder)
        b.record()
        torch.cuda.synchronize()
        sec = a.elapsed_time(b) / reps / 1e3
        sweeps = plan.state_sweeps()
        gbs = sweeps * 2 * (1 << n) * prec.itemsize / sec / 1e9
        # FP roofline of the gate arithmetic: FMAs per amplitude of the (structure-specialised)
        # gate bodies the plan applies, at the B200 FMA rate of that precision (FP64: 64 / clk /
        # SM, FP32: 128 / clk / SM) and the max SM clock
        fmas = sum(matrix_cost(g.matrix) for s_ in plan.steps if isinstance(s_, PassStep)
                   for g in s_.gates if g.kind in ("g1", "g2")) * (1 << n)
        rate = (64 if prec is q.Precision.F64 else 128) * 148 * sm_mhz * 1e6
        fp_s = fmas / rate
        hbm_s = sweeps * 2 * (1 << n) * prec.itemsize / (peak * 1e9)
        per = 4 if name == "trotter_tfim_4steps_c128" else 1
        if per > 1:
            sec, hbm_s, fp_s = sec / per, hbm_s / per, fp_s / per  # (effective GB/s is unchanged)
        out[name] = {"seconds": sec, "gates": len(circ.queue), "per": "Trotter step" if per > 1 else "circuit",
                     "passes": sum(1 for s_ in plan.steps if isinstance(s_, PassStep)),
                     "effective_gbs": gbs, "hbm_frac": gbs / peak,
                     "hbm_floor_s": hbm_s, "fp_floor_s": fp_s,
                     "bound": "fp64" if (fp_s > hbm_s and prec is q.Precision.F64) else
                              ("fp32" if fp_s > hbm_s else "hbm"),
                     "roofline_frac": max(hbm_s, fp_s) / sec}
        del st, holder
        torch.cuda.empty_cache()
    out.update(_api_workloads(q, n))
    out.update(_big_state_workloads(q, engine, n + 3, peak))
    return out


def _api_workloads(q, n):
    """Whole API calls (device-synchronised wall time, warm): exact sampling of all n qubits of a
    QFT state (1e5 shots; bit-identical to numpy's cumsum + searchsorted on the reference's
    probabilities) and a 20-step adiabatic TFIM evolution (dt 0.05, T 1; the evolution API with
    its windowed Trotter circuits, plan templates and host work included)."""
    import time

    import torch

    out = {}
    try:
        st = q.qft_circuit(n).execute(q.basis_state(n, 12345))
        q.sample(st, range(n), 100000, 42)
        torch.cuda.synchronize()
        best = float("inf")
        for _ in range(3):
            t0 = time.perf_counter()
            q.sample(st, range(n), 100000, 42)
            torch.cuda.synchronize()
            best = min(best, time.perf_counter() - t0)
        out[f"sample_all_{n}_qubits_1e5_shots"] = {"seconds": best, "per": "call (wall, device-synchronised)"}
        del st
        torch.cuda.empty_cache()
        cfg = q.EvolutionConfig(q.Solver.TROTTER, 0.05, 1.0)
        q.adiabatic_evolve(q.build_x(n), q.build_tfim(n, 0.9), q.Schedule.linear(), cfg)
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        psi = q.adiabatic_evolve(q.build_x(n), q.build_tfim(n, 1.0), q.Schedule.linear(), cfg)
        torch.cuda.synchronize()
        sec = time.perf_counter() - t0
        out[f"adiabatic_tfim_{n}_20steps_c128"] = {"seconds": sec / 20, "per": "Trotter step (wall, device-synchronised)",
                                                  "total_s": sec}
        del psi
        torch.cuda.empty_cache()
    except Exception as exc:  # the headline stands; say why these are missing
        torch.cuda.empty_cache()
        out["api_workloads"] = {"error": f"{type(exc).__name__}: {exc}"[:300]}
    return out


def _big_state_workloads(q, engine, n, peak):
    """QFT at n + 3 qubits (n = 33 c128: 137 GB, the per-GPU shard of the 36-qubit / 8-GPU
    target) through Circuit.execute's engine path: no room for an out-of-place scratch, so the
    final SWAPs become a qubit relabelling left on the state (its canonical read is timed apart).
    Skipped when the GPU lacks the memory."""
    import torch

    try:
        torch.cuda.empty_cache()
        free, _ = torch.cuda.mem_get_info()
        need = (1 << n) * 16
        if free < need + (8 << 30):
            return {f"qft_{n}_c128": {"skipped": f"needs {need / 2**30:.0f} GiB free, {free / 2**30:.0f} GiB free"}}
        q.set_max_qubits(max(n, q.max_qubits()))
        st = q.uniform_state(n)
        circ = q.qft_circuit(n)
        cache, holder = {}, {}
        engine.run_gates(st, circ.queue, None, holder, cache)
        st._canonicalize()
        torch.cuda.synchronize()
        a, b, c = (torch.cuda.Event(enable_timing=True) for _ in range(3))
        a.record()
        plan = engine.run_gates(st, circ.queue, None, holder, cache)
        b.record()
        st._canonicalize()
        c.record()
        torch.cuda.synchronize()
        sec = a.elapsed_time(b) / 1e3
        sweeps = plan.state_sweeps()
        gbs = sweeps * 2 * need / sec / 1e9
        res = {f"qft_{n}_c128": {"seconds": sec, "passes": plan.n_passes, "state_sweeps": sweeps,
                                 "effective_gbs": gbs, "hbm_frac": gbs / peak,
                                 "swaps": "relabelled (qubit map kept on the state)",
                                 "canonical_read_s": b.elapsed_time(c) / 1e3}}
        # BASELINE config 4's circuit (grid 3x11, 20 cycles) and config 5's TFIM Trotter steps
        # (four per circuit, as evolve() plans them) at the same 137 GB per GPU, in place
        step = q.trotter_step_circuit(q.combine(q.build_x(n), 0.5, q.build_tfim(n, 1.0), 0.5), 0.05)
        for name, circ, per in ((f"trotter_tfim_4steps_{n}_c128", q.Circuit(n).add([g for _ in range(4) for g in step.queue]), 4),
                                (f"random_grid_3x{n // 3}_20cycles_{n}_c128", q.random_grid_circuit(3, n // 3, 20, 42), 1)):
            plan = engine.plan_for_state(st, circ.queue)
            engine.run_plan(st, plan, holder)
            torch.cuda.synchronize()
            a.record()
            engine.run_plan(st, plan, holder)
            b.record()
            torch.cuda.synchronize()
            sec = a.elapsed_time(b) / 1e3
            sweeps = plan.state_sweeps()
            gbs = sweeps * 2 * need / sec / 1e9
            res[name] = {"seconds": sec / per, "per": "Trotter step" if per > 1 else "circuit", "passes": plan.n_passes,
                         "state_sweeps": sweeps / per, "effective_gbs": gbs, "hbm_frac": gbs / peak}
        del st, holder, cache
        torch.cuda.empty_cache()
        return res
    except Exception as exc:  # the headline stands; say why this one is missing
        torch.cuda.empty_cache()
        return {f"qft_{n}_c128": {"error": f"{type(exc).__name__}: {exc}"[:300]}}


def run_distributed_arm(args, rank, world):
    """N > 1: QFT on n = qubits + log2(N) qubits, one shard (2^qubits amplitudes) per rank;
    global<->local exchanges are batched all-to-alls (grouped NCCL send/recv, sharding.exchange)
    scheduled by the DAG planner (sharding.plan_batched) (weak scaling)."""
    import torch
    import torch.distributed as dist

    import paper_2009_01845_b200 as q
    from paper_2009_01845_b200 import sharding as sd

    # QSB_BENCH_DIST_BACKEND=gloo: a validation run of this arm with several ranks sharing one GPU
    # (NCCL refuses that): transfers staged through host memory, numbers not representative
    backend_name = os.environ.get("QSB_BENCH_DIST_BACKEND", "nccl")
    if not dist.is_initialized():
        if backend_name == "nccl":
            dist.init_process_group("nccl", device_id=torch.device("cuda", _local_device()))
        else:
            dist.init_process_group(backend_name)
    g = world.bit_length() - 1
    n = args.qubits + g
    prec = q.Precision.F64 if args.precision == "f64" else q.Precision.F32
    q.set_max_qubits(max(n, q.max_qubits()))
    circuit = q.qft_circuit(n)
    comm = sd.TorchComm() if backend_name == "nccl" else sd.HostStagedComm()
    backend = sd.CudaBackend(prec)
    exec_plan = sd.plan_batched(circuit, world)
    cache: dict = {}

    def step():
        return sd.run_sharded(circuit, world, None, prec, None, comm, backend, cache, exec_plan)

    for _ in range(args.warmup):
        sh = step()
        del sh
    torch.cuda.synchronize()
    comm.barrier()
    t0 = torch.cuda.Event(enable_timing=True)
    t1 = torch.cuda.Event(enable_timing=True)
    with ClockSampler(_local_device()) as clk:
        t0.record()
        for _ in range(args.steps):
            sh = step()
            del sh
        t1.record()
        torch.cuda.synchronize()
    ms = torch.tensor([t0.elapsed_time(t1) / args.steps], device="cuda")
    dist.all_reduce(ms, op=dist.ReduceOp.MAX)
    comm.barrier()
    # e2e: public API (execute_distributed) + a device->host read of the shard norm
    e2e_t = []
    for _ in range(2):
        w0 = time.perf_counter()
        sh = sd.execute_distributed(circuit, prec, comm=comm)
        loc = next(iter(sh.shards.values()))
        _ = float(torch.linalg.vector_norm(loc).item())
        comm.barrier()
        e2e_t.append(time.perf_counter() - w0)
        del sh, loc
    value = float(ms.item()) / 1e3
    shard_bytes = (1 << args.qubits) * prec.itemsize
    exch_bytes = int(exec_plan.shard_fraction_moved() * shard_bytes)
    nvlink, t_exch = _time_exchanges(sd, comm, backend, prec, n, exec_plan, shard_bytes)
    roofline, launches = _dist_summary(cache, exec_plan.n_exchanges, value, t_exch, shard_bytes, prec.itemsize,
                                       sd.TorchComm.CHUNK_BYTES, g)
    workloads = {"adiabatic_tfim_step": _dist_adiabatic(q, sd, comm, n, world),
                 "random_grid_20_cycles": _dist_grid(q, sd, comm, n, world, prec)}
    line = {
        "metric": METRIC, "value": value, "unit": "s", "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": value * 1e3, "higher_is_better": False, "scaling": "weak", "vs_baseline": None,
        "dtype": "c128" if prec is q.Precision.F64 else "c64", "data": "synthetic",
        "config": {"workload": f"QFT {n} qubits sharded over {world} GPUs (2^{args.qubits} amplitudes per GPU)",
                   "n_qubits": n, "parallelism": f"global-qubit sharding x{world}, batched NCCL all-to-all exchanges"
                   + ("" if backend_name == "nccl" else f" (VALIDATION RUN: {backend_name}, host-staged, ranks sharing GPUs)"),
                   "exchanges": exec_plan.n_exchanges, "reference_planner_reshuffles": sd.plan(circuit, world).n_reshuffles,
                   "global_qubits": list(exec_plan.global_qubits), "exchange_bytes_per_gpu": exch_bytes},
        "e2e": {"value": min(e2e_t), "unit": "s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 8,
                "api": "sharding.execute_distributed + per-rank norm readback"},
        "gpu_launches": launches,
        "roofline": roofline,
        "nvlink": nvlink,
        "workloads": workloads,
        "clocks": clk.summary(),
        "cpu_baseline": None,
    }
    if rank == 0:
        print(json.dumps(line), flush=True)
    dist.destroy_process_group()


def _dist_summary(cache, n_exchanges, value, t_exch, shard_bytes, itemsize, chunk_bytes, k=1):
    """(roofline, launches) of one sharded step: the local fused passes' HBM rate (step time minus
    the measured exchange time) and the kernels one step launches per GPU (k: qubits per
    exchange; each exchange packs and unpacks 2^k - 1 parts)."""
    # the per-shard fused plans of one step (the runner's cache holds exactly those)
    plans = [p for p in cache.values() if hasattr(p, "state_sweeps")]
    sweeps = sum(p.state_sweeps() for p in plans)
    local_s = value - (n_exchanges * t_exch if t_exch else 0.0)
    hbm_peak, peak_kind = _peaks()
    achieved = sweeps * 2 * shard_bytes / local_s / 1e9 if local_s > 0 and sweeps else None
    roofline = {"bound": "hbm", "achieved": achieved, "peak": hbm_peak, "unit": "GB/s",
                "frac": achieved / hbm_peak if achieved else None, "traffic": None, "peak_kind": peak_kind,
                "sweeps_per_step": sweeps,
                "note": "local fused passes per GPU: step time minus the measured exchange time"}
    peers = (1 << k) - 1
    part_amps = shard_bytes // itemsize >> k
    chunk = max(1, min(part_amps, chunk_bytes // itemsize // peers))
    chunks = -(-part_amps // chunk)
    # plan steps + (pack + unpack) per peer per chunk per exchange + the |0> initialisation
    launches = sum(len(p.steps) for p in plans) + n_exchanges * 2 * peers * chunks + 1
    return roofline, launches


def _dist_adiabatic(q, sd, comm, n, world, steps=4):
    """BASELINE config 5 at this scale: adiabatic TFIM Trotter steps (dt 0.05) on a state that
    stays sharded (|+>^n built per shard, every step's circuit applied to the resident shards,
    energy taken without a gather); device time per step, max over ranks."""
    import torch
    import torch.distributed as dist

    from paper_2009_01845_b200.evolution import trotter_step_circuit

    try:
        h0, h1 = q.build_x(n), q.build_tfim(n, 1.0)
        T = 1.0

        def h_at(t):
            s_ = min(max(t / T, 0.0), 1.0)
            return q.combine(h0, 1.0 - s_, h1, s_)

        sh = sd.uniform_sharded(n, world, q.Precision.F64, comm)
        circuits = [trotter_step_circuit(h_at(0.05 * (k + 1)), 0.05) for k in range(steps + 1)]
        sd.apply_sharded(sh, circuits[0])  # warm-up: kernels compiled, staging allocated
        torch.cuda.synchronize()
        comm.barrier()
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record()
        for c in circuits[1:]:
            sd.apply_sharded(sh, c)
        e1.record()
        torch.cuda.synchronize()
        t = torch.tensor([e0.elapsed_time(e1) / steps / 1e3], device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        energy = sd.expectation_sharded(h1, sh)
        del sh
        torch.cuda.empty_cache()
        return {"value": float(t.item()), "unit": "s per Trotter step", "n_qubits": n, "steps": steps,
                "gates_per_step": len(circuits[1].queue), "energy_after": energy,
                "exchanges_per_step": sd.plan_batched(circuits[1], world).n_exchanges,
                "reference_planner_reshuffles_per_step": sd.plan(circuits[1], world).n_reshuffles,
                "what": "adiabatic_evolve_sharded step, state resident in shards (no gather)"}
    except Exception as exc:  # the QFT line stands; say why this one is missing
        return {"error": f"{type(exc).__name__}: {exc}"[:300]}


def _dist_grid(q, sd, comm, n, world, prec, cycles=20):
    """BASELINE config 4 at this scale: the supremacy-style random circuit on a 3 x n/3 grid (2 x n/2
    or 1 x n when 3 does not divide n), sharded with the reference's reshuffle plan; device time of one
    circuit after a warm-up run, max over ranks."""
    import torch
    import torch.distributed as dist

    try:
        rows = 3 if n % 3 == 0 else (2 if n % 2 == 0 else 1)
        circuit = q.random_grid_circuit(rows, n // rows, cycles, 42)
        exec_plan = sd.plan_batched(circuit, world)
        cache: dict = {}
        sh = sd.run_sharded(circuit, world, None, prec, None, comm, sd.CudaBackend(prec), cache, exec_plan)
        del sh
        torch.cuda.synchronize()
        comm.barrier()
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record()
        sh = sd.run_sharded(circuit, world, None, prec, None, comm, sd.CudaBackend(prec), cache, exec_plan)
        e1.record()
        torch.cuda.synchronize()
        t = torch.tensor([e0.elapsed_time(e1) / 1e3], device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        del sh
        torch.cuda.empty_cache()
        return {"value": float(t.item()), "unit": "s", "n_qubits": n, "grid": f"{rows}x{n // rows}",
                "cycles": cycles, "gates": len(circuit.queue), "exchanges": exec_plan.n_exchanges,
                "reference_planner_reshuffles": sd.plan(circuit, world).n_reshuffles}
    except Exception as exc:  # the QFT line stands; say why this one is missing
        return {"error": f"{type(exc).__name__}: {exc}"[:300]}


def _time_exchanges(sd, comm, backend, prec, n, exec_plan, shard_bytes, reps=4):
    """One batched exchange of every global qubit with a local one in isolation (the all-to-all
    the planner issues: pack, grouped NCCL send/recv, unpack), max over ranks: the NVLink
    number (bytes each GPU sends / time, unidirectional)."""
    import torch
    import torch.distributed as dist

    try:
        sh = sd._make_sharded(None, exec_plan.global_qubits, comm, backend, prec, n)
        g = sh.n_global
        pairs = list(zip(sh.global_qubits, sh.local_qubits[:g]))
        back = [(b, a) for a, b in pairs]
        sd.exchange(sh, pairs)  # warm-up (staging buffers, NCCL channels)
        sd.exchange(sh, back)
        torch.cuda.synchronize()
        comm.barrier()
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record()
        for k in range(reps):
            sd.exchange(sh, pairs if k % 2 == 0 else back)
        e1.record()
        torch.cuda.synchronize()
        t = torch.tensor([e0.elapsed_time(e1) / reps / 1e3], device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        t_exch = float(t.item())
        sent = shard_bytes - (shard_bytes >> g)
        del sh
        torch.cuda.empty_cache()
        return ({"achieved": sent / t_exch / 1e9, "peak": 900.0, "unit": "GB/s", "frac": sent / t_exch / 900e9,
                 "bytes_per_exchange_per_gpu": sent, "ms_per_exchange": t_exch * 1e3, "qubits_per_exchange": g,
                 "what": f"{g}-qubit all-to-all exchange (2^{g}-1 peers), bytes sent per GPU / time (unidirectional)"},
                t_exch)
    except Exception as exc:  # the step's own number stands; say why this one is missing
        return {"error": f"{type(exc).__name__}: {exc}"[:300]}, None


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--qubits", type=int, default=30)
    ap.add_argument("--precision", choices=["f64", "f32"], default="f64")
    ap.add_argument("--workload", choices=["qft", "variational"], default="qft")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-extra-workloads", action="store_true")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3)
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    if args.impl == "reference":
        run_reference_arm(args, rank, world)
        return
    run_gpu_arm(args, rank, world)


if __name__ == "__main__":
    main()
