"""Runs planned gate sequences on a device state (the replacement of the reference's per-gate
loop, /root/reference/pkg/src/qsim/circuit.py:121-124).

A Plan (fusion.py) is a list of PassSteps (one qsb_run_pass launch = one HBM sweep for many
gates) and GateSteps (one qsb_apply_matrix launch for a sparse stand-alone gate).  Passes that
carry a tile-external permutation (folded SWAPs) write out of place into a scratch buffer
of the same size, after which the buffers trade places.
"""

from __future__ import annotations

import os
import warnings

import numpy as np

from . import _native as nat
from . import jit
from .errors import ShapeError, SimulationError
from .fusion import GEOMETRY, GEOMETRY_JIT, GateStep, PassStep, Plan, compile_pass, plan_circuit
from .gates import gate_matrix

# QSB_FUSION=0 disables pass fusion (every gate becomes its own kernel launch)
FUSION_DEFAULT = os.environ.get("QSB_FUSION", "1") != "0"


def _free_bytes() -> int:
    torch = nat.torch_mod()
    free, _total = torch.cuda.mem_get_info()
    return int(free)


# cudaMemGetInfo costs ~2 ms; scratch buffers up to this size are assumed to fit without asking
_SCRATCH_ASSUMED = 256 << 20


# (time, free bytes, torch-reserved bytes) of the last cudaMemGetInfo: reused for 0.5 s while
# this process's reserved memory has not moved by more than 256 MB
_FREE_CACHE = [0.0, 0, 0]


def scratch_fits(nbytes: int) -> bool:
    """Whether an out-of-place pass may allocate a scratch state of `nbytes` (plus headroom).
    The free-memory query (~2 ms) is cached briefly: a time-dependent evolution asks several
    times per step."""
    if nbytes <= _SCRATCH_ASSUMED:
        return True
    import time

    torch = nat.torch_mod()
    now = time.monotonic()
    reserved = int(torch.cuda.memory_reserved())
    if now - _FREE_CACHE[0] > 0.5 or abs(reserved - _FREE_CACHE[2]) > (256 << 20):
        _FREE_CACHE[:] = [now, _free_bytes(), reserved]
    return _FREE_CACHE[1] > nbytes + (512 << 20)


def default_geometry(dtype: int):
    """Tile geometry of the kernels that will run the plan: the specialised (NVRTC) kernels'
    when they are available, else the interpreter's."""
    return GEOMETRY_JIT[dtype] if jit.available() else GEOMETRY[dtype]


def plan_for_state(state, specs, fuse: bool | None = None) -> Plan:
    fuse = FUSION_DEFAULT if fuse is None else fuse
    bytes_needed = state.n_amps * state.precision.itemsize
    allow_ext = scratch_fits(bytes_needed)
    dtype = state.precision.qsb_dtype
    geo = default_geometry(dtype)
    return plan_circuit(specs, state.n_qubits, dtype, allow_ext_perm=allow_ext, fuse=fuse, geometry=geo)


def _apply_gate_step(ptr, n, dtype, g, stream):
    lib = nat.lib()
    tb = np.array(g.targets, dtype=np.int32)
    cb = np.array(g.controls or (0,), dtype=np.int32)
    if g.kind == "diag":
        dim = len(g.matrix)
        mat = np.ascontiguousarray(np.diag(g.matrix))
        kernel = nat.KERNEL_DIAGONAL
    elif g.kind == "swap":
        mat = np.array([[1, 0, 0, 0], [0, 0, 1, 0], [0, 1, 0, 0], [0, 0, 0, 1]], dtype=np.complex128)
        kernel = nat.KERNEL_PERMUTATION
    else:
        mat = np.ascontiguousarray(g.matrix, dtype=np.complex128)
        kernel = nat.KERNEL_AUTO
    nat.check(
        lib.qsb_apply_matrix(ptr, n, dtype, len(g.targets), tb.ctypes.data, len(g.controls), cb.ctypes.data,
                             mat.ctypes.data, kernel, stream),
        "apply_matrix",
    )


# qsb_apply_batch keeps states up to this size in shared memory, and walks larger ones with a
# grid-synchronised launch (include/qsb200.h).  A gate list seen for the first time goes through
# the grid walk up to GRID_BATCH_MAX_STATE_BYTES: below it the per-gate sweeps (L2-resident up to
# ~64 MB) cost less than planning the list into fused passes on the host (10-50 ms).
BATCH_MAX_STATE_BYTES = 131072
GRID_BATCH_MAX_STATE_BYTES = 256 << 20
# QSB_FIRST_RUN_BATCH=0: plan mid-size gate lists into fused passes from their first run
FIRST_RUN_BATCH = os.environ.get("QSB_FIRST_RUN_BATCH", "1") != "0"


def _gate_matrix_and_class(g):
    """The (matrix, kernel class) one stand-alone NGate is launched with (_apply_gate_step)."""
    if g.kind == "diag":
        return np.diag(g.matrix), nat.KERNEL_DIAGONAL
    if g.kind == "swap":
        return _SWAP4, nat.KERNEL_PERMUTATION
    return np.asarray(g.matrix, dtype=np.complex128), nat.KERNEL_AUTO


_SWAP4 = np.array([[1, 0, 0, 0], [0, 0, 1, 0], [0, 1, 0, 0], [0, 0, 0, 1]], dtype=np.complex128)


def pack_gate_batch(gates):
    """Host arrays of one qsb_apply_batch call: target counts, 2 target bits per gate, control
    counts, the control bits back to back, 32 doubles of matrix per gate, kernel classes."""
    k = len(gates)
    nt = np.zeros(k, dtype=np.int32)
    tb = np.zeros(2 * k, dtype=np.int32)
    nc = np.zeros(k, dtype=np.int32)
    cb = np.zeros(max(1, sum(len(g.controls) for g in gates)), dtype=np.int32)
    mats = np.zeros((k, 16), dtype=np.complex128)
    kc = np.zeros(k, dtype=np.int32)
    c = 0
    for i, g in enumerate(gates):
        m, kc[i] = _gate_matrix_and_class(g)
        t = len(g.targets)
        nt[i] = t
        tb[2 * i:2 * i + t] = g.targets
        nc[i] = len(g.controls)
        cb[c:c + nc[i]] = g.controls
        c += nc[i]
        mats[i, :m.size] = m.reshape(-1)
    return nt, tb, nc, cb, mats.view(np.float64).reshape(-1), kc


def pack_specs(specs, n):
    """pack_gate_batch straight from GateSpecs (qubit q -> bit n-1-q, kernel class AUTO)."""
    k = len(specs)
    nt = np.zeros(k, dtype=np.int32)
    tb = np.zeros(2 * k, dtype=np.int32)
    nc = np.zeros(k, dtype=np.int32)
    cbits = []
    mats = np.zeros((k, 16), dtype=np.complex128)
    for i, spec in enumerate(specs):
        m = gate_matrix(spec)
        t = len(spec.targets)
        if t > 2 or m.shape != (1 << t, 1 << t):
            raise ShapeError(f"gate {i} ({spec.targets}) is not a 1- or 2-target gate")
        nt[i] = t
        tb[2 * i:2 * i + t] = [n - 1 - int(x) for x in spec.targets]
        nc[i] = len(spec.controls)
        cbits.extend(n - 1 - int(x) for x in spec.controls)
        mats[i, :m.size] = m.reshape(-1)
    cb = np.array(cbits or [0], dtype=np.int32)
    kc = np.full(k, nat.KERNEL_AUTO, dtype=np.int32)
    return nt, tb, nc, cb, mats.view(np.float64).reshape(-1), kc


def _apply_gate_batch(ptr, n, dtype, packed, stream):
    nt, tb, nc, cb, mats, kc = packed
    nat.check(nat.lib().qsb_apply_batch(ptr, n, dtype, len(nt), nt.ctypes.data, tb.ctypes.data, nc.ctypes.data,
                                        cb.ctypes.data, mats.ctypes.data, kc.ctypes.data, stream),
              "apply_batch")


def _batchable(state) -> bool:
    return state.n_amps * state.precision.itemsize <= BATCH_MAX_STATE_BYTES


def _launch_pass(step, words, dtype, src, dst, n, st):
    """Specialised (NVRTC) kernel when available, else the interpreting pass kernel."""
    if not step.no_jit and jit.available():
        try:
            if step.jit is None:
                step.jit = jit.compile_words(words, dtype)
            compiled, coeffs = step.jit
            jit.run(words, dtype, src, dst, n, st, compiled, coeffs, step.dev_tables)
            return
        except Exception as exc:  # compile / TMA-plan failure: keep going on the interpreter
            step.no_jit = True
            warnings.warn(f"pass specialisation unavailable ({exc}); using the interpreted pass kernel")
    if int(words[3]) != GEOMETRY[dtype].nreg:
        # planned for the specialised kernel's register geometry: re-encode for the interpreter
        if getattr(step, "interp_words", None) is None:
            step.interp_words, _ = compile_pass(step.gates, set(step.tile_pos), n, dtype, GEOMETRY[dtype])
        words = step.interp_words
    nat.check(nat.lib().qsb_run_pass(src, dst, n, dtype, words.ctypes.data, len(words), st), "run_pass")


def own_device_tables(plan: Plan) -> None:
    """Give every pass of `plan` its own device copy of its pivot tables, so its launches read
    nothing staged from the host at launch time (required before CUDA-graph capture: a captured
    upload out of the library's shared host ring would replay whatever later launches left in
    that slot).  Raises when a pass cannot run as a specialised kernel (the interpreter stages
    its whole program per launch)."""
    torch = nat.torch_mod()
    for step in plan.steps:
        if not isinstance(step, PassStep):
            continue
        if step.jit is None and not step.no_jit and jit.available():
            step.jit = jit.compile_words(step.words, plan.dtype)
        if step.jit is None:
            raise SimulationError("CUDA-graph capture needs the specialised (NVRTC) pass kernels")
        tables = step.jit[1][1]
        if len(tables) and step.dev_tables is None:
            step.dev_tables = torch.from_numpy(np.ascontiguousarray(tables)).to("cuda")


def run_plan(state, plan: Plan, scratch_holder: dict | None = None, stream=None, events: list | None = None):
    """Execute every step of `plan` on `state` (in place; the tensor object may be swapped).

    `events`, when given, receives one (start, end) pair of CUDA events per pass launch,
    recorded on the launching stream (bench.py's per-kernel timing)."""
    st = nat.stream_ptr(stream)
    n = state.n_qubits
    dtype = state.precision.qsb_dtype
    holder = scratch_holder if scratch_holder is not None else {}
    jit.precompile([s for s in plan.steps if isinstance(s, PassStep)], dtype)
    batch = _batchable(state) and events is None
    packed = plan.__dict__.setdefault("_packed_runs", {}) if batch else None
    i = 0
    while i < len(plan.steps):
        step = plan.steps[i]
        if isinstance(step, GateStep):
            j = i + 1
            while batch and j < len(plan.steps) and isinstance(plan.steps[j], GateStep):
                j += 1
            if j - i > 1:
                # a small state: the whole run of stand-alone gates is one shared-memory launch
                run = packed.get(i)
                if run is None:
                    run = packed[i] = pack_gate_batch([s.gate for s in plan.steps[i:j]])
                _apply_gate_batch(state.raw_ptr, n, dtype, run, st)
            else:
                _apply_gate_step(state.raw_ptr, n, dtype, step.gate, st)
            i = j
            continue
        i += 1
        words = step.words
        if events is not None:
            ev0 = nat.torch_mod().cuda.Event(enable_timing=True)
            ev1 = nat.torch_mod().cuda.Event(enable_timing=True)
            ev0.record(stream)
        src = state.raw_ptr
        if step.ext_perm:
            scratch = holder.get("buf")
            if scratch is None or scratch.numel() != state.n_amps or scratch.dtype != state.raw_tensor.dtype:
                scratch = nat.torch_mod().empty_like(state.raw_tensor)
            dst_t = scratch
        else:
            dst_t = None
        dst = dst_t.data_ptr() if dst_t is not None else src
        _launch_pass(step, words, dtype, src, dst, n, st)
        if dst_t is not None:
            old = state._t
            state._t = dst_t
            holder["buf"] = old
        if events is not None:
            ev1.record(stream)
            events.append((ev0, ev1))


def _plan_key(n_qubits, dtype, fuse_, allow_ext, specs):
    return (n_qubits, dtype, fuse_, allow_ext, jit.available(), tuple(id(s) for s in specs))


def prepare_plan(n_qubits, precision, specs, fuse: bool | None = None, plan_cache: dict | None = None,
                 allow_ext: bool | None = None) -> Plan:
    """The plan run_gates will use for `specs` (from `plan_cache` when present), with its passes'
    specialised kernels compiled.  `allow_ext=None`: decided from the free device memory, as
    for an already allocated state of this size."""
    fuse_ = FUSION_DEFAULT if fuse is None else fuse
    dtype = precision.qsb_dtype
    if allow_ext is None:
        allow_ext = scratch_fits((1 << n_qubits) * precision.itemsize)
    key = _plan_key(n_qubits, dtype, fuse_, allow_ext, specs)
    hit = plan_cache.get(key) if plan_cache is not None else None
    if hit is not None:
        return hit[0]
    plan = plan_circuit(list(specs), n_qubits, dtype, allow_ext_perm=allow_ext, fuse=fuse_,
                        geometry=default_geometry(dtype))
    steps = [s for s in plan.steps if isinstance(s, PassStep)]
    jit.precompile(steps, dtype)
    for s in steps:  # precompile leaves single passes to the caller
        if s.jit is None and not s.no_jit and jit.available():
            try:
                s.jit = jit.compile_words(s.words, dtype)
            except Exception:  # run_plan retries and falls back to the interpreter with a warning
                pass
    if plan_cache is not None:
        if len(plan_cache) >= 8:
            plan_cache.clear()
        plan_cache[key] = (plan, list(specs))  # the specs are kept alive so their ids stay unique
    return plan


class _Relabelled:
    """A gate spec acting on other qubits (same kind, parameters and matrix)."""

    __slots__ = ("kind", "targets", "controls", "params", "matrix")

    def __init__(self, spec, targets, controls):
        self.kind = spec.kind
        self.targets = targets
        self.controls = controls
        self.params = getattr(spec, "params", ())
        self.matrix = getattr(spec, "matrix", None)


def relabel_specs(specs, layout, n_qubits):
    """Gates mapped through a logical -> physical qubit map, uncontrolled SWAPs absorbed into
    the map (no data moves).  Returns (mapped specs, final layout or None if canonical)."""
    from .gates import GateKind

    phys = list(layout) if layout is not None else list(range(n_qubits))
    out = []
    for spec in specs:
        kind = spec.kind if isinstance(spec.kind, GateKind) else GateKind(getattr(spec.kind, "value", spec.kind))
        if kind is GateKind.SWAP and not spec.controls:
            a, b = spec.targets
            phys[a], phys[b] = phys[b], phys[a]
            continue
        out.append(_Relabelled(spec, tuple(phys[q] for q in spec.targets), tuple(phys[q] for q in spec.controls)))
    final = None if phys == list(range(n_qubits)) else tuple(phys)
    return out, final


def _has_free_swap(specs) -> bool:
    from .gates import GateKind

    for spec in specs:
        k = spec.kind
        if (k is GateKind.SWAP or getattr(k, "value", k) == "SWAP") and not spec.controls:
            return True
    return False


def run_gates(state, specs, fuse: bool | None = None, scratch_holder: dict | None = None,
              plan_cache: dict | None = None):
    """Run `specs` on `state`.

    * Small states (<= BATCH_MAX_STATE_BYTES): no planning; the specs go straight to one
      shared-memory launch per 64 gates.
    * Mid-size states (<= GRID_BATCH_MAX_STATE_BYTES, fusion on): the first run of a
      gate list goes through the grid-synchronised batch launch (no host planning, which costs
      more than the whole circuit at this size); when the same list comes back -- or was
      prepared with prepare_plan -- it runs as planned fused passes.
    * Larger states: planned fused passes.
    With `plan_cache` (a Circuit's), packed lists and plans -- with the specialised kernels and
    coefficients attached to their passes -- are reused while the gate objects, precision,
    fusion switch and scratch availability are unchanged."""
    fuse_ = FUSION_DEFAULT if fuse is None else fuse
    n, precision = state.n_qubits, state.precision
    nbytes = state.n_amps * precision.itemsize
    if getattr(state, "layout", None) is not None or (fuse_ and _has_free_swap(specs) and hasattr(state, "layout")
                                                      and nbytes > GRID_BATCH_MAX_STATE_BYTES and not scratch_fits(nbytes)):
        # no room for an out-of-place pass (e.g. 33 qubits c128 = 137 GB): SWAPs become qubit
        # relabels instead of in-place half sweeps; the state keeps the map until a canonical read
        key = ("relabel", state.layout, tuple(id(s) for s in specs))
        hit = plan_cache.get(key) if plan_cache is not None else None
        if hit is None:
            hit = relabel_specs(specs, state.layout, n) + (list(specs),)
            if plan_cache is not None:
                plan_cache[key] = hit
        mapped, final, _keep = hit
        plan = prepare_plan(n, precision, mapped, fuse_, plan_cache)
        run_plan(state, plan, scratch_holder)
        state._layout = final
        return plan
    small = nbytes <= BATCH_MAX_STATE_BYTES
    if small or (fuse_ and FIRST_RUN_BATCH and nbytes <= GRID_BATCH_MAX_STATE_BYTES):
        planned = (not small and plan_cache is not None
                   and _plan_key(n, precision.qsb_dtype, fuse_, scratch_fits(nbytes), specs) in plan_cache)
        if not planned:
            bkey = ("batch", n, precision.qsb_dtype, tuple(id(s) for s in specs))
            entry = plan_cache.get(bkey) if plan_cache is not None else None
            if entry is None:
                entry = [pack_specs(specs, n), list(specs), 0]
                if plan_cache is not None:
                    if len(plan_cache) >= 8:
                        plan_cache.clear()
                    plan_cache[bkey] = entry
            if small or entry[2] == 0:
                entry[2] += 1
                if len(entry[0][0]):
                    _apply_gate_batch(state.raw_ptr, n, precision.qsb_dtype, entry[0], nat.stream_ptr())
                return None
    plan = prepare_plan(n, precision, specs, fuse_, plan_cache)
    run_plan(state, plan, scratch_holder)
    return plan
