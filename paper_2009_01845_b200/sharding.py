"""Sharded execution over global qubits (drop-in for /root/reference/pkg/src/qsim/sharding.py).

A state of n qubits with g global qubits is 2^g shards of 2^(n-g) amplitudes; shard s holds
the amplitudes whose global-qubit bits spell s (global_qubits[0] = MSB of s), local qubits in
significance order inside a shard -- sharding.py:30-81.

Two placements share one runner:
  * in-process (LocalComm): every shard is a separate HBM buffer of this GPU -- the reference's
    logical devices (SPEC "workers"), used for n_shards > GPUs and for single-GPU parity runs;
  * distributed (TorchComm): one shard per rank (one process per GPU), global<->local
    exchanges as NCCL send/recv pairs over NVLink, chunked through bounded staging buffers.

The schedule is the reference's: plan() picks the global qubits and Belady reshuffles with the
same locality rules (sharding.py:141-216), so reshuffle counts match the reference exactly.
Inside a LocalSegment every shard runs its own localised gate list through the fused pass
engine (global controls become shard filters, diagonal gates on global qubits become local
diagonals or a whole-shard phase, SWAPs with global qubits become half-shard exchanges or shard
relabels -- sharding.py:219-320).
"""

from __future__ import annotations

import bisect
import math
import os
from dataclasses import dataclass, field

import numpy as np

from . import _native as nat
from .circuit import Circuit
from .errors import CapacityError, ShapeError, SimulationError
from .fusion import NGate, diag_terms, normalize, plan_circuit
from .gates import GateKind, gate_matrix
from .state import Precision, StateVector, _check_cap, zero_state


# ------------------------------------------------------------------------------------------
# plan (reference semantics)
# ------------------------------------------------------------------------------------------
@dataclass
class LocalSegment:
    """Queue positions executable without moving any qubit."""

    positions: list


@dataclass
class Reshuffle:
    """Exchange one global qubit with one local qubit."""

    global_qubit: int
    local_qubit: int


@dataclass
class ExecutionPlan:
    n_qubits: int
    n_shards: int
    global_qubits: tuple
    steps: list = field(default_factory=list)
    # uncontrolled SWAPs are label swaps (plan_batched); the reference plan moves their data
    relabel_swaps: bool = False

    @property
    def n_reshuffles(self) -> int:
        return sum(1 for s in self.steps if isinstance(s, Reshuffle))

    @property
    def n_exchanges(self) -> int:
        """Data-moving steps: reshuffles plus batched exchanges."""
        return sum(1 for s in self.steps if isinstance(s, (Reshuffle, Exchange)))

    @property
    def swapped_qubits(self) -> int:
        return sum(1 if isinstance(s, Reshuffle) else s.k for s in self.steps if isinstance(s, (Reshuffle, Exchange)))

    def shard_fraction_moved(self) -> float:
        """Fraction of one shard every rank sends over the whole plan."""
        return sum(0.5 if isinstance(s, Reshuffle) else 1.0 - 2.0 ** -s.k
                   for s in self.steps if isinstance(s, (Reshuffle, Exchange)))


def _kind(spec):
    k = spec.kind
    return k if isinstance(k, GateKind) else GateKind(getattr(k, "value", k))


def _required_local(spec) -> tuple:
    """Targets that must be local (sharding.py:141-149)."""
    kind = _kind(spec)
    if kind in (GateKind.CZ, GateKind.CZPOW):
        return ()
    if kind is GateKind.SWAP and not spec.controls:
        return ()
    if kind is GateKind.CNOT:
        return (spec.targets[1],)
    return tuple(spec.targets)


def plan(circuit: Circuit, n_shards: int, global_qubits=None) -> ExecutionPlan:
    """Global qubits = the g least-required qubits (ties to the higher index); Belady victims
    for reshuffles (sharding.py:152-216)."""
    n = circuit.n_qubits
    if n_shards < 2 or n_shards & (n_shards - 1):
        raise ShapeError(f"n_shards must be a power of two >= 2, got {n_shards}")
    if n_shards > 1 << (n - 1):
        raise CapacityError(f"{n_shards} shards exceed the cap of {1 << (n - 1)} for {n} qubits")
    g = n_shards.bit_length() - 1
    need = [_required_local(s) for s in circuit.queue]
    if global_qubits is None:
        count = [0] * n
        for req in need:
            for q in req:
                count[q] += 1
        order = sorted(range(n), key=lambda q: (count[q], -q))
        global_qubits = tuple(sorted(order[:g]))
    else:
        global_qubits = tuple(global_qubits)
        if len(global_qubits) != g or len(set(global_qubits)) != g:
            raise ShapeError(f"{n_shards} shards need {g} distinct global qubits, got {global_qubits}")
    uses = [[] for _ in range(n)]
    for pos, req in enumerate(need):
        for q in req:
            uses[q].append(pos)

    def next_use(q, pos):
        i = bisect.bisect_left(uses[q], pos)
        return uses[q][i] if i < len(uses[q]) else math.inf

    glob = set(global_qubits)
    steps, seg = [], []
    for pos, req in enumerate(need):
        blocked = [q for q in req if q in glob]
        if blocked:
            if len(req) > n - g:
                raise CapacityError(
                    f"gate at position {pos} needs {len(req)} local qubits but only {n - g} exist with {n_shards} shards"
                )
            if seg:
                steps.append(LocalSegment(seg))
                seg = []
            for q in blocked:
                cands = [c for c in range(n) if c not in glob and c not in req]
                victim = max(cands, key=lambda c: (next_use(c, pos), c))
                steps.append(Reshuffle(q, victim))
                glob.remove(q)
                glob.add(victim)
        seg.append(pos)
    if seg:
        steps.append(LocalSegment(seg))
    return ExecutionPlan(n, n_shards, global_qubits, steps)


@dataclass
class Exchange:
    """Swap k global qubits with k local qubits in one all-to-all (pairs: (global, local));
    the batched form of k Reshuffles: (1 - 2^-k) of every shard moves once instead of half a
    shard k times."""

    pairs: tuple

    @property
    def k(self) -> int:
        return len(self.pairs)


def _is_free_swap(spec) -> bool:
    return _kind(spec) is GateKind.SWAP and not spec.controls


def _required_local_batched(spec) -> tuple:
    """Targets that must be local when global controls are shard filters, every diagonal gate
    is applied shard-locally (any kind, not only CZ/CZPow) and uncontrolled SWAPs are label
    swaps."""
    kind = _kind(spec)
    if kind in (GateKind.CZ, GateKind.CZPOW, GateKind.Z, GateKind.RZ) or _is_free_swap(spec):
        return ()
    if kind is GateKind.CNOT:
        return (spec.targets[1],)
    m = gate_matrix(spec)
    if not np.count_nonzero(m - np.diag(np.diagonal(m))):
        return ()
    return tuple(spec.targets)


def _diag_qubits(spec) -> set:
    """Qubits on which the gate acts diagonally (controls; every target of a diagonal gate):
    two gates commute when every qubit they share is diagonal for both."""
    kind = _kind(spec)
    ctrl = set(spec.controls)
    if kind in (GateKind.CZ, GateKind.CZPOW, GateKind.Z, GateKind.RZ):
        return ctrl | set(spec.targets)
    if kind is GateKind.SWAP:
        return ctrl
    m = gate_matrix(spec)
    if not np.count_nonzero(m - np.diag(np.diagonal(m))):
        return ctrl | set(spec.targets)
    if kind is GateKind.CNOT:
        return ctrl | {spec.targets[0]}
    return ctrl


def _gate_dag(queue):
    """Predecessor lists of the commutation DAG: gate j waits for gate i < j when they share a
    qubit on which at least one of them is not diagonal."""
    preds = [set() for _ in queue]
    last_nd: dict = {}  # qubit -> last gate non-diagonal on it
    diag_since: dict = {}  # qubit -> gates diagonal on it since then
    for j, spec in enumerate(queue):
        dq = _diag_qubits(spec)
        for q in set(spec.targets) | set(spec.controls):
            if q in last_nd:
                preds[j].add(last_nd[q])
            if q in dq:
                diag_since.setdefault(q, []).append(j)
            else:
                preds[j].update(diag_since.pop(q, ()))
                last_nd[q] = j
        preds[j].discard(j)
    return preds


def plan_batched(circuit: Circuit, n_shards: int, global_qubits=None, local_order=None) -> ExecutionPlan:
    """Exchange-minimising schedule for the resident multi-GPU path.

    Locality rules of plan() (sharding.py:141-149) widened to every diagonal gate, with
    uncontrolled SWAPs as free relabels.  Gates run in any order their commutation DAG allows
    (disjoint supports, or shared qubits that both act on diagonally): every gate whose
    qubits are local runs as soon as its predecessors have.  When only blocked gates remain,
    ONE exchange installs a new global set: the g qubits (outside the blocked gate's targets)
    whose first use lies deepest in the remaining DAG -- Belady on sets over DAG depth, which
    maximises how much runs before the next exchange -- keeping every current global whose
    first use is at or past that horizon, so k is as small as the horizon allows.  Among equal
    candidates, locals at higher bit positions enter (long contiguous runs for pack/unpack).
    `local_order`: the current local qubits in slot order (defaults to significance order)."""
    import heapq

    n = circuit.n_qubits
    if n_shards < 2 or n_shards & (n_shards - 1):
        raise ShapeError(f"n_shards must be a power of two >= 2, got {n_shards}")
    if n_shards > 1 << (n - 1):
        raise CapacityError(f"{n_shards} shards exceed the cap of {1 << (n - 1)} for {n} qubits")
    g = n_shards.bit_length() - 1
    queue = circuit.queue
    need = [_required_local_batched(s) for s in queue]
    for pos, req in enumerate(need):
        if len(req) > n - g:
            raise CapacityError(
                f"gate at position {pos} needs {len(req)} local qubits but only {n - g} exist with {n_shards} shards")
    if global_qubits is None:
        count = [0] * n
        for req in need:
            for q in req:
                count[q] += 1
        order = sorted(range(n), key=lambda q: (count[q], -q))
        global_qubits = tuple(sorted(order[:g]))
    else:
        global_qubits = tuple(global_qubits)
        if len(global_qubits) != g or len(set(global_qubits)) != g:
            raise ShapeError(f"{n_shards} shards need {g} distinct global qubits, got {global_qubits}")
    preds = _gate_dag(queue)
    succ = [[] for _ in queue]
    for j, ps in enumerate(preds):
        for i in ps:
            succ[i].append(j)
    indeg = [len(ps) for ps in preds]
    done = [False] * len(queue)
    glob = list(global_qubits)
    loc = list(local_order) if local_order is not None else [q for q in range(n) if q not in global_qubits]
    ready = [j for j in range(len(queue)) if not indeg[j]]
    heapq.heapify(ready)
    blocked: list = []
    steps, seg = [], []
    remaining = len(queue)
    while remaining:
        gset = set(glob)
        progressed = False
        while ready:
            j = heapq.heappop(ready)
            if any(q in gset for q in need[j]):
                blocked.append(j)
                continue
            progressed = True
            done[j] = True
            remaining -= 1
            seg.append(j)
            if _is_free_swap(queue[j]):
                a, b = queue[j].targets
                for lst in (glob, loc):
                    for i, q in enumerate(lst):
                        if q == a:
                            lst[i] = b
                        elif q == b:
                            lst[i] = a
                gset = set(glob)
            for k in succ[j]:
                indeg[k] -= 1
                if not indeg[k]:
                    heapq.heappush(ready, k)
        if not remaining:
            break
        if progressed and blocked:
            # a relabel may have unblocked some of them
            for j in blocked:
                heapq.heappush(ready, j)
            blocked = []
            if any(not any(q in set(glob) for q in need[j]) for j in ready):
                continue
            blocked = [heapq.heappop(ready) for _ in range(len(ready))]
        # only blocked gates are ready: one exchange
        if seg:
            steps.append(LocalSegment(seg))
            seg = []
        first = min(blocked)
        rs = set(need[first])
        # depth of every remaining gate from the current frontier; first use of each qubit
        depth = {}
        nu = {q: math.inf for q in range(n)}
        for j in range(len(queue)):  # queue order is a topological order of the DAG
            if done[j]:
                continue
            d = 0
            for i in preds[j]:
                if not done[i]:
                    d = max(d, depth[i] + 1)
            depth[j] = d
            for q in need[j]:
                if d < nu[q]:
                    nu[q] = d
        cand = {q: nu[q] for q in range(n) if q not in rs}
        horizon = sorted(cand.values(), reverse=True)[g - 1]
        keep = [q for q in glob if q not in rs and cand[q] >= horizon]
        outs = [q for q in glob if q not in keep]
        pool = sorted((q for q in loc if q not in rs and cand[q] >= horizon), key=lambda q: (-cand[q], loc.index(q)))
        ins = pool[:len(outs)]
        for a, b in zip(outs, ins):
            ja, mb = glob.index(a), loc.index(b)
            glob[ja], loc[mb] = b, a
        steps.append(Exchange(tuple(zip(outs, ins))))
        for j in blocked:
            heapq.heappush(ready, j)
        blocked = []
    if seg:
        steps.append(LocalSegment(seg))
    return ExecutionPlan(n, n_shards, global_qubits, steps, relabel_swaps=True)


# ------------------------------------------------------------------------------------------
# device backend (the product path) -- tests inject a CPU stand-in with the same methods
# ------------------------------------------------------------------------------------------
class CudaBackend:
    def __init__(self, precision: Precision):
        self.precision = precision
        self.dtype = precision.qsb_dtype

    def empty(self, n_amps):
        torch = nat.torch_mod()
        return torch.empty(n_amps, dtype=self.precision.torch_dtype, device=torch.device("cuda", torch.cuda.current_device()))

    def zeros(self, n_amps):
        t = self.empty(n_amps)
        t.zero_()
        return t

    def run_local(self, shard, n_local, ngates, cache):
        from . import engine

        if not ngates:
            return shard
        if (engine.FIRST_RUN_BATCH and engine.FUSION_DEFAULT
                and shard.numel() * shard.element_size() <= engine.GRID_BATCH_MAX_STATE_BYTES):
            # small shards: one batched launch per 64 gates, no planning or kernel specialisation
            # (every step of an evolution brings new coefficients and often new layouts)
            engine._apply_gate_batch(shard.data_ptr(), n_local, self.dtype, engine.pack_gate_batch(ngates),
                                     nat.stream_ptr())
            return shard
        # out-of-place passes (folded SWAPs) need one more shard-sized buffer
        allow_ext = engine.scratch_fits(shard.numel() * shard.element_size())
        fuse = engine.FUSION_DEFAULT
        key = (allow_ext, fuse) + tuple((g.kind, g.targets, g.controls, g.index,
                                          None if g.matrix is None else g.matrix.tobytes()) for g in ngates)
        plan_ = cache.get(key)
        if plan_ is None:
            plan_ = plan_circuit(ngates, n_local, self.dtype, allow_ext_perm=allow_ext, fuse=fuse,
                                 geometry=engine.default_geometry(self.dtype))
            cache[key] = plan_
        holder = {}
        view = _ShardView(shard, n_local, self.precision)
        engine.run_plan(view, plan_, holder)
        if _STATS is not None:
            _STATS["local_bytes"] += int(plan_.state_sweeps() * 2 * shard.numel() * shard.element_size())
        return view._t

    def scale(self, shard, phase):
        nat.check(nat.lib().qsb_scale(shard.data_ptr(), shard.numel(), self.dtype, phase.real, phase.imag,
                                      nat.stream_ptr()), "shard phase")

    def exchange_local(self, a, b, n_local, bit):
        nat.check(nat.lib().qsb_exchange_halves(a.data_ptr(), b.data_ptr(), n_local, self.dtype, bit,
                                                nat.stream_ptr()), "exchange_halves")

    def pack(self, shard, n_local, bit, half, first, count, staging):
        nat.check(nat.lib().qsb_pack_half(shard.data_ptr(), n_local, self.dtype, bit, half, first, count,
                                          staging.data_ptr(), nat.stream_ptr()), "pack_half")

    def unpack(self, shard, n_local, bit, half, first, count, staging):
        nat.check(nat.lib().qsb_unpack_half(shard.data_ptr(), n_local, self.dtype, bit, half, first, count,
                                            staging.data_ptr(), nat.stream_ptr()), "unpack_half")

    def exchange_parts(self, a, b, n_local, bits, a_bits, b_bits):
        pb = np.ascontiguousarray(bits, dtype=np.int32)
        nat.check(nat.lib().qsb_exchange_parts(a.data_ptr(), b.data_ptr(), n_local, self.dtype, len(bits), pb.ctypes.data,
                                               a_bits, b_bits, nat.stream_ptr()), "exchange_parts")

    def pack_part(self, shard, n_local, bits, part_bits, first, count, staging):
        pb = np.ascontiguousarray(bits, dtype=np.int32)
        nat.check(nat.lib().qsb_pack_part(shard.data_ptr(), n_local, self.dtype, len(bits), pb.ctypes.data, part_bits,
                                          first, count, staging.data_ptr(), nat.stream_ptr()), "pack_part")

    def unpack_part(self, shard, n_local, bits, part_bits, first, count, staging):
        pb = np.ascontiguousarray(bits, dtype=np.int32)
        nat.check(nat.lib().qsb_unpack_part(shard.data_ptr(), n_local, self.dtype, len(bits), pb.ctypes.data, part_bits,
                                            first, count, staging.data_ptr(), nat.stream_ptr()), "unpack_part")

    def permute(self, src, n_bits, dst_bit):
        out = self.empty(src.numel())
        perm = np.ascontiguousarray(dst_bit, dtype=np.int32)
        nat.check(nat.lib().qsb_permute_qubits(src.data_ptr(), out.data_ptr(), n_bits, self.dtype, perm.ctypes.data,
                                               nat.stream_ptr()), "permute_qubits")
        return out


class _ShardView:
    """Minimal StateVector-like wrapper so the fused engine runs on one shard buffer."""

    def __init__(self, t, n, precision):
        self._t = t
        self.n_qubits = n
        self.precision = precision

    @property
    def tensor(self):
        return self._t

    @property
    def data_ptr(self):
        return int(self._t.data_ptr())

    raw_ptr = data_ptr

    @property
    def raw_tensor(self):
        return self._t

    @property
    def n_amps(self):
        return 1 << self.n_qubits


# ------------------------------------------------------------------------------------------
# communicators
# ------------------------------------------------------------------------------------------
class LocalComm:
    """Every shard lives in this process."""

    rank = 0
    world = 1

    def owns(self, shard_id, owner):
        return True


class TorchComm:
    """One shard per rank over torch.distributed (NCCL on GPUs; gloo in the CPU tests)."""

    CHUNK_BYTES = int(os.environ.get("QSB_EXCHANGE_CHUNK_BYTES", str(1 << 30)))

    def __init__(self, group=None):
        import torch.distributed as dist

        self.dist = dist
        self.group = group
        self.rank = dist.get_rank(group)
        self.world = dist.get_world_size(group)
        # NCCL orders its transfers after the current stream's pending kernels (and wait() orders
        # the stream after the transfer); other backends need a host sync after packing
        try:
            self.stream_ordered = dist.get_backend(group) == "nccl"
        except Exception:
            self.stream_ordered = False

    def owns(self, shard_id, owner):
        return owner[shard_id] == self.rank

    def sendrecv(self, send, recv, peer):
        for req in self.isendrecv(send, recv, peer):
            req.wait()

    def isendrecv(self, send, recv, peer):
        """Start a paired send/recv; returns the works (NCCL: wait() orders the current CUDA stream
        after the transfer without blocking the host; gloo: wait() blocks)."""
        dist = self.dist
        ops = [dist.P2POp(dist.isend, send, peer, self.group), dist.P2POp(dist.irecv, recv, peer, self.group)]
        return dist.batch_isend_irecv(ops)

    def ialltoall(self, triples):
        """Start paired sends/receives with several peers as one group ((send, recv, peer) per
        peer); NCCL runs the group as an all-to-all among those ranks."""
        dist = self.dist
        ops = []
        for send, recv, peer in triples:
            ops.append(dist.P2POp(dist.isend, send, peer, self.group))
            ops.append(dist.P2POp(dist.irecv, recv, peer, self.group))
        return dist.batch_isend_irecv(ops)

    def all_gather(self, t):
        out = [t.new_empty(t.shape) for _ in range(self.world)]
        self.dist.all_gather(out, t, group=self.group)
        return out

    def barrier(self):
        self.dist.barrier(group=self.group)


class HostStagedComm(TorchComm):
    """TorchComm over a backend that cannot move CUDA tensors (gloo): every transfer is staged
    through host memory.  A validation transport only (several ranks sharing one GPU, where
    NCCL refuses to run); the compute stays on the device and the exchange pipeline is the same
    code as under NCCL, with host synchronisation instead of stream ordering."""

    stream_ordered = False

    def isendrecv(self, send, recv, peer):
        return self.ialltoall([(send, recv, peer)])

    def ialltoall(self, triples):
        torch = nat.torch_mod()
        staged = [(send.cpu(), torch.empty(send.shape, dtype=send.dtype), recv, peer) for send, recv, peer in triples]
        for w in super().ialltoall([(hs, hr, peer) for hs, hr, _, peer in staged]):
            w.wait()
        for _, hr, recv, _ in staged:
            recv.copy_(hr)
        return []

    def all_gather(self, t):
        return [x.to(t.device) for x in super().all_gather(t.cpu())]

    def barrier(self):
        self.dist.barrier(group=self.group)


# ------------------------------------------------------------------------------------------
# sharded state
# ------------------------------------------------------------------------------------------
@dataclass
class ShardedState:
    """2^g shards addressed by the global-qubit bits (sharding.py:30-50).

    `shards` maps logical shard id -> buffer for the shards this process holds; `owner` maps
    every logical shard id to the rank holding it (relabels only permute this map)."""

    n_qubits: int
    global_qubits: tuple
    shards: dict
    precision: Precision = Precision.F64
    local_qubits: tuple = ()
    owner: list = field(default_factory=list)
    comm: object = None
    backend: object = None

    def __post_init__(self):
        if not self.local_qubits:
            taken = set(self.global_qubits)
            self.local_qubits = tuple(q for q in range(self.n_qubits) if q not in taken)
        if not self.owner:
            self.owner = [0] * (1 << len(self.global_qubits))
        if self.comm is None:
            self.comm = LocalComm()
        if self.backend is None:
            self.backend = CudaBackend(self.precision)

    @property
    def n_global(self):
        return len(self.global_qubits)

    @property
    def n_local(self):
        return self.n_qubits - self.n_global

    def local_bit(self, q):
        return self.n_local - 1 - self.local_qubits.index(q)

    def shard_bit(self, q):
        return self.n_global - 1 - self.global_qubits.index(q)


def _stacked_to_canonical(n, global_qubits, local_qubits):
    """dst bit (canonical, qubit q at n-1-q) of every bit of the stacked (shard, local) index."""
    g = len(global_qubits)
    nl = n - g
    dst = [0] * n
    for j, q in enumerate(global_qubits):
        dst[n - 1 - j] = n - 1 - q
    for m, q in enumerate(local_qubits):
        dst[nl - 1 - m] = n - 1 - q
    return dst


def partition(state: StateVector, global_qubits, comm=None, backend=None) -> ShardedState:
    """Copy a state into shards addressed by the global-qubit bits (sharding.py:53-71)."""
    global_qubits = tuple(global_qubits)
    g = len(global_qubits)
    n = state.n_qubits
    if not 1 <= g <= n - 1:
        raise ShapeError(f"need between 1 and {n - 1} global qubits, got {g}")
    if len(set(global_qubits)) != g:
        raise ShapeError(f"duplicate global qubits {global_qubits}")
    for q in global_qubits:
        if not 0 <= q < n:
            raise ShapeError(f"qubit {q} out of range for {n} qubits")
    backend = backend or CudaBackend(state.precision)
    comm = comm or LocalComm()
    sh = ShardedState(n, global_qubits, {}, state.precision, comm=comm, backend=backend)
    fwd = _stacked_to_canonical(n, global_qubits, sh.local_qubits)
    inv = [0] * n
    for b, d in enumerate(fwd):
        inv[d] = b
    stacked = backend.permute(state.tensor, n, inv)
    nl = n - g
    world = comm.world
    for s in range(1 << g):
        sh.owner[s] = (s * world) >> g
        if comm.owns(s, sh.owner):
            sh.shards[s] = stacked[s << nl:(s + 1) << nl].clone()
    return sh


def gather(sharded: ShardedState) -> StateVector:
    """Reassemble the canonical state (sharding.py:74-81); distributed: on every rank."""
    return StateVector(sharded.n_qubits, gather_tensor(sharded), sharded.precision)


def gather_tensor(sharded: ShardedState):
    """Canonical-order amplitudes of a sharded state as one buffer (on every rank)."""
    n, g = sharded.n_qubits, sharded.n_global
    nl = n - g
    backend = sharded.backend
    comm = sharded.comm
    if isinstance(comm, LocalComm):
        parts = [sharded.shards[s] for s in range(1 << g)]
    else:
        mine = [s for s in sharded.shards]
        if len(mine) != 1:
            raise SimulationError("distributed gather expects one shard per rank")
        got = comm.all_gather(sharded.shards[mine[0]])
        by_rank = {r: t for r, t in enumerate(got)}
        parts = [by_rank[sharded.owner[s]] for s in range(1 << g)]
    torch = nat.torch_mod()
    stacked = torch.cat(parts)
    _ = nl
    return backend.permute(stacked, n, _stacked_to_canonical(n, sharded.global_qubits, sharded.local_qubits))


def _exchange(sharded: ShardedState, j_bit, p_bit):
    """Pairwise half exchange (sharding.py:100-111): shard s (jbit clear) trades its p=1 half
    for shard s|jbit's p=0 half."""
    g, nl = sharded.n_global, sharded.n_local
    backend, comm = sharded.backend, sharded.comm
    jmask = 1 << j_bit
    if isinstance(comm, LocalComm):
        for s in range(1 << g):
            if not s & jmask:
                backend.exchange_local(sharded.shards[s], sharded.shards[s | jmask], nl, p_bit)
        return
    half = 1 << (nl - 1)
    itemsize = sharded.precision.itemsize
    chunk = max(1, min(half, comm.CHUNK_BYTES // itemsize))
    for s, buf in list(sharded.shards.items()):
        partner_shard = s ^ jmask
        peer = sharded.owner[partner_shard]
        my_half = 1 if not s & jmask else 0
        # double-buffered pipeline: pack chunk k+1 and unpack chunk k-1 while chunk k is on the
        # wire; every wait() orders the stream (NCCL) before a staging buffer is reused
        send = [backend.empty(chunk), backend.empty(chunk)]
        recv = [backend.empty(chunk), backend.empty(chunk)]
        inflight = [None, None]

        def drain(b):
            works, first, cnt = inflight[b]
            for w in works:
                w.wait()
            backend.unpack(buf, nl, p_bit, my_half, first, cnt, recv[b])
            inflight[b] = None

        for k, first in enumerate(range(0, half, chunk)):
            b = k & 1
            if inflight[b] is not None:
                drain(b)
            cnt = min(chunk, half - first)
            backend.pack(buf, nl, p_bit, my_half, first, cnt, send[b])
            if not comm.stream_ordered:
                _sync_stream()
            inflight[b] = (comm.isendrecv(send[b][:cnt], recv[b][:cnt], peer), first, cnt)
        for b in (0, 1):
            if inflight[b] is not None:
                drain(b)


def _sync_stream():
    torch = nat.torch_mod()
    if torch.cuda.is_available():
        torch.cuda.current_stream().synchronize()


def reshuffle(sharded: ShardedState, global_qubit: int, local_qubit: int):
    """Swap the roles of a global and a local qubit in place (sharding.py:84-97)."""
    gl = list(sharded.global_qubits)
    lc = list(sharded.local_qubits)
    j = gl.index(global_qubit)
    m = lc.index(local_qubit)
    _exchange(sharded, sharded.n_global - 1 - j, sharded.n_local - 1 - m)
    gl[j], lc[m] = local_qubit, global_qubit
    sharded.global_qubits = tuple(gl)
    sharded.local_qubits = tuple(lc)


# Optional per-run counters for the CLI's metric fields (collect_stats): exchange count, bytes
# each rank sent, CUDA events around every exchange, local HBM bytes of the per-shard passes.
_STATS = None


def collect_stats(enable: bool | None = True):
    """Start (or with None, stop) collecting exchange / pass statistics; returns the dict."""
    global _STATS
    _STATS = {"exchanges": 0, "exchange_bytes": 0, "events": [], "local_bytes": 0} if enable else None
    return _STATS


def finish_stats(stats: dict) -> dict:
    """Resolve the CUDA events of a finished run into seconds (call after a synchronize)."""
    ev = stats.pop("events", [])
    stats["exchange_seconds"] = sum(a.elapsed_time(b) for a, b in ev) / 1e3
    return stats


def _part_bits(value, bits):
    """Local index pattern with bit i of `value` at local bit bits[i]."""
    out = 0
    for i, b in enumerate(bits):
        out |= ((value >> i) & 1) << b
    return out


def exchange(sharded: ShardedState, pairs) -> None:
    """Swap the roles of k global and k local qubits in place with ONE all-to-all (pairs:
    (global, local)); equal to k reshuffles (sharding.py:84-111) up to the order of the qubits'
    slots.  Shard s with swapped-global bits sJ = a trades its part whose swapped-local bits
    spell u with the part spelling a of the shard whose swapped-global bits are u: every rank
    sends (1 - 2^-k) of its shard, to 2^k - 1 peers at once, and each part comes back into
    the slots it left (in place, chunked staging)."""
    pairs = tuple(pairs)
    if not pairs:
        return
    k = len(pairs)
    g, nl = sharded.n_global, sharded.n_local
    gl, lc = list(sharded.global_qubits), list(sharded.local_qubits)
    jbits = [sharded.shard_bit(a) for a, _ in pairs]
    pbits = [sharded.local_bit(b) for _, b in pairs]
    if len(set(jbits)) != k or len(set(pbits)) != k:
        raise ShapeError(f"exchange pairs {pairs} repeat a qubit")
    backend, comm = sharded.backend, sharded.comm
    stats = _STATS
    if stats is not None:
        torch = nat.torch_mod()
        ev = (torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
        ev[0].record()
        stats["exchanges"] += 1
        stats["exchange_bytes"] += int(((1 << nl) - (1 << (nl - k))) * sharded.precision.itemsize)
        stats["nvlink"] = bool(getattr(comm, "stream_ordered", False)) and not isinstance(comm, LocalComm)
        stats["ranks"] = comm.world

    def s_val(s):
        return sum(((s >> j) & 1) << i for i, j in enumerate(jbits))

    def with_val(s, v):
        for i, j in enumerate(jbits):
            s = (s & ~(1 << j)) | (((v >> i) & 1) << j)
        return s

    if isinstance(comm, LocalComm):
        for s in range(1 << g):
            a = s_val(s)
            for u in range(a + 1, 1 << k):
                t = with_val(s, u)
                backend.exchange_parts(sharded.shards[s], sharded.shards[t], nl, pbits,
                                       _part_bits(u, pbits), _part_bits(a, pbits))
    else:
        _exchange_parts_dist(sharded, k, pbits, s_val, with_val)
    if stats is not None:
        ev[1].record()
        stats["events"].append(ev)
    for (a, b), j, p in zip(pairs, jbits, pbits):
        gl[g - 1 - j] = b
        lc[nl - 1 - p] = a
    sharded.global_qubits = tuple(gl)
    sharded.local_qubits = tuple(lc)


def _exchange_parts_dist(sharded, k, pbits, s_val, with_val):
    """All-to-all among the 2^k ranks that share the other global bits: every chunk round
    packs one chunk of each outgoing part, posts all sends and receives as one batched group
    (NCCL: a grouped send/recv = all-to-all), and unpacks the previous round's chunks into the
    parts they came for (double-buffered; stream-ordered under NCCL)."""
    nl = sharded.n_local
    backend, comm = sharded.backend, sharded.comm
    part = 1 << (nl - k)
    itemsize = sharded.precision.itemsize
    for s, buf in list(sharded.shards.items()):
        a = s_val(s)
        peers = [(u, sharded.owner[with_val(s, u)]) for u in range(1 << k) if u != a]
        chunk = max(1, min(part, comm.CHUNK_BYTES // itemsize // len(peers)))
        send = [[backend.empty(chunk) for _ in peers] for _ in range(2)]
        recv = [[backend.empty(chunk) for _ in peers] for _ in range(2)]
        inflight = [None, None]

        def drain(bi):
            works, first, cnt = inflight[bi]
            for w in works:
                w.wait()
            for pi, (u, _) in enumerate(peers):
                backend.unpack_part(buf, nl, pbits, _part_bits(u, pbits), first, cnt, recv[bi][pi])
            inflight[bi] = None

        for c, first in enumerate(range(0, part, chunk)):
            bi = c & 1
            if inflight[bi] is not None:
                drain(bi)
            cnt = min(chunk, part - first)
            for pi, (u, _) in enumerate(peers):
                backend.pack_part(buf, nl, pbits, _part_bits(u, pbits), first, cnt, send[bi][pi])
            if not comm.stream_ordered:
                _sync_stream()
            works = comm.ialltoall([(send[bi][pi][:cnt], recv[bi][pi][:cnt], peer)
                                    for pi, (_, peer) in enumerate(peers)])
            inflight[bi] = (works, first, cnt)
        for bi in (0, 1):
            if inflight[bi] is not None:
                drain(bi)


# ------------------------------------------------------------------------------------------
# runner
# ------------------------------------------------------------------------------------------
class _Runner:
    def __init__(self, sharded: ShardedState, cache: dict | None = None, relabel_swaps: bool = False):
        self.sh = sharded
        self.pending = {s: [] for s in sharded.shards}
        self.cache: dict = {} if cache is None else cache
        self.relabel_swaps = relabel_swaps

    def _relabel(self, a, b):
        """Uncontrolled SWAP as a label swap: the data stays, the two qubits trade slots
        (queued gates are already in bit terms, so nothing is flushed)."""
        sh = self.sh

        def sw(t):
            return tuple(b if q == a else a if q == b else q for q in t)

        sh.global_qubits = sw(sh.global_qubits)
        sh.local_qubits = sw(sh.local_qubits)

    def flush(self):
        sh = self.sh
        for s, gates in self.pending.items():
            if gates:
                sh.shards[s] = sh.backend.run_local(sh.shards[s], sh.n_local, gates, self.cache)
                gates.clear()

    def _shard_value(self, s, q):
        return (s >> self.sh.shard_bit(q)) & 1

    def apply(self, spec, index):
        sh = self.sh
        kind = _kind(spec)
        targets, controls = tuple(spec.targets), tuple(spec.controls)
        glob = set(sh.global_qubits)
        if kind is GateKind.SWAP and not controls and self.relabel_swaps:
            self._relabel(*targets)
            return
        if kind is GateKind.SWAP and not controls and (set(targets) & glob):
            self.flush()
            self._swap(targets)
            return
        m = gate_matrix(spec)
        is_diag = not np.count_nonzero(m - np.diag(np.diagonal(m)))
        if kind is GateKind.CNOT and targets[0] in glob:
            # first target acts as a control (sharding.py:253-256)
            targets, controls = targets[1:], controls + targets[:1]
            m = np.array([[0, 1], [1, 0]], dtype=np.complex128)
            is_diag = False
        for s in self.pending:
            if any(self._shard_value(s, c) == 0 for c in controls if c in glob):
                continue
            lctrl = tuple(c for c in controls if c not in glob)
            if is_diag:
                self._diag_on_shard(s, targets, lctrl, np.diagonal(m), index)
            else:
                if set(targets) & glob:
                    raise SimulationError(f"gate at {index} targets a global qubit; the plan should have reshuffled")
                g = self._local_ngate(targets, lctrl, m, index)
                if g is not None:
                    self.pending[s].append(g)

    def _local_ngate(self, targets, controls, m, index):
        sh = self.sh
        tb = tuple(sh.local_bit(q) for q in targets)
        cb = tuple(sh.local_bit(q) for q in controls)

        class _Spec:  # normalize() takes any object with the GateSpec attributes
            pass

        spec = _Spec()
        spec.kind = GateKind.UNITARY
        spec.targets = tuple(sh.n_local - 1 - b for b in tb)
        spec.controls = tuple(sh.n_local - 1 - b for b in cb)
        spec.params = ()
        spec.matrix = m
        return normalize(spec, sh.n_local, index)

    def _diag_on_shard(self, s, targets, lctrl, d, index):
        sh = self.sh
        glob = set(sh.global_qubits)
        t = len(targets)
        loc_t = [q for q in targets if q not in glob]
        # rows of the diagonal consistent with this shard's global target bits
        sub = []
        for j in range(1 << t):
            ok = True
            for i, q in enumerate(targets):
                if q in glob and ((j >> (t - 1 - i)) & 1) != self._shard_value(s, q):
                    ok = False
                    break
            if ok:
                sub.append(d[j])
        sub = np.array(sub, dtype=np.complex128)
        if not loc_t:
            phase = complex(sub[0])
            if lctrl:
                dd = np.ones(2, dtype=np.complex128)
                dd[1] = phase
                q0, rest = lctrl[0], lctrl[1:]
                g = self._local_ngate((q0,), rest, np.diag(dd), index)
                if g is not None:
                    self.pending[s].append(g)
            elif phase != 1.0:
                self.flush_one(s)
                sh.backend.scale(sh.shards[s], phase)
            return
        g = self._local_ngate(tuple(loc_t), lctrl, np.diag(sub), index)
        if g is not None:
            self.pending[s].append(g)

    def flush_one(self, s):
        sh = self.sh
        if self.pending[s]:
            sh.shards[s] = sh.backend.run_local(sh.shards[s], sh.n_local, self.pending[s], self.cache)
            self.pending[s] = []

    def _swap(self, targets):
        sh = self.sh
        a, b = targets
        glob = set(sh.global_qubits)
        if a in glob and b in glob:
            # shard relabel, no data movement (sharding.py:315-320)
            ja, jb = 1 << sh.shard_bit(a), 1 << sh.shard_bit(b)
            new_shards, new_owner = dict(sh.shards), list(sh.owner)
            for s in range(1 << sh.n_global):
                if bool(s & ja) != bool(s & jb):
                    t = s ^ ja ^ jb
                    new_owner[s] = sh.owner[t]
                    if t in sh.shards:
                        new_shards[s] = sh.shards[t]
                    elif s in new_shards and s not in sh.shards:
                        pass
            # keep only the shards this rank holds under the new labelling
            held = {s: new_shards[s] for s in range(1 << sh.n_global)
                    if sh.comm.owns(s, new_owner) and s in new_shards}
            sh.shards = held
            sh.owner = new_owner
            self.pending = {s: [] for s in sh.shards}
            return
        g_q, l_q = (a, b) if a in glob else (b, a)
        # the reshuffle data movement without the label swap is the gate (sharding.py:302-314)
        _exchange(sh, sh.shard_bit(g_q), sh.local_bit(l_q))


def _make_sharded(state, global_qubits, comm, backend, precision, n):
    if state is not None:
        return partition(state, global_qubits, comm, backend)
    # |0..0> built shard by shard (no full state ever materialised)
    g = len(global_qubits)
    sh = ShardedState(n, tuple(global_qubits), {}, precision, comm=comm, backend=backend)
    nl = n - g
    for s in range(1 << g):
        sh.owner[s] = (s * comm.world) >> g
        if comm.owns(s, sh.owner):
            t = backend.zeros(1 << nl)
            if s == 0:
                t[0] = 1.0
            sh.shards[s] = t
    return sh


def run_sharded(circuit: Circuit, n_shards: int, initial: StateVector | None = None,
                precision: Precision = Precision.F64, global_qubits=None, comm=None, backend=None,
                cache: dict | None = None, exec_plan: ExecutionPlan | None = None) -> ShardedState:
    """Plan + execute; returns the ShardedState (no gather).  `cache` keeps the per-shard fused
    plans (and their compiled kernels) across calls with the same circuit."""
    exec_plan = exec_plan or _default_plan(circuit, n_shards, global_qubits)
    comm = comm or LocalComm()
    backend = backend or CudaBackend(precision if initial is None else initial.precision)
    prec = precision if initial is None else initial.precision
    sh = _make_sharded(initial, exec_plan.global_qubits, comm, backend, prec, circuit.n_qubits)
    _run_steps(sh, circuit, exec_plan, cache)
    return sh


# QSB_SHARD_PLANNER=reference selects the reference's one-qubit Belady schedule (sharding.py:
# 152-216; reshuffle counts equal the reference's); the default is the batched schedule.
SHARD_PLANNER = os.environ.get("QSB_SHARD_PLANNER", "batched")


def _default_plan(circuit, n_shards, global_qubits=None, local_order=None):
    if SHARD_PLANNER == "reference":
        return plan(circuit, n_shards, global_qubits)
    return plan_batched(circuit, n_shards, global_qubits, local_order)


def _run_steps(sh, circuit, exec_plan, cache):
    runner = _Runner(sh, cache, relabel_swaps=exec_plan.relabel_swaps)
    for step in exec_plan.steps:
        if isinstance(step, Reshuffle):
            runner.flush()
            reshuffle(sh, step.global_qubit, step.local_qubit)
        elif isinstance(step, Exchange):
            runner.flush()
            exchange(sh, step.pairs)
        else:
            for pos in step.positions:
                runner.apply(circuit.queue[pos], pos)
    runner.flush()


def apply_sharded(sharded: ShardedState, circuit: Circuit, cache: dict | None = None) -> ShardedState:
    """Run `circuit` on an existing sharded state in place: planned from its current global
    qubits, the state stays sharded (no partition / gather around the circuit)."""
    exec_plan = _default_plan(circuit, 1 << sharded.n_global, sharded.global_qubits, sharded.local_qubits)
    _run_steps(sharded, circuit, exec_plan, cache)
    return sharded


def uniform_sharded(n_qubits: int, n_shards: int, precision: Precision = Precision.F64, comm=None, backend=None,
                    global_qubits=None) -> ShardedState:
    """|+>^n built shard by shard (every amplitude 2^(-n/2), as uniform_state / _plus_state,
    hamiltonians.py:115-117); the full state never exists in one place."""
    comm = comm or LocalComm()
    backend = backend or CudaBackend(precision)
    g = n_shards.bit_length() - 1
    if n_shards < 2 or n_shards & (n_shards - 1) or g >= n_qubits:
        raise ShapeError(f"n_shards must be a power of two in [2, 2^(n-1)], got {n_shards}")
    glob = tuple(global_qubits) if global_qubits is not None else tuple(range(g))
    sh = ShardedState(n_qubits, glob, {}, precision, comm=comm, backend=backend)
    nl = n_qubits - g
    value = float(1.0 / np.sqrt(float(1 << n_qubits)))
    for s_id in range(1 << g):
        sh.owner[s_id] = (s_id * comm.world) >> g
        if comm.owns(s_id, sh.owner):
            t = backend.empty(1 << nl)
            nat.check(nat.lib().qsb_init_uniform(t.data_ptr(), nl, precision.qsb_dtype, value, 0.0, nat.stream_ptr()),
                      "uniform shard")
            sh.shards[s_id] = t
    return sh


def _allreduce_sum(comm, value: float) -> float:
    if isinstance(comm, LocalComm):
        return value
    torch = nat.torch_mod()
    t = torch.tensor([value], dtype=torch.float64, device=torch.device("cuda", torch.cuda.current_device()))
    return float(sum(float(x.item()) for x in comm.all_gather(t)))


def expectation_sharded(h, sharded: ShardedState) -> float:
    """<psi|H|psi> of a Trotter-form Hamiltonian on a sharded state, without gathering it
    (hamiltonians.py:192-207).  Terms on local qubits are summed shard by shard; for the terms
    touching global qubits those globals are first reshuffled with local qubits outside the
    terms' support (the state is unchanged, only its layout)."""
    from .hamiltonians import TrotterHamiltonian, _expect_bit_terms, _fold_single_terms

    if h.n_qubits != sharded.n_qubits:
        raise ShapeError(f"Hamiltonian has {h.n_qubits} qubits, state has {sharded.n_qubits}")
    if not isinstance(h, TrotterHamiltonian):
        raise ShapeError("expectation_sharded needs a Trotter-form Hamiltonian")
    terms = _fold_single_terms(h.terms)

    def local_sum(ts):
        if not ts:
            return 0.0
        acc = 0.0
        for t in sharded.shards.values():
            view = _ShardView(t, sharded.n_local, sharded.precision)
            acc += _expect_bit_terms([(tuple(sharded.local_bit(q) for q in qs), m) for qs, m in ts], view)
        return _allreduce_sum(sharded.comm, acc)

    glob = set(sharded.global_qubits)
    here = [t for t in terms if not set(t[0]) & glob]
    rest = [t for t in terms if set(t[0]) & glob]
    total = local_sum(here)
    if rest:
        support = {q for qs, _ in rest for q in qs}
        for q in [q for q in sharded.global_qubits if q in support]:
            cand = next((x for x in sharded.local_qubits if x not in support), None)
            if cand is None:
                raise CapacityError("too few local qubits outside the terms' support to localise them")
            reshuffle(sharded, q, cand)
        total += local_sum(rest)
    return total


def _shard_vdot(a, b, precision) -> complex:
    from .state import _scalar_buffer

    out = _scalar_buffer(2)
    nat.check(nat.lib().qsb_vdot(a.data_ptr(), b.data_ptr(), a.numel(), precision.qsb_dtype, out.data_ptr(),
                                 nat.stream_ptr()), "shard vdot")
    re, im = out.tolist()
    return complex(re, im)


def norm_sharded(sharded: ShardedState) -> float:
    """Euclidean norm of a sharded state (state.py:109-111): per-shard device sums of |x|^2,
    summed over ranks; no gather."""
    acc = 0.0
    for t in sharded.shards.values():
        acc += _shard_vdot(t, t, sharded.precision).real
    return math.sqrt(_allreduce_sum(sharded.comm, acc))


def overlap_sharded(target, sharded: ShardedState) -> complex:
    """<target|psi> of a sharded state (state.py:114-122) without gathering psi.  `target`: a
    ShardedState of the same qubits (both are brought to the canonical layout) or a StateVector
    (partitioned into psi's canonical layout)."""
    if target.n_qubits != sharded.n_qubits:
        raise ShapeError(f"qubit counts differ: {target.n_qubits} vs {sharded.n_qubits}")
    if target.precision is not sharded.precision:
        raise ValueError("cannot mix f32 and f64 states in one operation")
    canonicalize(sharded)
    if isinstance(target, ShardedState):
        canonicalize(target)
        tgt = target
    else:
        tgt = partition(target, sharded.global_qubits, sharded.comm, sharded.backend)
    re = im = 0.0
    for s_id, t in sharded.shards.items():
        v = _shard_vdot(tgt.shards[s_id], t, sharded.precision)
        re += v.real
        im += v.imag
    return complex(_allreduce_sum(sharded.comm, re), _allreduce_sum(sharded.comm, im))


def canonicalize(sharded: ShardedState) -> None:
    """Bring a sharded state to the canonical layout in place: global qubits {0..g-1} (reshuffles
    with local qubits) and local qubits in significance order (a per-shard bit permutation), so
    that the shards, taken in index order, are the slices of the 1-GPU state vector."""
    g = sharded.n_global
    want = set(range(g))
    for q in list(sharded.global_qubits):
        if q not in want:
            lq = next(x for x in sharded.local_qubits if x in want and x not in sharded.global_qubits)
            reshuffle(sharded, q, lq)
    local = list(sharded.local_qubits)
    if local != sorted(local):
        nl = sharded.n_local
        order = sorted(local)
        dst = [0] * nl
        for m, q in enumerate(local):  # local slot m holds bit nl-1-m
            dst[nl - 1 - m] = nl - 1 - order.index(q)
        for s_id, t in list(sharded.shards.items()):
            sharded.shards[s_id] = sharded.backend.permute(t, nl, dst)
        sharded.local_qubits = tuple(order)


def _canonical_shard_ids(sharded: ShardedState):
    """Shard ids in canonical index order (qubit q < g is bit g-1-q of the canonical index)."""
    g = sharded.n_global
    ids = []
    for c in range(1 << g):
        s_id = 0
        for j, q in enumerate(sharded.global_qubits):
            s_id |= ((c >> (g - 1 - q)) & 1) << (g - 1 - j)
        ids.append(s_id)
    return ids


def sample_sharded(sharded: ShardedState, n_shots: int, seed: int):
    """Sample every qubit of a sharded state without gathering it -- bit-identical to
    measurement.sample(gather(sharded), range(n), n_shots, seed) (SURVEY.md section 8(e),
    exact mode; measurement.py:61-87).

    The state is first brought to the canonical layout (canonicalize).  The sequential cumsum is
    chained shard by shard in index order: each shard's exact cumsum starts from the previous
    shard's last value (prepended as element 0), so every partial sum is rounded exactly as in
    one np.cumsum over the whole vector; the total is the last shard's last value and every
    piece is divided by it.  Each shard then counts, per draw, its entries <= u (unclipped); the
    counts summed over shards (all-reduce across ranks) are np.searchsorted(cum, u, 'right'),
    clipped to [0, 2^n - 1]."""
    from .measurement import MeasurementResult, device_cdf, device_probabilities, device_sample_counts

    if n_shots < 1:
        raise ValueError(f"n_shots must be >= 1, got {n_shots}")
    torch = nat.torch_mod()
    canonicalize(sharded)
    comm = sharded.comm
    order = _canonical_shard_ids(sharded)
    dev = torch.device("cuda", torch.cuda.current_device())
    carry = None
    cums = {}
    for s_id in order:
        owned = s_id in sharded.shards
        if owned:
            view = _ShardView(sharded.shards[s_id], sharded.n_local, sharded.precision)
            p = device_probabilities(view)
            if carry is None:
                cum = device_cdf(p, normalize=False)
            else:
                cum = device_cdf(torch.cat([carry.reshape(1), p]), normalize=False)[1:]
            last = cum[-1:].clone()
            cums[s_id] = cum
        else:
            last = torch.zeros(1, dtype=torch.float64, device=dev)
        if isinstance(comm, LocalComm):
            carry = last
        else:  # the owner's last value reaches every rank (one element per shard, in order)
            parts = comm.all_gather(last)
            carry = parts[sharded.owner[s_id]].to(dev)
    total = carry
    counts = torch.zeros(int(n_shots), dtype=torch.int64, device=dev)
    for s_id, cum in cums.items():
        cum /= total  # numpy: cum /= cum[-1], element-wise IEEE division
        counts += device_sample_counts(cum, n_shots, seed)
    if not isinstance(comm, LocalComm):
        parts = comm.all_gather(counts)
        counts = sum(x.to(dev) for x in parts)
    samples = counts.clamp_(0, (1 << sharded.n_qubits) - 1).cpu().numpy()
    return MeasurementResult(int(n_shots), tuple(range(sharded.n_qubits)), samples, int(seed), {})


def _dist_comm_for(n_shards):
    try:
        import torch.distributed as dist

        if dist.is_available() and dist.is_initialized() and dist.get_world_size() == n_shards:
            return TorchComm()
    except Exception:
        pass
    return LocalComm()


def execute_sharded(circuit: Circuit, n_shards: int, n_workers: int = 1, initial: StateVector | None = None,
                    precision: Precision = Precision.F64, global_qubits=None) -> StateVector:
    """Run a circuit over n_shards shards; result equals Circuit.execute (sharding.py:323-364).

    When torch.distributed is initialised with world_size == n_shards, each rank holds one
    shard and exchanges go over NCCL; otherwise the shards are in-process HBM buffers."""
    if n_workers < 1:
        raise ShapeError(f"n_workers must be >= 1, got {n_workers}")
    if n_shards == 1:
        return circuit.execute(initial, precision=precision)
    if initial is not None and initial.n_qubits != circuit.n_qubits:
        raise ShapeError(f"initial state has {initial.n_qubits} qubits, circuit has {circuit.n_qubits}")
    comm = _dist_comm_for(n_shards)
    sh = run_sharded(circuit, n_shards, initial, precision, global_qubits, comm)
    return gather(sh)


def execute_distributed(circuit: Circuit, precision: Precision = Precision.F64, global_qubits=None,
                        comm=None) -> ShardedState:
    """One shard per rank of the initialised process group, |0..0> initial state, no gather
    (states larger than one GPU: up to 36 qubits on 8 B200)."""
    comm = comm or TorchComm()
    return run_sharded(circuit, comm.world, None, precision, global_qubits, comm)


__all__ = ["Exchange", "ExecutionPlan", "HostStagedComm", "LocalSegment", "Reshuffle", "exchange", "plan_batched", "ShardedState", "apply_sharded", "canonicalize",
           "execute_distributed", "execute_sharded", "expectation_sharded", "gather", "norm_sharded", "overlap_sharded", "partition", "plan", "reshuffle",
           "sample_sharded", "uniform_sharded"]
_ = (_check_cap, zero_state, diag_terms, NGate)
