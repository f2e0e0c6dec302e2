"""Pass planner: turns a gate sequence into fused HBM passes for qsb_run_pass.

The reference applies every gate as its own sweep over the state (circuit.py:121-124 ->
gates.py:380-469).  On B200 the sweep, not the arithmetic, is the cost, so this module packs
runs of gates into "passes": one streaming read + write of the state in which every gate
whose non-diagonal targets fall inside a 2**K-amplitude tile is applied in registers.

Rules (all sound by commutation, never by approximation):
  * a gate g may be hoisted over a deferred gate d iff targets(g) & support(d) == {} and
    targets(d) & support(g) == {} (diagonal gates have no targets; controls and diagonal
    supports are "support");
  * diagonal gates need no locality -> always absorbed (compiled to pivot / parity / term ops);
  * uncontrolled SWAPs are absorbed as relabels (tile-internal: free; tile-external: the pass
    writes tiles to permuted positions, which needs an out-of-place destination);
  * the tile's low L bits are always the low state bits (coalesced 256-byte runs).

The program word format is documented in paper_2009_01845_b200/csrc/pass.cu.
"""

from __future__ import annotations

import os
import struct
import threading
from dataclasses import dataclass, field

import numpy as np

from . import _native as nat
from .gates import KernelClass, classify_kernel, gate_matrix

MAGIC = 0x51534250
VERSION = 3
OP_END, OP_LAYOUT, OP_G1, OP_G2, OP_PIVOT, OP_PARITY, OP_TERM, OP_SCALE = range(8)
G_COMPLEX, G_REAL, G_SWAPX = 0, 1, 2
H_TILEPOS = 16
MAX_PROG_WORDS = 6144
MAX_PIVOTS = 32  # one producer lane per pivot computes its per-tile external factor
THREAD_BITS = 9  # interpreter: 512 consumer threads per CTA (5 lane bits + 4 warp bits)


@dataclass(frozen=True)
class TileGeometry:
    K: int  # tile bits
    G: int  # swizzle group (bank-conflict) bits
    L: int  # low bits always in the tile (256-byte runs)
    R: int = 0  # register (slot) bits per thread; 0 = K - THREAD_BITS (the interpreter's)
    halves: bool = False  # tile staged as two halves split on tile bit K-1 (128 KB tiles)
    # layout changes in two rounds through a half-tile buffer (consecutive layouts share a
    # register bit), so the stage is free as soon as the tile is in registers
    split: bool = False
    # two consumer groups per CTA taking alternate tiles, gate math handed back and forth
    pingpong: bool = False
    two_ctas: bool = False  # two CTAs per SM even with 256 consumers (one stage each, aliased)

    @property
    def nreg(self) -> int:
        return self.R if self.R else self.K - THREAD_BITS

    @property
    def thread_bits(self) -> int:
        return self.K - self.nreg

    @property
    def A(self) -> int:
        return 1 << self.nreg


# interpreter (csrc/pass.cu, fixed 512 consumers) and specialised-kernel (jit.py, 256 consumers
# holding 16 c128 / 32 c64 amplitudes each: fewer layout changes for 2-qubit-gate-heavy passes)
GEOMETRY = {nat.QSB_C128: TileGeometry(12, 3, 4), nat.QSB_C64: TileGeometry(13, 4, 5)}
GEOMETRY_JIT = {nat.QSB_C128: TileGeometry(12, 3, 4, 4), nat.QSB_C64: TileGeometry(13, 4, 5, 5)}
# 128 KB tiles (two 64 KB halves, 32/64 amplitudes per thread): 3-pass QFT-30 plans, but the
# straight-line kernels outgrow the instruction cache on 2-qubit-gate-heavy passes (measured
# round 1: variational c64 55 -> 74 ms, grid 799 -> 1166 ms), so they are opt-in
GEOMETRY_JIT_WIDE = {nat.QSB_C128: TileGeometry(13, 3, 4, 5, True), nat.QSB_C64: TileGeometry(14, 4, 5, 6, True)}
# 128 KB tiles held by 512 consumers (16 / 32 amplitudes each: 4 warps per scheduler)
GEOMETRY_JIT_WIDE512 = {nat.QSB_C128: TileGeometry(13, 3, 4, 4, True), nat.QSB_C64: TileGeometry(14, 4, 5, 5, True)}
# 32 KB tiles, 128 consumers, two CTAs per SM
GEOMETRY_JIT_K11 = {nat.QSB_C128: TileGeometry(11, 3, 4, 4), nat.QSB_C64: TileGeometry(12, 4, 5, 5)}
# c128 passes with dense two-qubit gates: same 64 KB tile, 128 consumers x 32 amplitudes and two
# CTAs per SM (one stage each, reused as the transpose buffer), so one CTA's FP64 work overlaps
# the other's loads and layout changes.  Measured (n = 30): variational 101 -> 94 ms, Trotter
# step 62 -> 58 ms, grid 366 -> 355 ms; QFT passes (no dense 2-qubit gates) keep the default,
# where this geometry was slower (22.6 -> 25.1 ms).
# c64 goes the other way: 512 consumers x 16 amplitudes (half the straight-line code per thread
# of the default 256 x 32), measured variational-30 c64 44.7 -> 41.7 ms; 128 x 64 with two CTAs
# per SM measured 48.2 ms
GEOMETRY_JIT_2Q = {nat.QSB_C128: TileGeometry(12, 3, 4, 5), nat.QSB_C64: TileGeometry(13, 4, 5, 4)}
# ... and its split variant for the lighter of those passes: a separate 32 KB transpose buffer
# (layout changes in two rounds on a shared register bit), so each CTA's stage is refilled
# while the CTA computes instead of after its stores.  Measured (round 2, variational-30 c128):
# passes of <= ~100 FP operations per amplitude 7.45 -> 7.0 ms (8 VariationalLayers, 2 layout
# changes), 7.47 -> 6.73 ms (1 layout change); the 16-layer pass 13.6 -> 15.0 ms, so it is
# chosen per pass (SPLIT_MAX_CODE, and only when it needs no extra layout change).
# QSB_SPLIT_2Q=0 disables it, =1 forces it for every 2-qubit-gate pass.
GEOMETRY_JIT_2Q_SPLIT = {nat.QSB_C128: TileGeometry(12, 3, 4, 5, split=True)}
# QSB_PINGPONG=1: one CTA with two 128-thread consumer groups taking alternate tiles and handing
# the gate-math turn back and forth (named barriers, FA3-style).  Correct, but measured slower
# (round 2, n = 30: variational c128 74.9 -> 86.5 ms, Trotter step 50.3 -> 56.1 ms): one
# group's four warps cannot keep the FP64 pipes busy alone, so serialising the math loses more
# than the overlap with the other group's loads gains.
if os.environ.get("QSB_PINGPONG", "0") == "1":
    GEOMETRY_JIT_2Q = {nat.QSB_C128: TileGeometry(12, 3, 4, 5, pingpong=True), nat.QSB_C64: GEOMETRY_JIT_2Q[nat.QSB_C64]}
    GEOMETRY_JIT_2Q_SPLIT = {}
if os.environ.get("QSB_2Q_GEOMETRY", "") == "x2s16":
    # experiment: c128 256 consumers x 16 amplitudes with two CTAs per SM (one aliased stage each)
    GEOMETRY_JIT_2Q = {nat.QSB_C128: TileGeometry(12, 3, 4, 4, two_ctas=True), nat.QSB_C64: GEOMETRY_JIT_2Q[nat.QSB_C64]}
    GEOMETRY_JIT_2Q_SPLIT = {}
if os.environ.get("QSB_C64_2Q", "") == "x2_256":
    # experiment: complex64 256 consumers x 32 amplitudes at two CTAs per SM
    GEOMETRY_JIT_2Q = {nat.QSB_C128: GEOMETRY_JIT_2Q[nat.QSB_C128], nat.QSB_C64: TileGeometry(13, 4, 5, 5, two_ctas=True)}
if os.environ.get("QSB_C64_2Q", "") == "x2_512":
    GEOMETRY_JIT_2Q = {nat.QSB_C128: GEOMETRY_JIT_2Q[nat.QSB_C128], nat.QSB_C64: TileGeometry(13, 4, 5, 4, two_ctas=True)}
if os.environ.get("QSB_2Q_GEOMETRY", "") == "c64s3":
    # experiment: complex64 512 x 16 with three 64 KB stages + the split 32 KB transpose buffer
    GEOMETRY_JIT_2Q = {nat.QSB_C128: GEOMETRY_JIT_2Q[nat.QSB_C128], nat.QSB_C64: TileGeometry(13, 4, 5, 4, split=True)}
if os.environ.get("QSB_2Q_GEOMETRY", "") == "s3":
    # experiment: 256 consumers x 16 amplitudes, one CTA per SM, three 64 KB stages + the split
    # 32 KB transpose buffer (half the straight-line code per thread, three tiles in flight)
    GEOMETRY_JIT_2Q = {nat.QSB_C128: TileGeometry(12, 3, 4, 4, split=True), nat.QSB_C64: GEOMETRY_JIT_2Q[nat.QSB_C64]}
    GEOMETRY_JIT_2Q_SPLIT = {}
SPLIT_2Q = os.environ.get("QSB_SPLIT_2Q", "auto")
# ... and the 256 x 16 two-CTA variant for the heavier ones (measured round 2, n = 30: variational
# passes of 21 / 32 / 25 gates 10.0 / 13.1 / 9.8 -> 9.6 / 12.2 / 9.6 ms, Trotter 9-gate passes
# 10.0 -> 9.4 ms; lighter passes are faster split).  QSB_X2_2Q=0 disables it.
GEOMETRY_JIT_2Q_X2 = {nat.QSB_C128: TileGeometry(12, 3, 4, 4, two_ctas=True),
                      nat.QSB_C64: TileGeometry(13, 4, 5, 5, two_ctas=True)}
X2_2Q = os.environ.get("QSB_X2_2Q", "1") != "0"
# passes whose gate code is too big for 32 amplitudes per thread (the grid's 16-gate passes) also
# run 256 x 16 at two CTAs per SM instead of one CTA with two stages (20.4 / 23.4 -> 19.5 / 22.4 ms)
X2_BIG = os.environ.get("QSB_X2_BIG", "1") != "0"
X2_C64 = os.environ.get("QSB_X2_C64", "0") == "1"
# complex64 passes of at least this much FP work per amplitude run 256 x 32 (0 disables)
C64_WIDE_MIN_CODE = float(os.environ.get("QSB_C64_WIDE_MIN_CODE", "90"))
C64_WIDE_MAX_CODE = 160.0
SPLIT_MAX_CODE = float(os.environ.get("QSB_SPLIT_MAX_CODE", "100"))
# ... unless the pass's straight-line gate code per thread (FP operations per amplitude x 32
# amplitudes) would outgrow the instruction cache: measured on grid-30, the two passes of 16
# dense complex 4x4 gates (~8,200 FP instructions per thread) ran 21.5 / 32.0 ms in that geometry
# and 19.0 / 20.0 ms in the default one, while variational's 16 real 4x4 gates (~4,100) and the
# grid's 10-gate passes (~5,100) are faster in it
MAX_2Q_CODE = int(os.environ.get("QSB_MAX_2Q_CODE", "6500"))
# QSB_BALANCE_DIAGONALS=1: spread the trailing diagonals of diagonal-heavy plans evenly over the
# passes.  Measured slower (round 2, QFT-30 c128: passes 212/149/92/27 gates 20.8 ms -> 155/156/
# 142/27 gates 23.2 ms): a deferred cross-tile phase costs more in the later passes (more
# pivots, tile-external partners) than in the first, so it is off.
BALANCE_DIAGONALS = os.environ.get("QSB_BALANCE_DIAGONALS", "0") == "1"
_GEO_ENV = os.environ.get("QSB_JIT_GEOMETRY", "")
if _GEO_ENV == "wide":
    GEOMETRY_JIT = GEOMETRY_JIT_WIDE
elif _GEO_ENV == "wide512":
    GEOMETRY_JIT = GEOMETRY_JIT_WIDE512
elif _GEO_ENV == "k11":
    GEOMETRY_JIT = GEOMETRY_JIT_K11
elif _GEO_ENV == "q512":
    # 512 consumers x 8 (c128) / 16 (c64) amplitudes: more warps per scheduler, but twice the
    # layout changes -- measured QFT-30 c128 22.7 -> 28.1 ms, so not the default
    GEOMETRY_JIT = {nat.QSB_C128: TileGeometry(12, 3, 4, 3), nat.QSB_C64: TileGeometry(13, 4, 5, 4)}
elif _GEO_ENV == "k12x2":
    # c128: 64 KB tiles, 128 consumers x 32 amplitudes, two CTAs per SM (one stage each, reused
    # as the transpose buffer) so one CTA's FP64 work overlaps the other's loads / transposes
    GEOMETRY_JIT = {nat.QSB_C128: TileGeometry(12, 3, 4, 5), nat.QSB_C64: GEOMETRY_JIT[nat.QSB_C64]}


def _f2w(x: float) -> int:
    return struct.unpack("<q", struct.pack("<d", float(x)))[0]


def _bits(positions) -> int:
    m = 0
    for p in positions:
        m |= 1 << p
    return m


# ------------------------------------------------------------------------------------------
# normalised gates (bit positions, not qubits)
# ------------------------------------------------------------------------------------------
@dataclass
class NGate:
    kind: str  # "diag" | "g1" | "g2" | "swap"
    targets: tuple  # bit positions; targets[0] = matrix MSB
    controls: tuple
    matrix: np.ndarray | None  # g1/g2: 2^t x 2^t; diag: the diagonal
    tmask: int
    smask: int
    index: int = -1  # position in the source queue
    # matrix (g1 / g2) or diagonal (diag) as a function of the source gates' matrices: how a
    # plan template (PlanTemplate) recomputes it for a circuit of the same structure
    build: object = None

    def touched_fraction(self) -> float:
        """Share of the state a stand-alone single-gate kernel reads+writes."""
        c = 2.0 ** -len(self.controls)
        if self.kind == "diag":
            rows = int(np.count_nonzero(self.matrix != 1.0))
            return c * rows / len(self.matrix)
        if self.kind == "swap":
            return 0.5
        return c


_SWAP = np.array([[1, 0, 0, 0], [0, 0, 1, 0], [0, 1, 0, 0], [0, 0, 0, 1]], dtype=np.complex128)
_XMAT = np.array([[0, 1], [1, 0]], dtype=np.complex128)


# Real or imaginary parts below this magnitude are rounding noise of the host matrix algebra
# (1e-17 .. 5e-16 where the step exponentials and gate products are exactly zero) and are
# planned as exact zeros: the kernels skip them, and a time-dependent circuit's structure does
# not flip between steps with the noise.  The dropped terms change an amplitude by at most
# ~1e-15 of its norm per gate, far inside the 1e-12 parity bound.  QSB_SNAP_TINY=0 disables.
SNAP_TINY = float(os.environ.get("QSB_SNAP_TINY", "1e-15"))


def _snap(m):
    m = np.array(m, dtype=np.complex128)
    if SNAP_TINY > 0:
        v = m.reshape(-1).view(np.float64)
        v[np.abs(v) < SNAP_TINY] = 0.0
    return m


def normalize(spec, n_qubits: int, index: int = -1, m=None) -> NGate | None:
    """GateSpec (or duck-typed reference GateSpec) -> NGate; None for exact identities.  `m`:
    the spec's gate matrix (as plan_circuit snaps it) when the caller has it already."""
    if m is None:
        m = _snap(gate_matrix(spec))
    tb = tuple(n_qubits - 1 - int(q) for q in spec.targets)
    cb = tuple(n_qubits - 1 - int(q) for q in spec.controls)
    support = _bits(tb + cb)
    i = index
    if classify_kernel(m) is KernelClass.DIAGONAL:
        d = np.ascontiguousarray(np.diagonal(m))
        if np.all(d == 1.0):
            return None  # the reference's diagonal body finds no rows and returns
        return NGate("diag", tb, cb, d, 0, support, index, lambda M: np.ascontiguousarray(np.diagonal(M[i])))
    if len(tb) == 2:
        if not cb and np.array_equal(m, _SWAP):
            return NGate("swap", tb, (), None, support, support, index)
        # controlled single-qubit form [[I, 0], [0, U]]: control targets[0], act on targets[1]
        if (
            np.array_equal(m[:2, :2], np.eye(2))
            and not np.any(m[:2, 2:])
            and not np.any(m[2:, :2])
        ):
            u = np.ascontiguousarray(m[2:, 2:])
            if classify_kernel(u) is KernelClass.DIAGONAL:
                d = np.ones(4, dtype=np.complex128)
                d[2:] = np.diagonal(u)
                return NGate("diag", tb, cb, d, 0, support, index,
                             lambda M: np.concatenate((np.ones(2, dtype=np.complex128), np.diagonal(M[i])[2:])))
            return NGate("g1", (tb[1],), cb + (tb[0],), u, 1 << tb[1], support, index,
                         lambda M: np.ascontiguousarray(M[i][2:, 2:]))
        return NGate("g2", tb, cb, np.ascontiguousarray(m), _bits(tb), support, index, lambda M: M[i])
    return NGate("g1", tb, cb, np.ascontiguousarray(m), _bits(tb), support, index, lambda M: M[i])


def _product_build(*parts):
    """build of a product of gate factors: each part is a build, a constant matrix, or
    ('kron', part, part) / ('embed', part, pos) / ('diag', part)."""

    def ev(p, M):
        if isinstance(p, tuple):
            if p[0] == "kron":
                return _kron2(ev(p[1], M), ev(p[2], M))
            if p[0] == "embed":
                return _embed_1q(ev(p[1], M), p[2])
            if p[0] == "diag":
                return np.diag(ev(p[1], M))
            if p[0] == "perm":
                return ev(p[1], M)[np.ix_(_PERM2, _PERM2)]
        if callable(p):
            return p(M)
        return p

    def known(p):
        if isinstance(p, tuple):
            return all(known(x) for x in p[1:] if not isinstance(x, int))
        return p is not None

    if not all(known(p) for p in parts):
        return None
    flat = list(parts)

    def build(M):
        out = ev(flat[0], M)
        for p in flat[1:]:
            out = out @ ev(p, M)
        return _snap(out)

    return build


_PERM2 = [0, 2, 1, 3]


def _entry_cost(z) -> float:
    """FP ops per use of one matrix entry in the specialised gate bodies (jit.matrix_coeffs)."""
    if z == 0:
        return 0.0
    if z == 1 or z == -1:
        return 1.0
    if z.imag == 0 or z.real == 0:
        return 2.0
    return 4.0


def matrix_cost(m: np.ndarray) -> float:
    """FP ops per amplitude of applying `m` (sum of entry costs / dimension, _entry_cost per
    entry; a plain loop: the matrices are at most 4 x 4 and numpy's per-call overhead dominated
    host planning)."""
    a = np.asarray(m, dtype=np.complex128)
    total = 0.0
    for z in a.reshape(-1).tolist():
        if z == 0:
            continue
        re, im = z.real, z.imag
        if im == 0 and (re == 1 or re == -1):
            total += 1.0
        elif re == 0 or im == 0:
            total += 2.0
        else:
            total += 4.0
    return total / a.shape[0]


_EYE2 = np.eye(2, dtype=np.complex128)


def _kron2(a: np.ndarray, b: np.ndarray) -> np.ndarray:
    """np.kron of two 2x2 matrices (a = MSB factor) without np.kron's per-call overhead."""
    return (np.asarray(a)[:, None, :, None] * np.asarray(b)[None, :, None, :]).reshape(4, 4)


def _embed_1q(u: np.ndarray, pos: int) -> np.ndarray:
    """4x4 of a single-qubit matrix on target `pos` (0 = matrix MSB) of a two-qubit gate."""
    return _kron2(u, _EYE2) if pos == 0 else _kron2(_EYE2, u)


def merge_1q_runs(gates: list) -> list:
    """Consecutive uncontrolled single-qubit gates on the same qubit (no other gate on it in
    between) become their product when that is cheaper (two dense 2x2 -> one)."""
    out = list(gates)
    alive = [True] * len(out)
    for i, g in enumerate(out):
        if not alive[i] or g.kind != "g1" or g.controls:
            continue
        bit = 1 << g.targets[0]
        j = next((k for k in range(i + 1, len(out)) if alive[k] and out[k].smask & bit), None)
        if j is None:
            continue
        h = out[j]
        if h.kind == "g1" and not h.controls and h.targets == g.targets:
            m = _snap(h.matrix @ g.matrix)
            if matrix_cost(m) < matrix_cost(h.matrix) + matrix_cost(g.matrix) - 1e-9:
                out[j] = NGate("g1", h.targets, (), m, h.tmask, h.smask, h.index, _product_build(h.build, g.build))
                alive[i] = False
    return [g for g, a in zip(out, alive) if a]


def sandwich_diagonals(gates: list) -> list:
    """Fold the single-qubit gates adjacent to an uncontrolled two-qubit diagonal gate (before
    and after it, on both of its bits) into one dense 4x4 when that is cheaper: the unfused
    variational layer RY RY . CZ . RY RY (4 x 4 FMAs per amplitude) becomes the fused
    VariationalLayer form (8).  Diagonals with a cheaper sandwich stay diagonal (the QFT's
    CZPow after an H: pivots make the diagonal nearly free)."""
    out = list(gates)
    alive = [True] * len(out)

    def neighbour(i, bit, step):
        k = i + step
        while 0 <= k < len(out):
            if alive[k] and out[k].smask & bit:
                return k
            k += step
        return None

    for i, d in enumerate(out):
        if not alive[i] or d.kind not in ("diag", "g2") or d.controls or len(d.targets) != 2:
            continue
        parts, pre, post = [], [_EYE2, _EYE2], [_EYE2, _EYE2]
        pre_b, post_b = [_EYE2, _EYE2], [_EYE2, _EYE2]
        for pos, t in enumerate(d.targets):
            bit = 1 << t
            for step, slot, slot_b in ((-1, pre, pre_b), (1, post, post_b)):
                k = neighbour(i, bit, step)
                if k is not None and out[k].kind == "g1" and not out[k].controls and out[k].targets == (t,):
                    parts.append(k)
                    slot[pos] = out[k].matrix
                    slot_b[pos] = out[k].build
        if not parts:
            continue
        core = np.diag(d.matrix) if d.kind == "diag" else d.matrix
        core_cost = 0.0 if d.kind == "diag" else matrix_cost(d.matrix)
        merged = _snap(_kron2(post[0], post[1]) @ core @ _kron2(pre[0], pre[1]))
        if matrix_cost(merged) < core_cost + sum(matrix_cost(out[k].matrix) for k in parts) - 1e-9:
            core_b = ("diag", d.build) if d.kind == "diag" else d.build
            out[i] = NGate("g2", d.targets, (), merged, _bits(d.targets), d.smask, d.index,
                           _product_build(("kron", post_b[0], post_b[1]), core_b, ("kron", pre_b[0], pre_b[1])))
            for k in parts:
                alive[k] = False
    return [g for g, a in zip(out, alive) if a]


def merge_single_qubit(gates: list, slack: float = 0.0) -> list:
    """Fold uncontrolled single-qubit gates into the neighbouring two-qubit gate on the same bit
    when the product is cheaper to apply than the two separately (entry-structure cost model:
    e.g. the X rotation of a Trotter ZZ + hX term's first qubit keeps its 8-entry block structure;
    both single-qubit layers around an fSim make it a dense 4x4, still cheaper than three gates).
    Only gates with no other gate on that bit in between are folded, so the product is exact
    algebra on adjacent operators (the reference applies them one by one: results agree to
    rounding, far inside the 1e-12 / 1e-5 parity bounds)."""
    out = list(gates)
    alive = [True] * len(out)
    for i, g in enumerate(out):
        if g.kind != "g1" or g.controls or not alive[i]:
            continue
        q = g.targets[0]
        bit = 1 << q
        u = g.matrix
        # forward: the next gate touching q
        j = next((k for k in range(i + 1, len(out)) if alive[k] and out[k].smask & bit), None)
        if j is not None and out[j].kind == "g2" and not out[j].controls and q in out[j].targets:
            h = out[j]
            merged = _snap(h.matrix @ _embed_1q(u, h.targets.index(q)))
            if matrix_cost(merged) < matrix_cost(h.matrix) + matrix_cost(u) + slack - 1e-9:
                out[j] = NGate("g2", h.targets, (), merged, h.tmask, h.smask, h.index,
                               _product_build(h.build, ("embed", g.build, h.targets.index(q))))
                alive[i] = False
                continue
        # backward: the previous gate touching q
        k = next((k for k in range(i - 1, -1, -1) if alive[k] and out[k].smask & bit), None)
        if k is not None and out[k].kind == "g2" and not out[k].controls and q in out[k].targets:
            h = out[k]
            merged = _snap(_embed_1q(u, h.targets.index(q)) @ h.matrix)
            if matrix_cost(merged) < matrix_cost(h.matrix) + matrix_cost(u) + slack - 1e-9:
                out[k] = NGate("g2", h.targets, (), merged, h.tmask, h.smask, h.index,
                               _product_build(("embed", g.build, h.targets.index(q)), h.build))
                alive[i] = False
    return [g for g, a in zip(out, alive) if a]


def merge_2q_runs(gates: list) -> list:
    """Consecutive uncontrolled two-qubit gates on the same bit pair (no other gate on either
    bit in between) become their product when that is cheaper: the trailing half step of one
    Trotter step and the leading half step of the next (with the single-qubit layer between
    them folded in by merge_single_qubit) are one 4x4 when evolve() plans steps together."""
    out = list(gates)
    alive = [True] * len(out)
    for i, g in enumerate(out):
        if not alive[i] or g.kind != "g2" or g.controls:
            continue
        j = next((k for k in range(i + 1, len(out)) if alive[k] and out[k].smask & g.smask), None)
        if j is None:
            continue
        h = out[j]
        if h.kind != "g2" or h.controls or set(h.targets) != set(g.targets):
            continue
        same = h.targets == g.targets
        gm = g.matrix if same else g.matrix[np.ix_(_PERM2, _PERM2)]
        m = _snap(h.matrix @ gm)
        if matrix_cost(m) < matrix_cost(h.matrix) + matrix_cost(g.matrix) - 1e-9:
            out[j] = NGate("g2", h.targets, (), m, h.tmask, h.smask, h.index,
                           _product_build(h.build, g.build if same else ("perm", g.build)))
            alive[i] = False
    return [g for g, a in zip(out, alive) if a]


def diag_terms(g: NGate):
    """(mask, value, phase) rows of a diagonal gate: exactly the rows the reference multiplies
    (diag entry != 1.0), restricted to the control subspace."""
    t = len(g.targets)
    cmask = _bits(g.controls)
    mask = _bits(g.targets) | cmask
    out = []
    for j, w in enumerate(g.matrix):
        if w == 1.0:
            continue
        val = cmask
        for i, b in enumerate(g.targets):
            if (j >> (t - 1 - i)) & 1:
                val |= 1 << b
        out.append((mask, val, complex(w)))
    return out


# ------------------------------------------------------------------------------------------
# plan
# ------------------------------------------------------------------------------------------
@dataclass
class PassStep:
    words: np.ndarray
    gates: list  # absorbed NGates
    tile_pos: tuple
    ext_perm: bool
    n_transposes: int
    n_pivots: int
    jit: object = None  # (compiled kernel, coefficient array) once specialised
    no_jit: bool = False
    interp_words: object = None  # re-encoding for the interpreter's geometry (fallback only)
    dev_tables: object = None  # device copy of the pivot tables (engine.own_device_tables; graph capture)
    tpl: object = None  # (geometry, dense-gate matrix word positions, has diagonals): PlanTemplate

    @property
    def n_gates(self) -> int:
        return len(self.gates)


@dataclass
class GateStep:
    gate: NGate


@dataclass
class Plan:
    n_qubits: int
    dtype: int
    steps: list = field(default_factory=list)

    @property
    def n_passes(self) -> int:
        return sum(1 for s in self.steps if isinstance(s, PassStep))

    def state_sweeps(self) -> float:
        """Algorithmic state read+write sweeps (the roofline's unit): 1 per pass, the touched
        fraction per stand-alone gate."""
        total = 0.0
        for s in self.steps:
            total += 1.0 if isinstance(s, PassStep) else s.gate.touched_fraction()
        return total


def _absorbed_cost(absorbed) -> float:
    return sum(matrix_cost(g.matrix) if g.kind in ("g1", "g2") else 0.25 for g in absorbed)


def _select_pass_best(gates, n, geo: TileGeometry, allow_ext: bool, max_runs=None, fp_budget=None):
    """The better of two absorption scans (by FP work absorbed): the greedy one, and one where
    single-qubit gates may not pull new bits into the tile (a run of 1-qubit gates on scattered
    bits otherwise fills the tile with bits no 2-qubit gate pairs up), whose tile is then
    re-scanned as fixed."""
    a1, d1, t1 = _select_pass(gates, n, geo, allow_ext, max_runs=max_runs, fp_budget=fp_budget)
    _, _, t_lazy = _select_pass(gates, n, geo, allow_ext, lazy_1q=True, max_runs=max_runs, fp_budget=fp_budget)
    a2, d2, t2 = _select_pass(gates, n, geo, allow_ext, fixed=t_lazy, fp_budget=fp_budget)
    if _absorbed_cost(a2) > _absorbed_cost(a1) + 1e-9:
        return a2, d2, t2
    return a1, d1, t1


def _select_pass(gates, n, geo: TileGeometry, allow_ext: bool, lazy_1q: bool = False, fixed=None,
                 max_runs=None, fp_budget=None):
    """Greedy absorption scan: returns (absorbed, deferred, tile position set).  `fixed`: the
    tile is given (no growth); `lazy_1q`: single-qubit gates never add tile bits."""
    K, L = geo.K, geo.L
    T = set(range(L)) if fixed is None else set(fixed)
    grow = fixed is None
    frozen = set()
    loc = list(range(n))
    blocked_support = 0
    blocked_targets = 0
    absorbed, deferred = [], []
    fp_used = 0.0
    for g in gates:
        take = False
        if (g.tmask & blocked_support) or (g.smask & blocked_targets):
            take = False
        elif g.kind == "diag":
            take = True
        elif g.kind == "swap":
            x, y = g.targets
            px, py = loc[x], loc[y]
            inx, iny = px in T, py in T
            if inx and iny:
                take = True
            elif not inx and not iny:
                # tile-external relabel: keep enough unfrozen positions to fill the tile
                take = allow_ext and n - len(frozen | {px, py}) >= K
                if take:
                    frozen.update((px, py))
            else:
                other = py if inx else px
                if grow and len(T) < K and other not in frozen and (max_runs is None
                                                                     or _tile_runs(T | {other}) <= max_runs):
                    T.add(other)
                    take = True
                elif allow_ext and other not in frozen and min(px, py) >= L:
                    # tile bit <-> external bit relabel (out of place): the tile bit is stored
                    # to the external position and vice versa.  Never for the low L bits: the
                    # output's contiguous runs must come from tile bits (measured: strided
                    # 16-byte stores made such a QFT-30 pass 2.5x slower)
                    frozen.add(other)
                    take = True
            if take:
                loc[x], loc[y] = loc[y], loc[x]
        elif fp_budget is not None and fp_used + matrix_cost(g.matrix) > fp_budget and fp_used > 0:
            take = False  # the pass has its share of gate arithmetic: later passes take the rest
        else:
            need = {loc[t] for t in g.targets}
            new = need - T
            if not new:
                take = True
            elif (grow and len(T) + len(new) <= K and not (new & frozen) and not (lazy_1q and len(need) == 1)
                  and (max_runs is None or _tile_runs(T | new) <= max_runs)):
                T |= new
                take = True
        if take:
            if fp_budget is not None and g.kind in ("g1", "g2"):
                fp_used += matrix_cost(g.matrix)
            absorbed.append(g)
        else:
            deferred.append(g)
            blocked_support |= g.smask
            blocked_targets |= g.tmask
    # fill the tile with the lowest free positions (longer contiguous runs)
    for p in range(n):
        if len(T) >= K:
            break
        if p not in T and p not in frozen:
            T.add(p)
    return absorbed, deferred, T


# ------------------------------------------------------------------------------------------
# plan templates: a circuit with the structure of one planned before -- the same qubits and
# controls gate by gate, and the same class (0, +-1, +-1/sqrt 2, rounding noise, other) for the
# real and imaginary part of every matrix entry: the values the planner's and the kernel
# generator's structure decisions test -- e.g. each step of a time-dependent Trotter evolution,
# reuses that plan: merged matrices are recomputed from the recorded products (NGate.build), and
# each pass's program gets the new matrix words patched in (passes with diagonal terms, whose
# words hold derived phase products, are re-encoded with the recorded tile and geometry).  An
# exact 0 where the template held rounding noise (1e-17 from the step exponentials in one step,
# 0 in the next) fits too: that entry's code multiplies by whatever is there.  Anything else
# that changes class -- an exact identity where the template had a rotation, which a fresh plan
# drops -- plans from scratch, and the new plan becomes the newest template for that gate
# layout.  QSB_PLAN_TEMPLATES=0 disables.
# ------------------------------------------------------------------------------------------
PLAN_TEMPLATES = os.environ.get("QSB_PLAN_TEMPLATES", "1") != "0"
_TEMPLATES: dict = {}
_TEMPLATES_LOCK = threading.Lock()  # ranks planning concurrently (thread ranks, precompile pools)
_TEMPLATES_MAX = 64
_HH = 0.7071067811865475
_GENERIC = 5
_TINY = 6
TEMPLATE_STATS = {"hits": 0, "misses": 0, "rejected": 0}


def _entry_classes(m) -> np.ndarray:
    """Class of every real and imaginary part of a matrix (uint8): 0, 1, -1, 1/sqrt 2,
    -1/sqrt 2 -> 0..4, rounding-noise size (0 < |x| <= 1e-12) -> _TINY, anything else ->
    _GENERIC."""
    v = np.ascontiguousarray(m, dtype=np.complex128).reshape(-1).view(np.float64)
    out = np.full(v.shape[0], _GENERIC, np.uint8)
    out[np.abs(v) <= 1e-12] = _TINY
    out[v == 0.0] = 0
    out[v == 1.0] = 1
    out[v == -1.0] = 2
    out[v == _HH] = 3
    out[v == -_HH] = 4
    return out


def _planner_switches():
    """Module switches the planner reads (part of a template's key: tests and experiments flip
    them at run time)."""
    return (SNAP_TINY, MERGE_SLACKS, FP_PER_SWEEP, FP_BUDGETS, BALANCE_DIAGONALS, REORDER_GATES, SEED_GATES, MINIMAL_LAYOUT_CHANGES, TMA_STORE_LAYOUT, SPLIT_2Q,
            SPLIT_MAX_CODE, MAX_2Q_CODE, X2_2Q, X2_BIG, X2_C64, C64_WIDE_MIN_CODE, id(GEOMETRY_JIT), id(GEOMETRY_JIT_2Q),
            id(GEOMETRY_JIT_2Q_SPLIT), id(GEOMETRY_JIT_2Q_X2))


def _compatible(old: np.ndarray, new: np.ndarray) -> bool:
    """New entries fit a template's: the same class, or an exact 0 where the template held
    rounding noise (its code multiplies by whatever is there)."""
    return old.shape == new.shape and bool(np.all((new == old) | ((old == _TINY) & (new == 0))))


class PlanTemplate:
    def __init__(self, plan: Plan, leaf_classes: np.ndarray):
        self.plan = plan
        self.leaf_classes = leaf_classes
        self.classes = {}  # id(gate) -> entry classes of its matrix in the template
        for st in plan.steps:
            for g in (st.gates if isinstance(st, PassStep) else [st.gate]):
                if g.kind != "swap" and g.matrix is not None:
                    self.classes[id(g)] = _entry_classes(g.matrix)

    def _rebuilt(self, g: NGate, M):
        if g.kind == "swap":
            return g
        if g.build is None:
            return None
        m = _snap(g.build(M))
        if m.shape != g.matrix.shape or not _compatible(self.classes[id(g)], _entry_classes(m)):
            return None
        return NGate(g.kind, g.targets, g.controls, m, g.tmask, g.smask, g.index, g.build)

    def instantiate(self, M) -> Plan | None:
        """The template's plan for the gate matrices M (None: a special entry changed)."""
        src = self.plan
        out = Plan(src.n_qubits, src.dtype)
        for st in src.steps:
            if isinstance(st, GateStep):
                g = self._rebuilt(st.gate, M)
                if g is None:
                    return None
                out.steps.append(GateStep(g))
                continue
            gates = []
            for g in st.gates:
                h = self._rebuilt(g, M)
                if h is None:
                    return None
                gates.append(h)
            geo, mpos, has_diag = st.tpl
            if has_diag:
                words, info = compile_pass(gates, set(st.tile_pos), src.n_qubits, src.dtype, geo,
                                           minimal=MINIMAL_LAYOUT_CHANGES)
                mp = info["mpos"]
            else:
                words = st.words.copy()
                where = {id(g): k for k, g in enumerate(st.gates)}
                mp = []
                for pos, g_old, swapped in mpos:
                    g = gates[where[id(g_old)]]
                    m = g.matrix[np.ix_(_PERM2, _PERM2)] if swapped else g.matrix
                    v = np.ascontiguousarray(m, dtype=np.complex128).reshape(-1).view(np.int64)
                    words[pos:pos + v.shape[0]] = v
                    mp.append((pos, g, swapped))
            out.steps.append(PassStep(words, gates, st.tile_pos, st.ext_perm, st.n_transposes, st.n_pivots,
                                      tpl=(geo, mp, has_diag)))
        return out


def plan_circuit(specs, n_qubits: int, dtype: int, allow_ext_perm: bool = True, fuse: bool = True,
                 geometry: TileGeometry | None = None) -> Plan:
    """Plan a gate list into PassSteps (fused) and GateSteps (stand-alone kernels).  `geometry`
    defaults to the interpreter's (GEOMETRY); the specialised kernels use GEOMETRY_JIT."""
    geo = geometry or GEOMETRY[dtype]
    use_tpl = (PLAN_TEMPLATES and fuse and n_qubits >= geo.K + 1 and len(specs) > 0
               and not any(isinstance(spec, NGate) for spec in specs))
    mats = key = leaf = None
    if use_tpl:
        mats = [_snap(gate_matrix(spec)) for spec in specs]
        key = (n_qubits, dtype, geo, allow_ext_perm, _planner_switches(),
               tuple((tuple(int(q) for q in spec.targets), tuple(int(q) for q in spec.controls), m.shape[0])
                     for spec, m in zip(specs, mats)))
        leaf = _entry_classes(np.concatenate([np.asarray(m, dtype=np.complex128).reshape(-1) for m in mats]))
        with _TEMPLATES_LOCK:
            tpls = list(_TEMPLATES.get(key, ()))
        for tpl in tpls:
            if not _compatible(tpl.leaf_classes, leaf):
                continue
            plan = tpl.instantiate(mats)
            if plan is not None:
                TEMPLATE_STATS["hits"] += 1
                return plan
            TEMPLATE_STATS["rejected"] += 1
        TEMPLATE_STATS["misses"] += 1
    gates = []
    for i, spec in enumerate(specs):
        if isinstance(spec, NGate):
            g = spec
        else:
            g = normalize(spec, n_qubits, i, mats[i] if mats is not None else None)
        if g is not None:
            gates.append(g)
    plan = Plan(n_qubits, dtype)
    if not fuse or n_qubits < geo.K + 1:
        plan.steps = [GateStep(g) for g in gates]
        return plan
    base = sandwich_diagonals(merge_1q_runs(gates))
    best = None
    seen = {}

    def trial(cand, budget, runs):
        nonlocal best
        alt = _plan_passes(Plan(n_qubits, dtype), cand, n_qubits, dtype, geo, allow_ext_perm, None,
                           max_runs=runs, fp_budget=budget, estimate_only=True)
        est = plan_estimate(alt)
        if best is None or est < best[0] - 1e-9:
            best = (est, alt, cand, budget, runs)

    for slack in MERGE_SLACKS:
        # folding a single-qubit gate into a 2-qubit neighbour that gets a little dearer can
        # let two 2-qubit gates on the same pair meet and merge (consecutive Trotter steps: 383
        # -> 315 FMAs per amplitude per step at n = 30), or just cost more; and capping the
        # gate arithmetic a pass absorbs re-orders the greedy selection, sometimes into fewer
        # passes: each variant is planned (tiles only) and the lowest estimate encoded
        cand = merge_2q_runs(merge_single_qubit(base, slack))
        sig = tuple((g.kind, g.targets, g.controls, round(matrix_cost(g.matrix), 6) if g.kind in ("g1", "g2") else 0)
                    for g in cand)
        if sig in seen:
            continue
        seen[sig] = cand
        for budget in (None,) + FP_BUDGETS:
            trial(cand, budget, None)
    if any(_tile_runs(st.tile_pos) > MAX_TILE_RUNS for st in best[1].steps if isinstance(st, PassStep)):
        # a tile of scattered bits (e.g. a layer of single-qubit gates on every other qubit
        # pulled into one pass) loads in pieces: also plan with tiles of at most five runs
        for cand in seen.values():
            for budget in (None,) + FP_BUDGETS:
                trial(cand, budget, MAX_TILE_RUNS)
    _, _, gates, budget, runs = best
    plan = _plan_passes(plan, gates, n_qubits, dtype, geo, allow_ext_perm, None, max_runs=runs, fp_budget=budget)
    if BALANCE_DIAGONALS:
        # diagonal-heavy plans (the QFT: 204 / 141 / 84 / 21 diagonal gates in its four passes
        # at n = 30) keep their early passes compute-bound; the trailing diagonals of a pass
        # (nothing later in it acts non-diagonally on their qubits) may run in any later pass
        # that precedes their next non-diagonal use, so spread them evenly
        passes = [st for st in plan.steps if isinstance(st, PassStep)]
        counts = [sum(1 for g in st.gates if g.kind == "diag") for st in passes]
        if len(passes) >= 3 and max(counts) > 1.5 * (sum(counts) / len(counts)) + 8:
            # passes that cannot pass diagonals on (their qubits are used right after) end up
            # above the budget: try a few budgets and keep the plan with the lowest maximum
            mean = sum(counts) / len(counts)
            best, best_max = plan, max(counts)
            for f in (1.0, 1.1, 1.2, 1.35, 1.5):
                budget = int(mean * f + 0.5)
                if budget >= best_max:
                    break
                alt = _plan_passes(Plan(n_qubits, dtype), gates, n_qubits, dtype, geo, allow_ext_perm, budget)
                if alt.n_passes != plan.n_passes or alt.state_sweeps() > plan.state_sweeps() + 1e-9:
                    continue
                m = max(sum(1 for g in st.gates if g.kind == "diag") for st in alt.steps if isinstance(st, PassStep))
                if m < best_max:
                    best, best_max = alt, m
            plan = best
    if use_tpl:
        tpl = PlanTemplate(plan, leaf)
        with _TEMPLATES_LOCK:
            if len(_TEMPLATES) >= _TEMPLATES_MAX and key not in _TEMPLATES:
                _TEMPLATES.pop(next(iter(_TEMPLATES)))
            # newest first; a few per gate layout (e.g. the first steps of an adiabatic
            # schedule, where a zero coefficient makes gates exact identities)
            _TEMPLATES[key] = [tpl] + _TEMPLATES.get(key, [])[:3]
    return plan


# merge_single_qubit cost slacks tried by plan_circuit (QSB_MERGE_SLACKS, comma separated)
MERGE_SLACKS = tuple(float(x) for x in os.environ.get("QSB_MERGE_SLACKS", "0,4,8").split(",") if x.strip())
# Pass time model (in state sweeps), fitted to per-pass device times of the n = 30 complex128
# Trotter / variational / grid passes (tools/variant_sweep.py, round 2): the longer of one sweep
# and 0.15 + (FP work per amplitude) / FP_PER_SWEEP (~75: B200 copy bandwidth over the FP64
# FMA rate at the ~0.75 the dense-gate passes reach; complex64 has twice the FP32 rate and half
# the bytes, so the same), and at least 1 + (runs - 5) / 4 for a tile of more than five runs of
# contiguous state bits (the rank-5 TMA box covers five; the rest become separate loads -- a
# tile of nine runs measured two sweeps)
FP_PER_SWEEP = float(os.environ.get("QSB_FP_PER_SWEEP", "75"))


MAX_TILE_RUNS = 5  # runs of contiguous state bits one rank-5 TMA box covers
# per-pass FP work caps (FMAs per amplitude) tried besides the greedy absorption, kept when the
# estimate prefers them (QSB_FP_BUDGETS, comma separated).  Measured (tools/budget_probe.py,
# n = 30 c128): a cap re-orders the greedy absorption -- the grid 3x10 in 34 passes at 128 and
# 32 at 192 instead of 36 (294 -> 291 / 279 ms), the windowed Trotter step in 13 passes at 192
# (130 -> 126 ms); caps below ~100 only add passes (variational 74 -> 78-81 ms)
FP_BUDGETS = tuple(float(x) for x in os.environ.get("QSB_FP_BUDGETS", "128,192").split(",") if x.strip())


def _tile_runs(tile_pos) -> int:
    runs, prev = 0, -2
    for p in sorted(tile_pos):
        if p != prev + 1:
            runs += 1
        prev = p
    return runs


def plan_estimate(plan: Plan) -> float:
    """Estimated time of a plan in state sweeps (see FP_PER_SWEEP); a stand-alone gate costs its
    touched fraction."""
    t = 0.0
    for st in plan.steps:
        if isinstance(st, PassStep):
            fp = sum(matrix_cost(g.matrix) for g in st.gates if g.kind in ("g1", "g2"))
            t += max(1.0 + max(0, _tile_runs(st.tile_pos) - MAX_TILE_RUNS) / 4.0, 0.15 + fp / FP_PER_SWEEP)
        else:
            t += st.gate.touched_fraction()
    return t


def _defer_trailing_diagonals(absorbed, deferred, budget):
    """Move the trailing diagonal gates of a pass beyond `budget` diagonals (latest first) to the
    head of the deferred list.  A trailing diagonal has no later gate of the pass acting
    non-diagonally on its qubits, and it commutes with every deferred gate that preceded it (the
    absorption rule), so running it at the start of the next passes is exact reordering."""
    diags = [i for i, g in enumerate(absorbed) if g.kind == "diag"]
    excess = len(diags) - budget
    if excess <= 0:
        return absorbed, deferred
    later_nondiag = 0
    move = set()
    for i in range(len(absorbed) - 1, -1, -1):
        g = absorbed[i]
        if g.kind == "diag":
            if not (g.smask & later_nondiag) and len(move) < excess:
                move.add(i)
        else:
            later_nondiag |= g.tmask
    if not move:
        return absorbed, deferred
    kept = [g for i, g in enumerate(absorbed) if i not in move]
    moved = [g for i, g in enumerate(absorbed) if i in move]
    return kept, moved + list(deferred)


def _plan_passes(plan, gates, n_qubits, dtype, geo, allow_ext_perm, diag_budget, max_runs=None, fp_budget=None,
                 estimate_only=False):
    """Greedy pass selection over `gates`.  estimate_only: passes carry their gates and tile but
    no program (enough for plan_estimate; plan_circuit compares variants that way and encodes
    only the one it keeps)."""
    remaining = gates
    while remaining:
        absorbed, deferred, T = _select_pass_best(remaining, n_qubits, geo, allow_ext_perm, max_runs, fp_budget)
        if diag_budget is not None:
            absorbed, deferred = _defer_trailing_diagonals(absorbed, deferred, diag_budget)
        if not absorbed:  # cannot happen with K >= L + 2, but never loop forever
            absorbed, deferred = [remaining[0]], remaining[1:]
            plan.steps.append(GateStep(absorbed[0]))
            remaining = deferred
            continue
        stand_alone = sum(g.touched_fraction() for g in absorbed)
        if stand_alone < 1.0:
            # cheaper as sparse single-gate kernels than as a full sweep
            plan.steps.extend(GateStep(g) for g in absorbed)
        elif estimate_only:
            plan.steps.append(PassStep(None, absorbed, tuple(sorted(T)), False, 0, 0))
        else:
            pgeo = geo
            if geo == GEOMETRY_JIT[dtype] and dtype in GEOMETRY_JIT_2Q and any(g.kind == "g2" for g in absorbed):
                code = sum(matrix_cost(g.matrix) for g in absorbed if g.kind in ("g1", "g2"))
                if code * GEOMETRY_JIT_2Q[dtype].A <= MAX_2Q_CODE:
                    pgeo = GEOMETRY_JIT_2Q[dtype]
                elif X2_BIG and dtype in GEOMETRY_JIT_2Q_X2:
                    pgeo = GEOMETRY_JIT_2Q_X2[dtype]
            words, info = compile_pass(absorbed, T, n_qubits, dtype, pgeo, minimal=MINIMAL_LAYOUT_CHANGES)
            used_geo = pgeo
            if (pgeo is GEOMETRY_JIT_2Q.get(dtype) and dtype == nat.QSB_C64 and X2_C64
                    and dtype in GEOMETRY_JIT_2Q_X2):
                # complex64: 256 x 32 at two CTAs per SM when it saves a layout change, or for the
                # heaviest passes (measured variational-30 c64: 32-gate pass 6.22 -> 5.72 ms,
                # a 16-gate pass with one layout change fewer 3.55 -> 3.24 ms).  Off by default:
                # at n = 18-24 whole variational layers fit one pass and ptxas needs minutes for
                # the 32-amplitude straight-line kernel (QSB_X2_C64=1 enables it)
                code = sum(matrix_cost(g.matrix) for g in absorbed if g.kind in ("g1", "g2"))
                w3, i3 = compile_pass(absorbed, T, n_qubits, dtype, GEOMETRY_JIT_2Q_X2[dtype],
                                      minimal=MINIMAL_LAYOUT_CHANGES)
                if i3["transposes"] < info["transposes"] or (i3["transposes"] == info["transposes"]
                                                             and code > SPLIT_MAX_CODE):
                    words, info, used_geo = w3, i3, GEOMETRY_JIT_2Q_X2[dtype]
            if pgeo is GEOMETRY_JIT_2Q.get(dtype) and dtype == nat.QSB_C64 and C64_WIDE_MIN_CODE > 0:
                # complex64: the default 256 x 32 (one CTA, two stages) for the heavier passes or
                # when it needs fewer layout changes (measured round 2, variational-30 c64: the
                # 96 / 128 FMA/amp passes 5.00 / 6.23 -> 4.72 / 5.76 ms, a 56 FMA/amp pass with
                # one layout change fewer 3.55 -> 3.21 ms; the 64 FMA/amp passes tie)
                # -- but never for the very large passes of mid-size circuits, whose 32-amplitude
                # straight-line kernels take ptxas minutes (the X2_C64 lesson)
                code = sum(matrix_cost(g.matrix) for g in absorbed if g.kind in ("g1", "g2"))
                if code <= C64_WIDE_MAX_CODE:
                    w4, i4 = compile_pass(absorbed, T, n_qubits, dtype, geo, minimal=MINIMAL_LAYOUT_CHANGES)
                    if i4["transposes"] < info["transposes"] or (code >= C64_WIDE_MIN_CODE
                                                                 and i4["transposes"] <= info["transposes"]):
                        words, info, used_geo = w4, i4, geo
            if pgeo is GEOMETRY_JIT_2Q.get(dtype) and dtype in GEOMETRY_JIT_2Q_SPLIT and SPLIT_2Q != "0":
                code = sum(matrix_cost(g.matrix) for g in absorbed if g.kind in ("g1", "g2"))
                chosen = False
                if SPLIT_2Q == "1" or code <= SPLIT_MAX_CODE:
                    w2, i2 = compile_pass(absorbed, T, n_qubits, dtype, GEOMETRY_JIT_2Q_SPLIT[dtype],
                                          minimal=MINIMAL_LAYOUT_CHANGES)
                    if SPLIT_2Q == "1" or i2["transposes"] <= info["transposes"]:
                        words, info, used_geo = w2, i2, GEOMETRY_JIT_2Q_SPLIT[dtype]
                        chosen = True
                if not chosen and dtype in GEOMETRY_JIT_2Q_X2 and X2_2Q:
                    # heavier passes: 256 consumers x 16 amplitudes at two CTAs per SM (half the
                    # straight-line code per thread, twice the warps) unless it needs more layout
                    # changes
                    w3, i3 = compile_pass(absorbed, T, n_qubits, dtype, GEOMETRY_JIT_2Q_X2[dtype],
                                          minimal=MINIMAL_LAYOUT_CHANGES)
                    if i3["transposes"] <= info["transposes"]:
                        words, info, used_geo = w3, i3, GEOMETRY_JIT_2Q_X2[dtype]
            plan.steps.append(PassStep(words, absorbed, tuple(sorted(T)), info["ext_perm"],
                                       info["transposes"], info["pivots"],
                                       tpl=(used_geo, info["mpos"], info["has_diag"])))
        remaining = deferred
    return plan


# ------------------------------------------------------------------------------------------
# compile one pass
# ------------------------------------------------------------------------------------------
def plan_expectation(terms, n_qubits: int, dtype: int, geometry: TileGeometry):
    """Read-only passes evaluating sum_t <psi|M_t|psi> for 1-/2-qubit terms [(bits, matrix)]
    (bits[0] = matrix MSB): terms are independent (nothing is written), so each pass takes every
    remaining term whose bits fit its tile; programs are flagged as expectation passes (the JIT
    kernel accumulates instead of storing).  Returns a list of program word arrays."""
    geo = geometry
    gates = []
    for i, (bits, m) in enumerate(terms):
        bits = tuple(int(b) for b in bits)
        kind = "g1" if len(bits) == 1 else "g2"
        gates.append(NGate(kind, bits, (), np.asarray(m, dtype=np.complex128), _bits(bits), _bits(bits), i))
    out = []
    remaining = gates
    while remaining:
        T = set(range(geo.L))
        absorbed, deferred = [], []
        for g in remaining:
            new = set(g.targets) - T
            if len(T) + len(new) <= geo.K:
                T |= new
                absorbed.append(g)
            else:
                deferred.append(g)
        for p in range(n_qubits):
            if len(T) >= geo.K:
                break
            T.add(p)
        words, _ = compile_pass(absorbed, T, n_qubits, dtype, geo, expect=True)
        out.append(words)
        remaining = deferred
    return out


class _Layout:
    def __init__(self, R, Tb):
        self.R = list(R)  # slot bit i <-> tile bit R[i]
        self.Tb = list(Tb)  # thread bit b <-> tile bit Tb[b] (0..4 lanes, 5..8 warps)

    def slot_of(self, tile_bit):
        return self.R.index(tile_bit)


def _order_thread_bits(cands, geo, prefer, natural=False):
    """Order the THREAD_BITS thread tile-bits: lanes first.  natural=True keeps tile bits 0..G-1 on
    lanes 0..G-1 (reads of the TMA stage are unswizzled)."""
    cands = sorted(cands)
    if natural:
        lanes = [b for b in range(geo.G)]
        rest = [b for b in cands if b not in lanes]
        rest.sort(key=lambda b: (b not in prefer, b))
        order = lanes + rest
        return order
    # lanes 0..G-1 with distinct residues mod G (conflict-free swizzled transposes)
    pri = sorted(cands, key=lambda b: (b not in prefer, b))
    lanes, used = [], set()
    for b in pri:
        if len(lanes) == geo.G:
            break
        if b % geo.G not in used:
            lanes.append(b)
            used.add(b % geo.G)
    for b in pri:
        if len(lanes) == geo.G:
            break
        if b not in lanes:
            lanes.append(b)
    rest = [b for b in pri if b not in lanes]
    return lanes + rest


# Minimal layout changes (swap only the needed bits; jit emits predicated transposes that move
# only the amplitudes whose swapped bits differ).  Measured round 1: slower on every workload
# (variational-30 c128 100 -> 146 ms, QFT-30 22.6 -> 23.6 ms) -- the kept lane assignment loses
# the conflict-free swizzle and predicated half-warp accesses save no wavefronts -- so off.
MINIMAL_LAYOUT_CHANGES = os.environ.get("QSB_MINIMAL_LAYOUT", "0") == "1"
# QSB_TMA_STORE_LAYOUT=1: final layouts chosen for conflict-free staging of the jit's bulk tensor
# stores instead of the coalesced-register-store rule.  Measured round 2 (QFT-30 pass 4): bank
# conflicts 162 M -> 33 M but shared-memory wavefronts 762 M -> 901 M, 5.07 -> 5.18 ms (c128)
# and 2.57 -> 2.84 ms (c64), so off by default
TMA_STORE_LAYOUT = os.environ.get("QSB_TMA_STORE_LAYOUT", "0") == "1"


# Gates of a pass are re-ordered within their dependencies so that each register layout serves as
# many gates as fit (QSB_REORDER=0: queue order).
REORDER_GATES = os.environ.get("QSB_REORDER", "1") != "0"
SEED_GATES = int(os.environ.get("QSB_REORDER_SEEDS", "6"))


def _event_bits(ev) -> int:
    m = 0
    if ev[0] == "diag":
        for pm, _pv, _w in ev[1]:
            m |= pm
        return m
    for p in tuple(ev[2]) + tuple(ev[3]):
        m |= 1 << p
    return m


def _reorder_events(events, tidx, nreg, first_forbid=frozenset()):
    """Dependency-respecting order of a pass's events that groups the gates sharing one register
    layout.  Two events depend on each other when their bit supports (targets, controls, diagonal
    masks) intersect, except two diagonal events, which commute.  Each round walks the remaining
    events in queue order: a gate joins the round when its target bits fit the round's register
    set (at most `nreg` tile bits; the first round may not use `first_forbid`) and nothing it
    depends on is left behind; skipped events hold back every later event on their bits
    (skipped diagonals hold back only gates)."""
    n_ev = len(events)
    bits = [_event_bits(ev) for ev in events]
    diag = [ev[0] == "diag" for ev in events]
    need = [None if diag[i] else frozenset(tidx[p] for p in events[i][2]) for i in range(n_ev)]
    remaining = list(range(n_ev))
    order = []
    first = True

    def walk(seed):
        R = set(seed)
        blocked_all = 0  # bits of skipped gates: later events on them wait
        blocked_gates = 0  # bits of skipped diagonals: later gates on them wait
        taken, left = [], []
        for i in remaining:
            if diag[i]:
                if bits[i] & blocked_all:
                    blocked_gates |= bits[i]
                    left.append(i)
                else:
                    taken.append(i)
                continue
            ok = not (bits[i] & (blocked_all | blocked_gates))
            if ok and first and need[i] & first_forbid:
                ok = False
            if ok and len(R | need[i]) > nreg:
                ok = False
            if ok:
                R |= need[i]
                taken.append(i)
            else:
                blocked_all |= bits[i]
                left.append(i)
        return taken, left

    while remaining:
        # seeds: the register bits of each of the first few gates that could run now; keep the
        # round that runs the most gates (ties: the earlier seed)
        best = walk(())
        seeds, seen, blk, blk_g = [], set(), 0, 0
        for i in remaining:
            if len(seeds) >= SEED_GATES:
                break
            if diag[i]:
                if bits[i] & blk:
                    blk_g |= bits[i]
                continue
            if not bits[i] & (blk | blk_g) and need[i] not in seen and not (first and need[i] & first_forbid):
                seeds.append(need[i])
                seen.add(need[i])
            blk |= bits[i]
        for seed in seeds:
            cand = walk(seed)
            if sum(not diag[i] for i in cand[0]) > sum(not diag[i] for i in best[0]):
                best = cand
        taken, left = best
        if first and not any(not diag[i] for i in taken) and left:
            first = False  # nothing fits the forbidden-free first layout: drop the restriction
        else:
            first = False
        order.extend(taken)
        remaining = left
    return [events[i] for i in order]


def compile_pass(absorbed, T, n, dtype, geo: TileGeometry | None = None, minimal: bool = False,
                 expect: bool = False):
    """Encode one pass.  `minimal`: layout changes swap only the needed bits (see
    MINIMAL_LAYOUT_CHANGES); otherwise every change re-lays the thread bits for a conflict-free
    swizzle and the coalesced store."""
    geo = geo or GEOMETRY[dtype]
    K, NREG, A = geo.K, geo.nreg, geo.A
    tile_pos = sorted(T)
    tidx = {p: b for b, p in enumerate(tile_pos)}
    ext_pos = [p for p in range(n) if p not in T]

    # ---- pass 1: physical mapping of every absorbed gate (relabels applied in order) ----
    loc = list(range(n))
    events = []  # ("diag", terms) | ("g1"/"g2", NGate, phys targets, phys controls)
    for g in absorbed:
        if g.kind == "swap":
            x, y = g.targets
            loc[x], loc[y] = loc[y], loc[x]
            continue
        if g.kind == "diag":
            terms = []
            for mask, val, w in diag_terms(g):
                pm = pv = 0
                for b in range(n):
                    if (mask >> b) & 1:
                        pm |= 1 << loc[b]
                        if (val >> b) & 1:
                            pv |= 1 << loc[b]
                terms.append((pm, pv, w))
            events.append(("diag", terms))
            continue
        pt = tuple(loc[t] for t in g.targets)
        pc = tuple(loc[c] for c in g.controls)
        events.append((g.kind, g, pt, pc))
    inv = [0] * n
    for x, p in enumerate(loc):
        inv[p] = x
    out_pos = [inv[p] for p in tile_pos]  # output global bit of each tile bit
    # tile counter order: external bits that land on the low (contiguous-run) output bits vary
    # fastest, so the tiles that together fill each output run are processed concurrently
    ext_pos.sort(key=lambda p: (inv[p] >= geo.L, p))
    ext_out = [inv[p] for p in ext_pos]
    ext_perm = ext_out != ext_pos
    store_bits = {b for b in range(K) if out_pos[b] < geo.L}

    if REORDER_GATES:
        events = _reorder_events(events, tidx, NREG, frozenset(range(geo.G)) if not geo.halves else frozenset())
    needs = [frozenset(tidx[p] for p in ev[2]) for ev in events if ev[0] in ("g1", "g2")]

    def pick_R(i, forbid=frozenset(), keep=None, must=(), sticky=()):
        """Register bits of the next layout: the tile bits of as many upcoming gates as fit.
        `must` bits are always included; with `keep` (split-tile geometry) the new layout
        shares at least one register bit with `keep` (transposes run in two halves on it)."""

        def greedy(cap):
            R = [b for b in must]
            j = i
            while j < len(needs):
                nd = needs[j]
                if nd & forbid:
                    break
                merged = set(R) | nd
                if len(merged) > cap:
                    break
                for b in sorted(nd):
                    if b not in R:
                        R.append(b)
                j += 1
            return R

        R = greedy(NREG)
        if keep is not None and not set(R) & set(keep):
            R = greedy(NREG - 1)
            if not set(R) & set(keep):
                R.append(sorted(keep, key=lambda b: (b in store_bits, -b))[0])
        filler = sorted((b for b in range(K) if b not in R and b not in forbid),
                        key=lambda b: (keep is not None and b not in keep, b not in sticky, b in store_bits, -b))
        for b in filler:
            if len(R) >= NREG:
                break
            R.append(b)
        return R

    words = []
    n_trans = 0

    def slot_offsets(bits):
        # offsets of all A slots: slot s = OR of bits[i] for the set bits i of s (built by doubling)
        offs = [0]
        for b in bits:
            v = 1 << b
            offs += [o | v for o in offs]
        return offs

    def layout_words(lay):
        w = [OP_LAYOUT, 0]
        w += lay.R
        w += lay.Tb
        w += slot_offsets([tile_pos[b] for b in lay.R])
        w += [tile_pos[b] for b in lay.Tb]
        w += slot_offsets([out_pos[b] for b in lay.R])
        w += [out_pos[b] for b in lay.Tb]
        w += slot_offsets(list(lay.R))
        w[1] = len(w)
        return w

    def make_layout(R, natural=False):
        cands = [b for b in range(K) if b not in R]
        return _Layout(R, _order_thread_bits(cands, geo, store_bits, natural))

    def change_layout(cur, R):
        """Minimal change from `cur` to register set R: every incoming tile bit takes the slot of
        an outgoing one and vice versa (other slots and thread positions unchanged), so the
        transpose only moves the amplitudes whose swapped bits differ (jit: predicated
        transposes).  Lane positions < G keep distinct residues mod G where possible."""
        incoming = [b for b in R if b not in cur.R]
        outgoing = [b for b in cur.R if b not in R]
        newR, newTb = list(cur.R), list(cur.Tb)
        # incoming bits in lane positions first, so outgoing store bits (which must end on lanes
        # for the coalesced store) can take lane positions
        incoming.sort(key=lambda x: cur.Tb.index(x))
        left = sorted(outgoing, key=lambda y: y not in store_bits)
        for x in incoming:
            j = cur.Tb.index(x)
            y = left[0]
            if j < geo.G and y not in store_bits:
                y = next((c for c in left if c % geo.G == x % geo.G), left[0])
            left.remove(y)
            newR[newR.index(y)] = x
            newTb[j] = y
        return _Layout(newR, newTb)

    # initial layout: its lanes 0..G-1 must be tile bits 0..G-1 (natural-order stage read)
    nat_forbid = frozenset(range(geo.G))
    R0 = pick_R(0, nat_forbid, must=(K - 1,) if geo.halves else ())
    cur = make_layout(R0, natural=True)
    words += layout_words(cur)

    pivot_count = 0
    pending_diag = []
    mpos = []  # (word index, gate, rows/columns exchanged) of every dense gate matrix

    def flush_diag():
        nonlocal pivot_count
        if not pending_diag:
            return
        ops, npiv = _compile_diag(pending_diag, cur, tile_pos, tidx, geo, pivot_count)
        pivot_count += npiv
        words.extend(ops)
        pending_diag.clear()

    gi = 0
    for ev in events:
        if ev[0] == "diag":
            pending_diag.extend(ev[1])
            continue
        kind, g, pt, pc = ev
        need = needs[gi]
        if not need <= set(cur.R):
            flush_diag()
            if geo.halves or geo.split:
                cur = make_layout(pick_R(gi, keep=cur.R))
            elif not minimal:
                cur = make_layout(pick_R(gi))
            else:
                cur = change_layout(cur, pick_R(gi, sticky=tuple(cur.R)))
            words += layout_words(cur)
            n_trans += 1
        flush_diag()
        op, swapped = _gate_op(kind, g, pt, pc, cur, tidx)
        mpos.append((len(words) + (8 if kind == "g1" else 9), g, swapped))
        words += op
        gi += 1
    flush_diag()
    # bulk tensor stores (jit: in-place passes without dense 2-qubit gates in the two-stage
    # geometry) write the tile through shared memory in the TMA image order of the output
    # positions: lanes 0..G-1 on the tile bits stored to output bits 0..G-1 make those writes
    # bank-conflict free; no other lane constraint (the bulk store is coalesced by construction)
    tma_store = (TMA_STORE_LAYOUT and not expect and not ext_perm and not geo.halves and not geo.split
                 and geo.thread_bits > 7 and not any(ev[0] == "g2" for ev in events))
    if tma_store:
        want = sorted((b for b in range(K) if out_pos[b] < geo.G), key=lambda b: out_pos[b])
        if set(cur.Tb[:geo.G]) != set(want):
            Rs = [b for b in cur.R if b not in want]
            for b in sorted(range(K), key=lambda b: -b):
                if len(Rs) >= NREG:
                    break
                if b not in Rs and b not in want:
                    Rs.append(b)
            rest = [b for b in range(K) if b not in Rs and b not in want]
            cur = _Layout(Rs, want + rest)
            words += layout_words(cur)
            n_trans += 1
    # store layout: lanes must cover the tile bits that land on the low output bits
    elif not expect and not store_bits <= set(cur.Tb[:5]):
        Rs = [b for b in cur.R if b not in store_bits]
        for b in sorted(range(K), key=lambda b: -b):
            if len(Rs) >= NREG:
                break
            if b not in Rs and b not in store_bits:
                Rs.append(b)
        if (geo.halves or geo.split) and not set(Rs) & set(cur.R):
            # split-tile transposes need a common register bit: go through an intermediate layout
            Rm = list(cur.R[:NREG // 2]) + [b for b in Rs if b not in cur.R][:NREG - NREG // 2]
            cur = make_layout(Rm)
            words += layout_words(cur)
            n_trans += 1
        cur = make_layout(Rs)
        words += layout_words(cur)
        n_trans += 1
    words.append(OP_END)
    words.append(2)

    header = [0] * H_TILEPOS
    header[0] = MAGIC
    header[1] = VERSION
    header[2] = K
    header[3] = NREG
    header[4] = n
    header[5] = dtype
    header[6] = 1 << (n - K)
    header[7] = ((1 if ext_perm else 0) | (2 if expect else 0) | (4 if geo.split else 0) | (8 if geo.pingpong else 0)
                 | (16 if geo.two_ctas else 0))
    contig = 0
    while contig < K and tile_pos[contig] == contig:
        contig += 1
    header[8] = contig
    header[9] = pivot_count
    prog = header + tile_pos + ext_pos + ext_out + words
    header_len = len(prog)
    prog[10] = header_len
    if len(prog) > MAX_PROG_WORDS or pivot_count > MAX_PIVOTS:
        raise _TooLarge()
    arr = np.array(prog, dtype=np.int64)
    base = len(prog) - len(words)
    return arr, {"ext_perm": ext_perm, "transposes": n_trans, "pivots": pivot_count,
                 "mpos": [(base + w, g, sw) for w, g, sw in mpos],
                 "has_diag": any(ev[0] == "diag" for ev in events)}


class _TooLarge(Exception):
    pass


def _matrix_words(m):
    out = []
    for v in np.asarray(m, dtype=np.complex128).reshape(-1):
        out.append(_f2w(v.real))
        out.append(_f2w(v.imag))
    return out


def _gate_op(kind, g, pt, pc, lay, tidx):
    """Program words of a dense gate, and whether its 4x4 was re-ordered (row / column bits
    exchanged so that row bit 1 is the higher register slot)."""
    gmask = rmask = 0
    swapped = False
    for c in pc:
        if c in tidx and tidx[c] in lay.R:
            rmask |= 1 << lay.slot_of(tidx[c])
        else:
            gmask |= 1 << c
    m = g.matrix
    if kind == "g1":
        ib = lay.slot_of(tidx[pt[0]])
        if np.array_equal(m, _XMAT):
            gk = G_SWAPX
        elif not np.any(m.imag):
            gk = G_REAL
        else:
            gk = G_COMPLEX
        w = [OP_G1, 0, ib, gk, gmask, gmask, rmask, rmask] + _matrix_words(m)
    else:
        i0 = lay.slot_of(tidx[pt[0]])
        i1 = lay.slot_of(tidx[pt[1]])
        if i0 > i1:
            ih, il, mm = i0, i1, m
        else:
            # exchange the two row/column bits so that row bit 1 <-> the higher slot
            ih, il, mm = i1, i0, m[np.ix_(_PERM2, _PERM2)]
            swapped = True
        gk = G_REAL if not np.any(mm.imag) else G_COMPLEX
        w = [OP_G2, 0, ih, il, gk, gmask, gmask, rmask, rmask] + _matrix_words(mm)
    w[1] = len(w)
    return w, swapped


def _compile_diag(terms, lay, tile_pos, tidx, geo, slot0):
    """Compile a commuting batch of diagonal terms (physical positions) for layout `lay`."""
    A = geo.A
    parity_single = 0
    parity_pairs = {}  # distance -> mask of the lower bits
    pairs = {}  # (a, b) a > b -> phase
    singles = {}  # bit -> phase
    generic = []
    for mask, val, w in terms:
        pc = bin(mask).count("1")
        if val == mask and pc <= 2:
            bits = [b for b in range(64) if (mask >> b) & 1]
            if w == -1.0:
                if pc == 1:
                    parity_single ^= mask
                else:
                    hi, lo = bits[1], bits[0]
                    parity_pairs[hi - lo] = parity_pairs.get(hi - lo, 0) ^ (1 << lo)
                continue
            if pc == 2:
                key = (bits[1], bits[0])
                pairs[key] = pairs.get(key, 1.0 + 0j) * w
                continue
            singles[bits[0]] = singles.get(bits[0], 1.0 + 0j) * w
            continue
        generic.append((mask, val, w))
    ops = []
    # pivots: greedy vertex cover of the pair graph, highest degree first
    adj = {}
    for (a, b), w in pairs.items():
        adj.setdefault(a, {})[b] = w
        adj.setdefault(b, {})[a] = w
    pivots = []
    while adj:
        p = max(adj, key=lambda q: (len(adj[q]), q in singles, -q))
        partners = adj.pop(p)
        for q in partners:
            adj[q].pop(p, None)
            if not adj[q]:
                del adj[q]
        pivots.append((p, partners))
    npiv = 0
    for p, partners in pivots:
        self_w = singles.pop(p, 1.0 + 0j)
        ops += _pivot_op(p, partners, self_w, lay, tile_pos, tidx, A, slot0 + npiv, geo.thread_bits)
        npiv += 1
    for b, w in singles.items():
        generic.append((1 << b, 1 << b, w))
    if parity_single or parity_pairs:
        w = [OP_PARITY, 0, parity_single, len(parity_pairs)]
        for d, m in sorted(parity_pairs.items()):
            w += [d, m]
        w[1] = len(w)
        ops += w
    for mask, val, ph in generic:
        ops += [OP_TERM, 6, mask, val, _f2w(ph.real), _f2w(ph.imag)]
    return ops, npiv


def _pivot_op(p, partners, self_w, lay, tile_pos, tidx, A, slot, thread_bits):
    if p in tidx and tidx[p] in lay.R:
        ptype, pval = 0, lay.slot_of(tidx[p])
    else:
        ptype, pval = 1, 1 << p
    ext = []
    ta = np.ones(16, dtype=np.complex128) * self_w
    tb = np.ones(1 << (thread_bits - 4), dtype=np.complex128)
    rt = np.ones(A, dtype=np.complex128)
    for q, w in sorted(partners.items()):
        if q not in tidx:
            ext.append((q, w))
            continue
        b = tidx[q]
        if b in lay.R:
            i = lay.slot_of(b)
            for s in range(A):
                if (s >> i) & 1:
                    rt[s] *= w
        else:
            tbit = lay.Tb.index(b)
            if tbit < 4:
                for u in range(16):
                    if (u >> tbit) & 1:
                        ta[u] *= w
            else:
                for u in range(len(tb)):
                    if (u >> (tbit - 4)) & 1:
                        tb[u] *= w
    use_rt = int(np.any(rt != 1.0))
    w = [OP_PIVOT, 0, slot, ptype, pval, use_rt, len(ext)]
    for q, ph in ext:
        w += [q, _f2w(ph.real), _f2w(ph.imag)]
    w += _matrix_words(ta) + _matrix_words(tb) + _matrix_words(rt)
    w[1] = len(w)
    return w
