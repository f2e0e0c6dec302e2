"""Pass specialisation: generate straight-line CUDA for one fused pass and compile it with NVRTC.

The interpreted pass kernel (csrc/pass.cu) dispatches ops at run time; ptxas then shuffles the
whole register-resident tile at every op (measured: ~38% of all instructions were register
moves).  Here the op list of a pass program (the same int64 word stream, fusion.py) becomes
C++ source: every amplitude is a named register, every gate an unrolled butterfly, every layout
change a transpose with compile-time slot offsets.  Gate coefficients (matrix entries, phases,
pivot tables) are NOT baked in: they are read from a per-launch coefficient array, so passes
with the same structure (e.g. every Trotter step) share one compiled kernel.  Kernels are
cached in-process by source text.
"""

from __future__ import annotations

import ctypes
import hashlib
import os
import struct
import threading

import numpy as np

from . import _native as nat

OP_END, OP_LAYOUT, OP_G1, OP_G2, OP_PIVOT, OP_PARITY, OP_TERM, OP_SCALE = range(8)
H_TILEPOS = 16
CONSUMERS = 512  # default (interpreter geometry); a kernel uses 2**(K - NREG) consumer threads
THREADS = CONSUMERS + 32
STAGES = 2
MAX_PIV = 32
# setmaxnreg split between the consumers and the 128-thread producer warpgroup.  setmaxnreg.inc
# can only take registers the CTA was launched with (threads x the launch-bound register count,
# a multiple of 8), or it waits forever: 384 threads launch with 168 each = 64,512 -> 256 x 232 +
# 128 x 40; 640 threads launch with 96 each = 61,440 -> 512 x 112 + 128 x 24.
def _reg_split(consumers: int, ctas: int = 1):
    threads = consumers + 128
    per = min(255, 65536 // (threads * ctas)) // 8 * 8
    pool = per * threads
    prod = 40 if (consumers <= 256 and not (consumers == 256 and ctas == 2)) else 24
    cons = min(248, (pool - 128 * prod) // consumers // 8 * 8)
    return cons, prod


def ctas_per_sm(consumers: int) -> int:
    """Resident CTAs per SM: 128-consumer kernels (32 KB tiles) run two per SM so one CTA's
    transposes / stores overlap the other's FP64 work."""
    return 2 if consumers <= 128 else 1


REG_SPLIT = {c: _reg_split(c, ctas_per_sm(c)) for c in (128, 256, 512)}

# Tiles per CTA (0 = persistent grid-stride loop).  Measured on the B200 (tools/probes/
# stream_probe.cu, 2^30 complex128 in place): a persistent one-CTA-per-SM sweep with a static
# tile split runs at 6.2-6.3 TB/s, while one-shot CTAs of 4 consecutive 64 KB tiles -- the grid
# covering the state once, the block scheduler handing out the next CTA to whichever SM
# finishes first -- reach 6.9 TB/s, the speed of the plain streaming kernels.
# Measured sweep at n = 30 (tools/tpc_sweep.sh, round 2): one-shot CTAs win on light passes
# (QFT pass 4: 5.97 -> 5.17 ms at 16 tiles per CTA) but lose on passes with heavy per-CTA
# set-up (pivot tables, pipeline ramp: QFT pass 1 5.76 -> 6.19 ms), so the default is a
# persistent grid that takes DYN_CHUNK consecutive tiles at a time from a global counter
# (dynamic balance without per-CTA restarts).  Expectation passes keep a static split: their
# per-CTA partial sums must not depend on timing.
TILES_PER_CTA = int(os.environ.get("QSB_TILES_PER_CTA", "16"))
PASS_SCHED = os.environ.get("QSB_PASS_SCHED", "dynamic")  # dynamic | oneshot | static
TMA_STORE = os.environ.get("QSB_TMA_STORE", "1") != "0"
# Immediate coefficient offsets (constant-bank operands, no per-op zero pin): complex64 passes
# (measured round 2: variational-30 c64 42.0 -> 38.0 ms, QFT-30 c64 11.0 -> 10.5 ms, no spills)
# and, with QSB_IMMEDIATE_C128=1, complex128 passes without dense 2-qubit gates (measured on the
# QFT-30 passes: 20.87 -> 20.95 ms, so off; the variational passes would spill 296 bytes)
IMMEDIATE_C64 = os.environ.get("QSB_IMMEDIATE_C64", "1") == "1"
IMMEDIATE_C128 = os.environ.get("QSB_IMMEDIATE_C128", "0") == "1"
DYN_CHUNK = int(os.environ.get("QSB_DYN_CHUNK", "2"))
# complex128 sign flips of a parity op as one three-input LOP3 per word (QSB_SIGN_LOP3=0: the
# shared AND mask + XOR form)
SIGN_LOP3 = os.environ.get("QSB_SIGN_LOP3", "1") != "0"


def tiles_per_cta(ext_bits: int, consumers: int) -> int:
    """TPC of a one-shot pass over 2**ext_bits tiles (0 when the state has too few tiles to
    matter)."""
    n_tiles = 1 << ext_bits
    if TILES_PER_CTA <= 0 or n_tiles < 4 * 148 * TILES_PER_CTA:
        return 0
    return TILES_PER_CTA


def pass_schedule(ext_bits: int, consumers: int, expect: bool, halves: bool):
    """(tpc, dyn_chunk) of a pass: dyn_chunk > 0 = persistent grid with a tile counter."""
    n_tiles = 1 << ext_bits
    if PASS_SCHED == "dynamic" and not expect and not halves and n_tiles >= 4 * 148 * max(1, DYN_CHUNK):
        return 0, max(1, DYN_CHUNK)
    if PASS_SCHED == "static":
        return 0, 0
    return tiles_per_cta(ext_bits, consumers), 0


def pass_grid(n_tiles: int, consumers: int, tpc: int, sms: int) -> int:
    if tpc:
        return -(-n_tiles // tpc)
    return min(n_tiles, sms * ctas_per_sm(consumers))


def _w2d(w):
    return struct.unpack("<d", struct.pack("<q", int(w)))[0]


class _Tagged(float):
    """A coefficient word read as a double, remembering its word position (recipe recording:
    arithmetic on it yields a plain float, which the recipe check below then catches)."""

    __slots__ = ("p",)

    def __new__(cls, value, pos):
        x = float.__new__(cls, value)
        x.p = pos
        return x


_PRELUDE = r"""
typedef unsigned long long u64;
typedef unsigned int u32;
typedef long long i64;
struct __align__(64) TMap { u64 w[16]; };
__device__ __forceinline__ u32 smem_u32(const void* p) { return (u32)__cvta_generic_to_shared(p); }
// hi ^ (s & 0x80000000) as one LOP3 (the parity ops' sign flips)
__device__ __forceinline__ u32 sgnx(u32 hi, u32 s) {
  u32 d;
  asm("lop3.b32 %0, %1, %2, %3, 0x78;" : "=r"(d) : "r"(hi), "r"(s), "r"(0x80000000u));
  return d;
}
__device__ __forceinline__ void mbar_init(u64* b, u32 c) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" :: "r"(smem_u32(b)), "r"(c)); }
__device__ __forceinline__ void mbar_expect_tx(u64* b, u32 n) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" :: "r"(smem_u32(b)), "r"(n) : "memory"); }
__device__ __forceinline__ void mbar_arrive(u64* b) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" :: "r"(smem_u32(b)) : "memory"); }
__device__ __forceinline__ void mbar_wait(u64* b, u32 par) {
  asm volatile("{\n\t.reg .pred P;\nW_%=:\n\tmbarrier.try_wait.parity.shared::cta.b64 P, [%0], %1;\n\t@!P bra W_%=;\n}"
               :: "r"(smem_u32(b)), "r"(par) : "memory"); }
__device__ __forceinline__ void tma5(void* d, const TMap* m, const int* c, u64* b) {
  asm volatile("cp.async.bulk.tensor.5d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4, %5, %6}], [%7];"
               :: "r"(smem_u32(d)), "l"((u64)m), "r"(c[0]), "r"(c[1]), "r"(c[2]), "r"(c[3]), "r"(c[4]), "r"(smem_u32(b)) : "memory"); }
__device__ __forceinline__ void tma5_store(const TMap* m, const int* c, const void* s) {
  asm volatile("cp.async.bulk.tensor.5d.global.shared::cta.bulk_group [%0, {%1, %2, %3, %4, %5}], [%6];"
               :: "l"((u64)m), "r"(c[0]), "r"(c[1]), "r"(c[2]), "r"(c[3]), "r"(c[4]), "r"(smem_u32(s)) : "memory"); }
__device__ __forceinline__ void bulk_commit() { asm volatile("cp.async.bulk.commit_group;" ::: "memory"); }
__device__ __forceinline__ void bulk_wait_read0() { asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory"); }
__device__ __forceinline__ void bulk_wait0() { asm volatile("cp.async.bulk.wait_group 0;" ::: "memory"); }
__device__ __forceinline__ void csync_all() { asm volatile("bar.sync 1, %0;" :: "n"(CONSUMERS) : "memory"); }
// ping-pong: barrier 1 + g syncs consumer group g; barrier 3 + g is group g's gate-math turn
__device__ __forceinline__ void csync_grp(int g) { asm volatile("bar.sync %0, %1;" :: "r"(1 + g), "n"(CONSUMERS) : "memory"); }
__device__ __forceinline__ void pp_sync(int g) { asm volatile("bar.sync %0, %1;" :: "r"(3 + g), "n"(2 * CONSUMERS) : "memory"); }
__device__ __forceinline__ void pp_arrive(int g) { asm volatile("bar.arrive %0, %1;" :: "r"(3 + g), "n"(2 * CONSUMERS) : "memory"); }
#if PINGPONG
#define csync() csync_grp(grp)
#else
#define csync() csync_all()
#endif
__device__ __forceinline__ void fence_async() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }
__device__ __forceinline__ C cm(C a, C b) { C r; r.x = a.x * b.x - a.y * b.y; r.y = a.x * b.y + a.y * b.x; return r; }
__device__ __forceinline__ double2 dm(double2 a, double2 b) {
  return make_double2(a.x * b.x - a.y * b.y, a.x * b.y + a.y * b.x); }
__device__ __forceinline__ double2 cfz(const double* cf, int k) { return make_double2(cf[k], cf[k + 1]); }
__device__ __forceinline__ C toC(double2 z) { C r; r.x = (R)z.x; r.y = (R)z.y; return r; }
struct CP { PR v[NCOEF]; };
__device__ __forceinline__ C mkC(R a, R b) { C r; r.x = a; r.y = b; return r; }
#if QSB_F32X2
// packed FP32 pairs (sm_100 FFMA2/FADD2): one instruction per complex64 component pair
__device__ __forceinline__ unsigned long long pk(float2 v) {
  unsigned long long r; asm("mov.b64 %0, {%1, %2};" : "=l"(r) : "f"(v.x), "f"(v.y)); return r; }
__device__ __forceinline__ float2 upk(unsigned long long v) {
  float2 r; asm("mov.b64 {%0, %1}, %2;" : "=f"(r.x), "=f"(r.y) : "l"(v)); return r; }
__device__ __forceinline__ float2 f2fma(float s, float2 x, float2 y) {  // s*x + y
  unsigned long long r; asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(r) : "l"(pk(make_float2(s, s))), "l"(pk(x)), "l"(pk(y)));
  return upk(r); }
__device__ __forceinline__ float2 f2mul(float s, float2 x) {
  unsigned long long r; asm("mul.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(pk(make_float2(s, s))), "l"(pk(x))); return upk(r); }
__device__ __forceinline__ float2 f2add(float2 x, float2 y) {
  unsigned long long r; asm("add.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(pk(x)), "l"(pk(y))); return upk(r); }
__device__ __forceinline__ float2 f2sub(float2 x, float2 y) {
  unsigned long long r; asm("sub.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(pk(x)), "l"(pk(y))); return upk(r); }
#endif
// coefficient reads are indexed by `zo` (always 0, re-read from shared memory before every op):
// ptxas can neither hoist them out of the tile loop nor bundle them across ops, so each op's
// coefficients occupy (uniform) registers only while that op runs
#define PZ(k) mkC(cp.v[(k) + ZO], cp.v[(k) + 1 + ZO])
#define PV(k) cp.v[(k) + ZO]
__device__ __forceinline__ int zpin(const u32* z) {
  u32 v; asm volatile("ld.shared.u32 %0, [%1];" : "=r"(v) : "r"(smem_u32(z))); return (int)(v & 1u); }
__device__ __forceinline__ u32 swz(u32 j) {
  u32 f = 0;
#pragma unroll
  for (int s = GB; s < HBB; s += GB) f ^= (j >> s);
  return j ^ (f & ((1u << GB) - 1u));
}
struct Smem { C stage[STAGES][1 << SBB]; C tbuf[ALIAS ? 1 : (1 << HBB)]; double2 ep[4][MAXPIV]; u64 full[STAGES]; u64 empty[STAGES]; u64 base[STAGES][2]; u32 zero; };
"""


MAX_TMA_ITER_BITS = 7  # at most 128 TMA calls per tile


def tma_plan(tile_pos, n, amp_bytes, max_iter=MAX_TMA_ITER_BITS):
    """Cover one tile (amplitudes whose index bits outside `tile_pos` are fixed) with rank-5
    TMA tensor loads.

    The state is described as a rank-5 tensor whose dims are contiguous ranges of index bits:
    a *box* dim spans only tile bits (box extent = dim extent), a *coordinate* dim has box
    extent 1 and its coordinate comes from the tile base.  Tile bits inside coordinate dims are
    *iterated*: one TMA call per combination.  A DP over the bit ranges picks the <= 5 dims that
    minimise the iterated bits (= log2 calls).  The stage then holds the tile in order
    [call index | box index] -- `sigma[b]` is the stage bit of tile bit b.

    Returns dict(dims=[(lo, nb, is_box)], iter_pos=[...], sigma=[...], tdesc=[15 ints]) or None.
    """
    tile = set(int(p) for p in tile_pos)
    epa = amp_bytes // 8  # 8-byte TMA elements per amplitude
    INF = (1 << 30, 0)
    # dp[d][p]: ((iterated bits, -innermost box width), back-pointer) covering bits [0, p) with d
    # dims; among equal call counts the widest innermost box (longest TMA rows) wins
    dp = [[(INF, None)] * (n + 1) for _ in range(6)]
    dp[0][0] = ((0, 0), None)
    tile_prefix = [0] * (n + 1)
    for p in range(n):
        tile_prefix[p + 1] = tile_prefix[p] + (1 if p in tile else 0)
    for d in range(5):
        for p in range(n):
            c0 = dp[d][p][0]
            if c0 >= INF:
                continue
            # box range: only tile bits, extent <= 256 elements
            lim = (8 if epa == 1 else 7) if d == 0 else 8
            w = 0
            while w < lim and p + w < n and (p + w) in tile:
                w += 1
                cand = ((c0[0], -w) if d == 0 else c0, (p, d, True))
                if cand[0] < dp[d + 1][p + w][0]:
                    dp[d + 1][p + w] = cand
            if d == 0:
                continue  # the innermost dim must be a (contiguous) box
            for w in range(1, min(31, n - p) + 1):
                cost = (c0[0] + tile_prefix[p + w] - tile_prefix[p], c0[1])
                if cost < dp[d + 1][p + w][0]:
                    dp[d + 1][p + w] = (cost, (p, d, False))
    best = min(range(1, 6), key=lambda d: (dp[d][n][0], d))
    if dp[best][n][0][0] > max_iter:
        return None
    dims = []
    p, d = n, best
    while d > 0:
        cost, bp = dp[d][p]
        lo, dprev, is_box = bp
        dims.append((lo, p - lo, is_box))
        p, d = lo, dprev
    dims.reverse()
    box_bits = [b for lo, nb, bx in dims if bx for b in range(lo, lo + nb)]
    iter_pos = [b for lo, nb, bx in dims if not bx for b in range(lo, lo + nb) if b in tile]
    order = sorted(int(p) for p in tile_pos)
    stage_of = {p: i for i, p in enumerate(box_bits)}
    stage_of.update({p: len(box_bits) + i for i, p in enumerate(iter_pos)})
    sigma = [stage_of[p] for p in order]
    gdim, gstride, box = [], [], []
    for i in range(5):
        if i < len(dims):
            lo, nb, bx = dims[i]
            ext = (1 << nb) * (epa if i == 0 else 1)
            gdim.append(ext)
            box.append(ext if bx else 1)
            if i > 0:
                gstride.append((1 << lo) * amp_bytes)
        else:
            gdim.append(1)
            box.append(1)
            gstride.append((1 << n) * amp_bytes)
    return dict(dims=dims, iter_pos=iter_pos, sigma=sigma, tdesc=[5] + gdim + gstride + box,
                box_amps=1 << len(box_bits))


def parity_quadratic(z: int, s1: int, pairs) -> int:
    """Q(z) = |z & s1| + sum_d |z & (z >> d) & m_d|  (mod 2): the sign bit of amplitude z under
    Z gates on the bits of s1 and CZ gates on the bit pairs (b, b + d), b in m_d."""
    t = bin(z & s1).count("1")
    for d, m in pairs:
        t += bin(z & (z >> d) & m).count("1")
    return t & 1


def parity_sign_plan(s1: int, pairs, goff, nreg: int):
    """Compile-time part of a parity op for one register layout: C = the slots' own signs
    Q(goff[s]) as a bit mask, and per register bit i the cross-term mask K_i (sign contribution
    |x & K_i| mod 2 of the runtime bits x) with M_i = the slots that have bit i.  At run time
    W = C ^ (Q(x) ? all : 0) ^ XOR_i (|x & K_i| odd ? M_i : 0); bit s of W is Q(x | goff[s])."""
    A = 1 << nreg
    C = sum(parity_quadratic(goff[sl], s1, pairs) << sl for sl in range(A))
    cross = []
    for i in range(nreg):
        p_i = goff[1 << i].bit_length() - 1
        K = 0
        for d, m in pairs:
            if (m >> p_i) & 1:
                K |= 1 << (p_i + d)
            if p_i >= d and (m >> (p_i - d)) & 1:
                K |= 1 << (p_i - d)
        if K:
            cross.append((K, sum(1 << sl for sl in range(A) if (sl >> i) & 1)))
    return C, cross


class _Gen:
    def __init__(self, words, dtype):
        self.w = [int(x) for x in words]
        self.dtype = dtype
        w = self.w
        self.K, self.NREG, self.n = w[2], w[3], w[4]
        self.TB = self.K - self.NREG
        self.A = 1 << self.NREG
        self.consumers = 1 << self.TB
        self.G = 3 if dtype == nat.QSB_C128 else 4
        n, K = self.n, self.K
        self.tile_pos = w[H_TILEPOS:H_TILEPOS + K]
        self.ext_pos = w[H_TILEPOS + K:H_TILEPOS + n]
        self.ext_out = w[H_TILEPOS + n:H_TILEPOS + 2 * n - K]
        self.ext_perm = bool(w[7] & 1)
        self.expect = bool(w[7] & 2)  # read-only expectation pass: accumulate, never store
        self.ops0 = H_TILEPOS + 2 * n - K
        self.coeffs: list = []
        self.tables: list = []
        self.lines: list = []
        self.ep_waited = False
        self.h_scale = 0  # deferred 1/sqrt(2) factors of uncontrolled Hadamard butterflies
        self.vm = list(range(self.A))  # slot of the current layout -> register variable v<i>
        self.n_cops = 0  # ops with coefficient reads emitted so far
        # coefficient-only mode (structure templates): no source text, only the parameter /
        # table vectors, the word positions read as doubles and the value-dependent structure
        # decisions (entry classes, Hadamard detection, unit pivot factors) -- together with
        # the other words they determine the source exactly (compile_words' template cache)
        self.quiet = False
        self.dpos: set = set()
        self.trace: list = []
        # recipe recording (coefficient_recipe): the word position each coefficient is read
        # from (-1: a constant of the structure)
        self.record = False
        self.csrc: list = []
        self.tsrc: list = []
        amp_bytes = 16 if dtype == nat.QSB_C128 else 8
        # 128 KB tiles are staged as two 64 KB halves split on tile bit K-1 (a register bit of
        # the first layout); layout changes then run in two rounds through a 64 KB buffer
        self.halves = (1 << K) * amp_bytes > 65536
        # split: one 64 KB stage released as soon as the tile is in registers and a separate
        # 32 KB transpose buffer (two-round layout changes), two CTAs per SM
        self.split = bool(w[7] & 4) and not self.halves
        # ping-pong: two consumer groups of CONSUMERS threads in one CTA, each with its own
        # stage (doubling as its transpose buffer), taking alternate tiles; a pair of named
        # barriers hands the gate-math turn back and forth, so one group's FP work always
        # overlaps the other's tile load / stores instead of both computing (and both waiting)
        # at the same time as two independent CTAs drift into doing
        self.pingpong = bool(w[7] & 8) and not self.halves and not self.split
        self.groups = 2 if self.pingpong else 1
        # resident CTAs per SM: 2 for 128-consumer kernels, or (header flag 16) for 256 consumers
        self.ctas = 1 if self.pingpong else (2 if (ctas_per_sm(self.consumers) == 2 or (w[7] & 16)) else 1)
        self.regs = _reg_split(self.consumers * self.groups, self.ctas)
        # two CTAs per SM with 64 KB tiles: one stage per CTA, reused as the transpose buffer
        self.alias = (not self.halves and not self.split and (self.ctas == 2 or self.pingpong)
                      and (1 << K) * amp_bytes == 65536)
        # split geometry: one stage per CTA at two CTAs per SM; three stages (3 x 64 KB + the
        # 32 KB transpose buffer) at one CTA per SM
        self.stages = 2 if self.pingpong else (1 if self.alias else (split_stages(self.consumers) if self.split else STAGES))
        self.sched = pass_schedule(self.n - K, self.consumers, self.expect, self.halves)
        self.HB = K - 1 if (self.halves or self.split) else K  # bits of a transpose-buffer index
        self.SB = K - 1 if self.halves else K  # bits of a stage index
        # bulk tensor stores through the transpose buffer (2-stage geometry) for passes without
        # dense two-qubit gates: measured (round 2, n = 30) QFT c128 21.6 -> 20.9 ms, c64 11.5 ->
        # 11.0 ms, but passes with dense 2-qubit gates in this geometry got slower (variational
        # c64 44.4 -> 46.0 ms, grid c128 300 -> 308 ms): their FP work already hides the store
        # back-pressure and the extra staging costs shared memory bandwidth.  Out-of-place
        # passes store through a second tensor map over the destination.  QSB_TMA_STORE=0
        # disables it.
        ops = []
        q = self.ops0
        while w[q] != OP_END:
            ops.append(w[q])
            q += w[q + 1]
        self.tma_store_ok = (TMA_STORE and not (self.halves or self.split or self.alias or self.expect)
                             and OP_G2 not in ops)
        # the bulk-store path needs the transpose buffer free of an in-flight store before a
        # layout change writes it (set once the store plan is known, see the store section)
        self.tma_store = self.tma_store_ok
        self.oplan = None
        self.immediate = (IMMEDIATE_C64 if dtype == nat.QSB_C64
                          else (IMMEDIATE_C128 and OP_G2 not in ops and not self.expect))
        self.uses_tma_store = False

    # uniform coefficients (gate matrices, phases): a kernel-parameter array of R, read as
    # constant-bank operands (no registers held across the tile); returns the first index
    def cf(self, values):
        k = len(self.coeffs)
        if self.record:
            self.csrc.extend(v.p if type(v) is _Tagged else -1 for v in values)
        self.coeffs.extend(float(v) for v in values)
        return k

    # per-thread-indexed tables (pivot factor tables): doubles staged in shared memory
    def tf(self, values):
        k = len(self.tables)
        if self.record:
            self.tsrc.extend(v.p if type(v) is _Tagged else -1 for v in values)
        self.tables.extend(float(v) for v in values)
        return k

    def emit(self, s):
        if not self.quiet:
            self.lines.append(s)

    def d(self, i):
        """Word i read as a double (a coefficient: recorded for the structure key)."""
        self.dpos.add(i)
        if self.record:
            return _Tagged(_w2d(self.w[i]), i)
        return _w2d(self.w[i])

    # ---- layouts ------------------------------------------------------------------------
    def parse_layout(self, a):
        w, NREG, TB, A = self.w, self.NREG, self.TB, self.A
        R = w[a:a + NREG]
        Tb = w[a + NREG:a + NREG + TB]
        goff = w[a + NREG + TB:a + NREG + TB + A]
        gpos = w[a + NREG + TB + A:a + NREG + 2 * TB + A]
        ooff = w[a + NREG + 2 * TB + A:a + NREG + 2 * TB + 2 * A]
        opos = w[a + NREG + 2 * TB + 2 * A:a + NREG + 3 * TB + 2 * A]
        jt = w[a + NREG + 3 * TB + 2 * A:a + NREG + 3 * TB + 3 * A]
        return dict(R=R, Tb=Tb, goff=goff, gpos=gpos, ooff=ooff, opos=opos, jt=jt)

    def swz_const(self, j):
        f = 0
        s = self.G
        while s < self.HB:
            f ^= j >> s
            s += self.G
        return j ^ (f & ((1 << self.G) - 1))

    def thread_expr(self, positions, width):
        """OR of ((tid >> i) & 1) << positions[i]  as a C expression of `width` bits."""
        parts = []
        for i, p in enumerate(positions):
            if width == 64:
                parts.append(f"((u64)((tid >> {i}) & 1) << {p})")
            else:
                parts.append(f"(((u32)tid >> {i} & 1u) << {p})")
        return " | ".join(parts) if parts else "0"

    def set_layout(self, lay, idx):
        self.emit(f"    const u32 jt{idx} = {self.thread_expr(lay['Tb'], 32)};")
        self.emit(f"    const u64 gt{idx} = {self.thread_expr(lay['gpos'], 64)};")
        self.lay = lay
        self.li = idx

    # ---- generation ---------------------------------------------------------------------
    def generate(self, name):
        w = self.w
        A = self.A
        p = self.ops0
        assert w[p] == OP_LAYOUT
        first = self.parse_layout(p + 2)
        # pivots (per-tile external factors)
        piv_ops = []
        q = p
        while w[q] != OP_END:
            if w[q] == OP_PIVOT:
                piv_ops.append(q)
            q += w[q + 1]
        self.npiv = len(piv_ops)
        # external pivot factors: producer lane p computes pivot p's product over the partner
        # bits outside the tile (per tile, one stage ahead of the consumers)
        ep = []
        if piv_ops:
            # per-pivot partner tables in the coefficient array: [count, bits..., (re, im)...];
            # lane p walks pivot p's table in a uniform loop (no divergent per-lane code paths)
            tables = []
            maxn = 1
            for q in piv_ops:
                a = q + 2
                slot, ne = w[a], w[a + 4]
                maxn = max(maxn, ne)
                tables.append((slot, ne, a))
            offs = [0] * len(tables)
            for slot, ne, a in tables:
                vals = [float(ne)] + [float(w[a + 5 + 3 * k]) for k in range(ne)]
                for k in range(ne):
                    vals += [self.d(a + 6 + 3 * k), self.d(a + 7 + 3 * k)]
                offs[slot] = self.tf(vals)
            offtab = self.tf([float(o) for o in offs])
            ep.append("        if (lane < NPIV) {")
            ep.append(f"          const int o = (int)scf[{offtab} + lane];")
            ep.append("          const int cnt = (int)scf[o];")
            ep.append("          double2 f = make_double2(1.0, 0.0);")
            ep.append(f"          for (int k = 0; k < cnt; ++k) {{")
            ep.append("            const int bit = (int)scf[o + 1 + k];")
            ep.append("            if ((base >> bit) & 1ull) f = dm(f, cfz(scf, o + 1 + cnt + 2 * k));")
            ep.append("          }")
            ep.append("          sm.ep[tno & 3][lane] = f;")
            ep.append("        }")
        self.ep_code = "\n".join(ep)
        body_start = len(self.lines)
        # initial load: the TMA stage holds tile bit b at stage bit sigma[b] (tma_plan)
        amp_bytes = 16 if self.dtype == nat.QSB_C128 else 8
        stage_pos = self.tile_pos[:self.SB]
        self.tplan = tma_plan(stage_pos, self.n, amp_bytes)
        if self.tplan is None:
            raise ValueError("tile has too many bit runs for the TMA tile fetch")
        sig = self.tplan["sigma"]
        self.set_layout(first, 0)
        self.emit(f"    const u32 sg0 = {self.thread_expr([sig[b] for b in first['Tb']], 32)};")
        if not self.halves:
            for s in range(A):
                off = sum(1 << sig[first['R'][i]] for i in range(self.NREG) if (s >> i) & 1)
                self.emit(f"    C v{s} = buf[sg0 | {off}u];")
            # the stage is consumed: hand it back to the producer before any compute
            if self.alias:
                self.emit("@@RELEASE@@")  # the stage doubles as the transpose buffer: release at tile end
            else:
                self.emit("    fence_async();")
                self.emit("    mbar_arrive(&sm.empty[s]);")
        else:
            ih = first['R'].index(self.K - 1)
            self.emit(f"    C {', '.join(f'v{s}' for s in range(A))};")
            for half in (0, 1):
                if half:
                    self.emit("    mbar_wait(&sm.full[1], it & 1);")
                for s in range(A):
                    if ((s >> ih) & 1) != half:
                        continue
                    off = sum(1 << sig[first['R'][i]] for i in range(self.NREG) if (s >> i) & 1 and i != ih)
                    self.emit(f"    v{s} = sm.stage[{half}][sg0 | {off}u];")
                self.emit("    fence_async();")
                self.emit(f"    mbar_arrive(&sm.empty[{half}]);")
        self.emit("@@REFILL@@")
        q = p + w[p + 1]
        li = 0
        while w[q] != OP_END:
            op, ln = w[q], w[q + 1]
            a = q + 2
            if op == OP_LAYOUT and _PROBE == "notransposes":
                # timing probe only: relabel without moving data (results are wrong)
                new = self.parse_layout(a)
                li += 1
                self.set_layout(new, li)
            elif op == OP_LAYOUT and self.quiet:
                li += 1
                self.lay = self.parse_layout(a)  # layout changes carry no coefficients
                self.li = li
            elif op == OP_LAYOUT:
                new = self.parse_layout(a)
                li += 1
                pairs = None if (self.halves or self.split or not _MINIMAL) else self.swap_pairs(self.lay, new)
                if pairs:
                    self.gen_predicated_transpose(new, li, pairs)
                elif not (self.halves or self.split):
                    if self.tma_store:
                        self.emit("    if (tid < 32) bulk_wait_read0();  // the last tile's store has read tbuf")
                    self.emit("    csync();")
                    self.emit("    { const u32 sj = swz(jt%d);" % self.li)
                    for s in range(A):
                        self.emit(f"      TBUF[sj ^ {self.swz_const(self.lay['jt'][s])}u] = v{self.vm[s]};")
                    self.emit("    }")
                    self.emit("    csync();")
                    self.set_layout(new, li)
                    self.emit("    { const u32 sj = swz(jt%d);" % li)
                    for s in range(A):
                        self.emit(f"      v{self.vm[s]} = TBUF[sj ^ {self.swz_const(new['jt'][s])}u];")
                    self.emit("    }")
                else:
                    self.gen_split_transpose(new, li)
            elif op == OP_PARITY:
                self.gen_parity(a)
            elif _PROBE == "nogates":
                pass  # timing probe only: gate bodies omitted (results are wrong)
            else:
                gen = {OP_G1: self.gen_g1, OP_G2: self.gen_g2, OP_PIVOT: self.gen_pivot, OP_TERM: self.gen_term,
                       OP_SCALE: self.gen_scale}[op]
                if self.expect and op in (OP_G1, OP_G2):
                    gen = lambda a_, op_=op: self.gen_expect(a_, op_)  # noqa: E731
                # this op's coefficient reads are indexed by zo<k>; zo<k+1> is loaded now so the
                # next op's coefficients can be fetched while this op computes
                k = self.n_cops
                if self.immediate:
                    # immediate coefficient offsets (constant-bank operands); the zero-pin
                    # guard below keeps ptxas from hoisting every coefficient into registers
                    self.emit("#define ZO 0")
                else:
                    if k == 0:
                        self.emit("    const int zo0 = zpin(&sm.zero);")
                    self.emit(f"    const int zo{k + 1} = zpin(&sm.zero);")
                    self.emit(f"#define ZO zo{k}")
                gen(a)
                self.emit("#undef ZO")
                self.n_cops += 1
            q += ln
        if self.quiet:
            return ""
        body = "\n".join(self.lines[body_start:])
        if self.expect:
            return self._kernel(name, body, "")
        # output offsets of the final layout
        lay = self.lay
        store = []
        if self.h_scale:
            k = self.h_scale
            scale = 2.0 ** (-(k // 2)) * (0.7071067811865476 if k % 2 else 1.0)
            store.append(f"    const R hs = (R){scale!r};")
            for s in range(A):
                store.append(f"    v{self.vm[s]}.x *= hs; v{self.vm[s]}.y *= hs;")
        # output global position of every tile bit of the final layout
        out_of = {b: p for b, p in zip(lay['Tb'], lay['opos'])}
        for i, b in enumerate(lay['R']):
            out_of[b] = lay['ooff'][1 << i].bit_length() - 1
        tpos = list(self.tile_pos)
        opos = sorted(out_of.values())
        if self.tma_store_ok:
            if opos == sorted(tpos):
                self.oplan = self.tplan  # the tile lands on its own positions: one tensor map
            else:
                # out of place, tile bits landing on other positions (SWAPs across the tile
                # boundary): a second tensor map over the destination, planned for the output
                # positions
                amp_bytes = 16 if self.dtype == nat.QSB_C128 else 8
                self.oplan = tma_plan(opos, self.n, amp_bytes)
        if self.oplan is not None:
            # the tile goes back through the transpose buffer in the TMA image order of its
            # OUTPUT positions and one warp issues bulk tensor stores, so the consumers never
            # wait for HBM write back-pressure
            sig = self.oplan["sigma"]
            img = {b: sig[opos.index(out_of[b])] for b in out_of}
            so = self.thread_expr([img[b] for b in lay['Tb']], 32)
            store.append("    if (tid < 32) bulk_wait_read0();")
            store.append("    csync();")
            store.append(f"    {{ const u32 so = {so};")
            for s in range(A):
                off = sum(1 << img[lay['R'][i]] for i in range(self.NREG) if (s >> i) & 1)
                store.append(f"      sm.tbuf[so | {off}u] = v{self.vm[s]};")
            store.append("    }")
            store.append("    fence_async();")
            store.append("    csync();")
            store.append("@@TMASTORE@@")
            self.uses_tma_store = True
            return self._kernel(name, body, "\n".join(store))
        store.append(f"    const u64 ot = obase | {self.thread_expr(lay['opos'], 64)};")
        for s in range(A):
            if _PROBE == "nostores":  # timing probe: keep the values live, store (almost) nothing
                store.append(f"    if (v{self.vm[s]}.x == (R)1234.5) dst[ot | {lay['ooff'][s]}ull] = v{self.vm[s]};")
            else:
                store.append(f"    dst[ot | {lay['ooff'][s]}ull] = v{self.vm[s]};")
        return self._kernel(name, body, "\n".join(store))

    def gen_expect(self, a, op):
        """Accumulate Re <x| M |x> over this op's pairs / quads (expectation pass).  Per group:
        sum_r Re(M_rr) |x_r|^2 + sum_{r<c} (Re M_rc + Re M_cr) Re z + (Im M_cr - Im M_rc) Im z
        with z = conj(x_r) x_c -- exact for any M, zero pairs skipped, in double precision."""
        w, A = self.w, self.A
        if op == OP_G1:
            slots_bits = [w[a]]
            m = [self.d(i) for i in range(a + 6, a + 14)]
            d = 2
        else:
            slots_bits = [w[a], w[a + 1]]  # ih, il
            m = [self.d(i) for i in range(a + 7, a + 39)]
            d = 4
        M = [[complex(m[2 * (r * d + c)], m[2 * (r * d + c) + 1]) for c in range(d)] for r in range(d)]
        diag = [(r, M[r][r].real) for r in range(d) if M[r][r].real != 0.0]
        offs = []
        for r in range(d):
            for c in range(r + 1, d):
                ar = M[r][c].real + M[c][r].real
                bi = M[c][r].imag - M[r][c].imag
                if ar != 0.0 or bi != 0.0:
                    offs.append((r, c, ar, bi))
        self.trace.append(("expect", tuple(r for r, _ in diag), tuple((r, c, ar != 0.0, bi != 0.0) for r, c, ar, bi in offs)))
        dci = self.cf([v for _, v in diag]) if diag else 0
        oci = self.cf([x for _, _, ar, bi in offs for x in (ar, bi)]) if offs else 0
        if self.quiet:
            return
        mask = sum(1 << b for b in slots_bits)
        self.emit(f"    {{ // expectation term on slot bits {slots_bits}")
        for s in range(A):
            if s & mask:
                continue
            if d == 2:
                idx = [s, s | (1 << slots_bits[0])]
            else:
                ih, il = slots_bits
                idx = [s, s | (1 << il), s | (1 << ih), s | (1 << ih) | (1 << il)]
            xs = [f"v{self.vm[i]}" for i in idx]
            self.emit("      { " + " ".join(f"const double r{c} = (double){xs[c]}.x, i{c} = (double){xs[c]}.y;"
                                          for c in range(d)))
            for k, (r, _) in enumerate(diag):
                self.emit(f"        ea = fma(PV({dci + k}), fma(r{r}, r{r}, i{r} * i{r}), ea);")
            for k, (r, c, ar, bi) in enumerate(offs):
                # real (imaginary) coupling only: the other half of z is never formed
                if ar != 0.0:
                    self.emit(f"        ea = fma(PV({oci + 2 * k}), fma(r{r}, r{c}, i{r} * i{c}), ea);")
                if bi != 0.0:
                    self.emit(f"        ea = fma(PV({oci + 2 * k + 1}), fma(r{r}, i{c}, -(i{r} * r{c})), ea);")
            self.emit("      }")
        self.emit("    }")

    def gen_scale(self, a):
        ci = self.cf([self.d(a), self.d(a + 1)])
        if self.quiet:
            return
        self.emit(f"    {{ const C ph = PZ({ci});")
        for s in range(self.A):
            self.emit(f"      v{self.vm[s]} = cm(v{self.vm[s]}, ph);")
        self.emit("    }")

    def swap_pairs(self, old, new):
        """[(slot i, thread position j)] when `new` differs from `old` only by exchanging register
        slot i's tile bit with thread position j's (fusion.compile_pass change_layout), else None."""
        pairs = []
        for i in range(self.NREG):
            if new['R'][i] == old['R'][i]:
                continue
            if new['R'][i] not in old['Tb']:
                return None
            j = old['Tb'].index(new['R'][i])
            if new['Tb'][j] != old['R'][i]:
                return None
            pairs.append((i, j))
        for j in range(self.TB):
            if new['Tb'][j] != old['Tb'][j] and not any(j == jj for _, jj in pairs):
                return None
        return pairs or None

    def gen_predicated_transpose(self, new, li, pairs):
        """Layout change that exchanges register slots with thread positions: an amplitude whose
        swapped slot bits equal the thread's swapped thread bits stays in its register, so only
        the others go through shared memory (1 pair: half, 2 pairs: 3/4 of the tile)."""
        A = self.A
        old = self.lay
        tp = " | ".join(f"((((u32)tid >> {j}) & 1u) << {p})" for p, (_, j) in enumerate(pairs))

        def pat(s):
            return sum(((s >> i) & 1) << p for p, (i, _) in enumerate(pairs))

        self.emit("    csync();")
        self.emit(f"    const u32 tp{li} = {tp};")
        self.emit("    { const u32 sj = swz(jt%d);" % self.li)
        for s in range(A):
            self.emit(f"      if (tp{li} != {pat(s)}u) TBUF[sj ^ {self.swz_const(old['jt'][s])}u] = v{self.vm[s]};")
        self.emit("    }")
        self.emit("    csync();")
        self.set_layout(new, li)
        self.emit("    { const u32 sj = swz(jt%d);" % li)
        for s in range(A):
            self.emit(f"      if (tp{li} != {pat(s)}u) v{self.vm[s]} = TBUF[sj ^ {self.swz_const(new['jt'][s])}u];")
        self.emit("    }")

    def gen_split_transpose(self, new, li):
        """Layout change through the 64 KB buffer in two rounds: round r moves the amplitudes
        whose tile bit h (a register bit of both layouts) is r.  Buffer index = tile index with
        bit h removed; the register variables of round r are reused for the same round's
        reads (slot -> variable map), so no temporaries are needed."""
        old = self.lay
        A, G = self.A, self.G
        common = [b for b in old['R'] if b in new['R']]
        assert common, "split transposes need a common register bit"

        def squeeze(p, h):
            return p - 1 if p > h else p

        def ok(h, Tb):
            res = {squeeze(b, h) % G for b in Tb[:G]}
            return len(res) == G

        h = sorted(common, key=lambda b: (not (ok(b, old['Tb']) and ok(b, new['Tb'])), b))[0]
        io, inew = old['R'].index(h), new['R'].index(h)

        def slot_index(R, s):
            j = 0
            for i, b in enumerate(R):
                if (s >> i) & 1 and b != h:
                    j |= 1 << squeeze(b, h)
            return j

        jw = self.thread_expr([squeeze(b, h) for b in old['Tb']], 32)
        jr = self.thread_expr([squeeze(b, h) for b in new['Tb']], 32)
        nvm = [0] * A
        for r in (0, 1):
            olds = [s for s in range(A) if ((s >> io) & 1) == r]
            news = [s for s in range(A) if ((s >> inew) & 1) == r]
            for s_new, s_old in zip(news, olds):
                nvm[s_new] = self.vm[s_old]
            self.emit("    csync();")
            self.emit(f"    {{ const u32 sj = swz({jw});")
            for s in olds:
                self.emit(f"      TBUF[sj ^ {self.swz_const(slot_index(old['R'], s))}u] = v{self.vm[s]};")
            self.emit("    }")
            self.emit("    csync();")
            self.emit(f"    {{ const u32 sj = swz({jr});")
            for s in news:
                self.emit(f"      v{nvm[s]} = TBUF[sj ^ {self.swz_const(slot_index(new['R'], s))}u];")
            self.emit("    }")
        self.vm = nvm
        self.set_layout(new, li)

    def gen_g1(self, a):
        w, A = self.w, self.A
        ib, kind, gmask, gval, rmask, rval = w[a:a + 6]
        m = [self.d(i) for i in range(a + 6, a + 14)]
        hh = 0.7071067811865475
        is_h = (kind == 1 and not gmask and not rmask and m[0] == hh and m[2] == hh and m[4] == hh and m[6] == -hh
                and not any(m[1::2]))
        self.trace.append(("h", is_h))
        if is_h:
            # uncontrolled Hadamard: sum/difference butterfly, the 1/sqrt(2) is applied once at the store
            self.h_scale += 1
            if self.quiet:
                return
            self.emit(f"    {{ // H butterfly slot bit {ib}")
            for s in range(A):
                if s & (1 << ib):
                    continue
                t = s | (1 << ib)
                if self.dtype == nat.QSB_C64:
                    self.emit(f"      {{ const C x0 = v{self.vm[s]}, x1 = v{self.vm[t]}; v{self.vm[s]} = f2add(x0, x1);"
                              f" v{self.vm[t]} = f2sub(x0, x1); }}")
                    continue
                self.emit(f"      {{ const C x0 = v{self.vm[s]}, x1 = v{self.vm[t]}; v{self.vm[s]}.x = x0.x + x1.x; v{self.vm[s]}.y = x0.y + x1.y;"
                          f" v{self.vm[t]}.x = x0.x - x1.x; v{self.vm[t]}.y = x0.y - x1.y; }}")
            self.emit("    }")
            return
        self.emit(f"    {{ // G1 slot bit {ib}")
        if gmask:
            self.emit(f"    if (((base | gt{self.li}) & {gmask}ull) == {gval}ull) {{")
        if kind == 2:
            for s in range(A):
                if s & (1 << ib) or (s & rmask) != rval:
                    continue
                t = s | (1 << ib)
                self.emit(f"      {{ const C x = v{self.vm[s]}; v{self.vm[s]} = v{self.vm[t]}; v{self.vm[t]} = x; }}")
        else:
            mat = [complex(m[2 * k], m[2 * k + 1]) for k in range(4)]
            coef = self.matrix_coeffs(mat, 2, m)
            for s in range(A):
                if s & (1 << ib) or (s & rmask) != rval:
                    continue
                self.emit_matvec(coef, [s, s | (1 << ib)])
        if gmask:
            self.emit("    }")
        self.emit("    }")

    def matrix_coeffs(self, mat, d, parts=None):
        """Per-entry structure of a d x d gate matrix: ('z',) exact zero (skipped), ('1',)/('-1',)
        exact +-1 (no multiply), ('r', k) real, ('i', k) imaginary, ('c', k) complex -- k indexes
        the parameter array.  The structure is part of the kernel source (so e.g. every fSim or
        every Trotter ZZ+X term shares one kernel), the values are runtime coefficients."""
        out = []
        for k, z in enumerate(mat):
            # the real / imaginary words themselves when given (recipe recording keeps their positions)
            re, im = (parts[2 * k], parts[2 * k + 1]) if parts is not None else (z.real, z.imag)
            if z == 0:
                out.append(("z",))
            elif z == 1:
                out.append(("1",))
            elif z == -1:
                out.append(("-1",))
            elif z.imag == 0:
                out.append(("r", self.cf([re])))
            elif z.real == 0:
                out.append(("i", self.cf([im])))
            else:
                out.append(("c", self.cf([re, im])))
        self.trace.append(("m", tuple(e[0] for e in out)))
        return out

    def emit_matvec_f32x2(self, coef, slots):
        """complex64 y = M x with packed FP32 pairs: a real entry is one FFMA2 on (x.re, x.im),
        an imaginary one an FFMA2 on i*x = (-x.im, x.re) (formed once per input column)."""
        d = len(slots)
        names = [f"v{self.vm[s]}" for s in slots]
        self.emit("      { const C " + ", ".join(f"x{c} = {names[c]}" for c in range(d)) + ";")
        for c in range(d):
            if any(coef[r * d + c][0] in ("i", "c") for r in range(d)):
                self.emit(f"        const C ix{c} = mkC(-x{c}.y, x{c}.x);")
        for r in range(d):
            y = None
            for c in range(d):
                e = coef[r * d + c]
                if e[0] == "z":
                    continue
                if e[0] == "1":
                    y = f"x{c}" if y is None else f"f2add({y}, x{c})"
                elif e[0] == "-1":
                    y = f"mkC(-x{c}.x, -x{c}.y)" if y is None else f"f2sub({y}, x{c})"
                elif e[0] == "r":
                    y = f"f2mul(PV({e[1]}), x{c})" if y is None else f"f2fma(PV({e[1]}), x{c}, {y})"
                elif e[0] == "i":
                    y = f"f2mul(PV({e[1]}), ix{c})" if y is None else f"f2fma(PV({e[1]}), ix{c}, {y})"
                else:
                    y = f"f2mul(PV({e[1]}), x{c})" if y is None else f"f2fma(PV({e[1]}), x{c}, {y})"
                    y = f"f2fma(PV({e[1] + 1}), ix{c}, {y})"
            self.emit(f"        {names[r]} = {y if y is not None else 'mkC(0.f, 0.f)'};")
        self.emit("      }")

    def emit_matvec(self, coef, slots):
        """y = M x over the amplitudes in `slots` (matrix row/col index = position in `slots`),
        skipping zero entries; one FMA chain per output component."""
        if self.quiet:
            return
        if self.dtype == nat.QSB_C64:
            return self.emit_matvec_f32x2(coef, slots)
        d = len(slots)
        names = [f"v{self.vm[s]}" for s in slots]
        self.emit("      { const C " + ", ".join(f"x{c} = {names[c]}" for c in range(d)) + ";")
        for r in range(d):
            ex, ey = None, None  # expressions accumulated so far (strings) for .x and .y

            def acc(cur, term_mul, a, b):
                # cur + a*b (a*b when cur is None); a may be None for +-1 (pure add / copy)
                if cur is None:
                    return term_mul
                return f"fma({a}, {b}, {cur})" if a is not None else f"({cur} + {b})"

            lines = []
            for c in range(d):
                e = coef[r * d + c]
                xc = f"x{c}"
                if e[0] == "z":
                    continue
                if e[0] in ("1", "-1"):
                    sg = "" if e[0] == "1" else "-"
                    ex = f"{sg}{xc}.x" if ex is None else (f"({ex} + {xc}.x)" if not sg else f"({ex} - {xc}.x)")
                    ey = f"{sg}{xc}.y" if ey is None else (f"({ey} + {xc}.y)" if not sg else f"({ey} - {xc}.y)")
                elif e[0] == "r":
                    a = f"PV({e[1]})"
                    ex = f"{a} * {xc}.x" if ex is None else f"fma({a}, {xc}.x, {ex})"
                    ey = f"{a} * {xc}.y" if ey is None else f"fma({a}, {xc}.y, {ey})"
                elif e[0] == "i":
                    b = f"PV({e[1]})"
                    ex = f"-{b} * {xc}.y" if ex is None else f"fma(-{b}, {xc}.y, {ex})"
                    ey = f"{b} * {xc}.x" if ey is None else f"fma({b}, {xc}.x, {ey})"
                else:
                    a, b = f"PV({e[1]})", f"PV({e[1] + 1})"
                    ex = f"{a} * {xc}.x" if ex is None else f"fma({a}, {xc}.x, {ex})"
                    ex = f"fma(-{b}, {xc}.y, {ex})"
                    ey = f"{a} * {xc}.y" if ey is None else f"fma({a}, {xc}.y, {ey})"
                    ey = f"fma({b}, {xc}.x, {ey})"
            if ex is None:
                ex = ey = "(R)0"
            self.emit(f"        {names[r]}.x = {ex}; {names[r]}.y = {ey};")
        self.emit("      }")

    def gen_g2(self, a):
        w, A = self.w, self.A
        ih, il, kind, gmask, gval, rmask, rval = w[a:a + 7]
        m = [self.d(i) for i in range(a + 7, a + 39)]
        self.emit(f"    {{ // G2 slot bits {ih},{il}")
        if gmask:
            self.emit(f"    if (((base | gt{self.li}) & {gmask}ull) == {gval}ull) {{")
        mat = [complex(m[2 * k], m[2 * k + 1]) for k in range(16)]
        coef = self.matrix_coeffs(mat, 4, m)
        for s in range(A):
            if s & ((1 << ih) | (1 << il)) or (s & rmask) != rval:
                continue
            self.emit_matvec(coef, [s, s | (1 << il), s | (1 << ih), s | (1 << ih) | (1 << il)])
        if gmask:
            self.emit("    }")
        self.emit("    }")

    def gen_pivot(self, a):
        w, A, TB = self.w, self.A, self.TB
        slot, ptype, pval, use_rt, ne = w[a:a + 5]
        nb = 1 << (TB - 4)
        ta_w = w[a + 5 + 3 * ne:a + 5 + 3 * ne + 32]
        tb_w = w[a + 5 + 3 * ne + 32:a + 5 + 3 * ne + 32 + 2 * nb]
        rt_w = w[a + 5 + 3 * ne + 32 + 2 * nb:a + 5 + 3 * ne + 32 + 2 * nb + 2 * A]
        o_ta = a + 5 + 3 * ne
        o_tb = o_ta + 32
        o_rt = o_tb + 2 * nb
        ta_p = [self.d(o_ta + k) for k in range(32)]
        tb_p = [self.d(o_tb + k) for k in range(2 * nb)]
        rt_p = [self.d(o_rt + k) for k in range(2 * A)]
        ta = [complex(ta_p[2 * k], ta_p[2 * k + 1]) for k in range(16)]
        tb = [complex(tb_p[2 * k], tb_p[2 * k + 1]) for k in range(nb)]
        rt = [complex(rt_p[2 * k], rt_p[2 * k + 1]) for k in range(A)]
        self.emit(f"    {{ // pivot {slot}")
        if ptype == 1:
            self.emit(f"    if (((base | gt{self.li}) & {pval}ull) != 0ull) {{")
        ta_all_one = all(z == 1 for z in ta)
        tb_all_one = all(z == 1 for z in tb)
        self.trace.append(("pivot", ta_all_one, tb_all_one, tuple(bool(use_rt and rt[s] != 1) for s in range(A))))
        self.emit(f"      double2 fd = sm.ep[it & 3][{slot}];")
        if not ta_all_one:
            ci = self.tf(ta_p)
            self.emit(f"      fd = dm(fd, cfz(scf, {ci} + 2 * (tid & 15)));")
        if not tb_all_one:
            ci = self.tf(tb_p)
            self.emit(f"      fd = dm(fd, cfz(scf, {ci} + 2 * (tid >> 4)));")
        self.emit("      const C f = toC(fd);")
        # which slots carry a register-partner factor (structure: RT entry != 1 from a partner bit)
        rt_ci = None
        if use_rt:
            rt_ci = self.cf(rt_p)
        for s in range(A):
            if ptype == 0 and not (s >> pval) & 1:
                continue
            if use_rt and rt[s] != 1:
                self.emit(f"      v{self.vm[s]} = cm(v{self.vm[s]}, cm(f, PZ({rt_ci + 2 * s})));")
            else:
                self.emit(f"      v{self.vm[s]} = cm(v{self.vm[s]}, f);")
        if ptype == 1:
            self.emit("    }")
        self.emit("    }")

    def gen_parity(self, a):
        """Sign flips of a batch of -1-phase diagonal gates (Z: single bits s1; CZ: bit pairs (b,
        b + d) for the bits b of mask m_d): the sign of amplitude gi is the GF(2) quadratic form
        Q(gi) = |gi & s1| + sum_d |gi & (gi >> d) & m_d|  (mod 2).  With gi = x | z, x = the
        tile-external and thread bits (runtime), z = the slot's register bits (compile-time),
        Q(x | z) = Q(x) + Q(z) + sum_i z_i L_i(x) with L_i(x) = |x & K_i| (mod 2) the bilinear
        cross terms of register bit i.  So one 32-bit sign word per thread and tile -- a few
        popcounts -- replaces per-amplitude 64-bit popcounts, and each amplitude costs one bit
        test and its negation."""
        if self.quiet:
            return  # integer words only: no coefficients
        w, A, NREG = self.w, self.A, self.NREG
        s1, nd = w[a], w[a + 1]
        pairs = [(w[a + 2 + 2 * q], w[a + 3 + 2 * q]) for q in range(nd)]
        C, cross = parity_sign_plan(s1, pairs, self.lay['goff'], NREG)
        full = (1 << A) - 1
        qx = " + ".join([f"__popcll(x & {s1}ull)"] + [f"__popcll(x & (x >> {d}) & {m}ull)" for d, m in pairs])
        self.emit("    { // parity (sign word)")
        self.emit(f"      const u64 x = base | gt{self.li};")
        self.emit(f"      u32 W = {C}u ^ ((({qx}) & 1) ? {full}u : 0u);")
        for K, Mi in cross:
            self.emit(f"      if (__popcll(x & {K}ull) & 1) W ^= {Mi}u;")
        for sl in range(A):
            v = f"v{self.vm[sl]}"
            if self.dtype == nat.QSB_C128:
                # flip the sign bits of both high words with bit sl of W moved to bit 31: each word
                # is one three-input LOP3, hi ^ (s & 0x80000000) (no predicate, no select)
                sh = f"(W << {31 - sl})" if sl < 31 else "W"
                if SIGN_LOP3:
                    self.emit(f"      {{ const unsigned s = {sh}; "
                              f"{v}.x = __hiloint2double((int)sgnx((unsigned)__double2hiint({v}.x), s), __double2loint({v}.x)); "
                              f"{v}.y = __hiloint2double((int)sgnx((unsigned)__double2hiint({v}.y), s), __double2loint({v}.y)); }}")
                else:
                    self.emit(f"      {{ const int m = (int)({sh} & 0x80000000u); "
                              f"{v}.x = __hiloint2double(__double2hiint({v}.x) ^ m, __double2loint({v}.x)); "
                              f"{v}.y = __hiloint2double(__double2hiint({v}.y) ^ m, __double2loint({v}.y)); }}")
            else:
                self.emit(f"      if (W & {1 << sl}u) {{ {v}.x = -{v}.x; {v}.y = -{v}.y; }}")
        self.emit("    }")

    def gen_term(self, a):
        w, A = self.w, self.A
        mask, val = w[a], w[a + 1]
        ci = self.cf([self.d(a + 2), self.d(a + 3)])
        if self.quiet:
            return
        self.emit(f"    {{ const C ph = PZ({ci});")
        for s in range(A):
            gi = f"(base | gt{self.li} | {self.lay['goff'][s]}ull)"
            self.emit(f"      if (({gi} & {mask}ull) == {val}ull) v{self.vm[s]} = cm(v{self.vm[s]}, ph);")
        self.emit("    }")

    def _kernel(self, name, body, store):
        K, n = self.K, self.n
        real = "double" if self.dtype == nat.QSB_C128 else "float"
        n_ext = n - K
        base_terms = [f"((c >> {m}) & 1ull) << {self.ext_pos[m]}" for m in range(n_ext)]
        out_terms = [f"((c >> {m}) & 1ull) << {self.ext_out[m]}" for m in range(n_ext)]
        base_expr = " | ".join(base_terms) if base_terms else "0ull"
        out_expr = " | ".join(out_terms) if (out_terms and self.ext_perm) else "base"
        tp = self.tplan
        ncalls = 1 << len(tp["iter_pos"])
        koff = " | ".join(f"((u64)((k >> {j}) & 1) << {b})" for j, b in enumerate(tp["iter_pos"])) or "0ull"
        coords = []
        for lo, nb, bx in tp["dims"]:
            coords.append("0" if bx else f"(int)((b >> {lo}) & {(1 << nb) - 1}ull)")
        coords += ["0"] * (5 - len(coords))
        call_bytes = tp["box_amps"] * (16 if self.dtype == nat.QSB_C128 else 8)
        hbit = f" | ((u64)HALF << {self.tile_pos[K - 1]})" if self.halves else ""
        produce = (f"        for (int k = lane; k < {ncalls}; k += 32) {{\n"
                   f"          const u64 b = base{hbit} | {koff};\n"
                   f"          const int co[5] = {{{', '.join(coords)}}};\n"
                   f"          tma5(d + (u64)k * {call_bytes}u, &tmap, co, &sm.full[s]);\n"
                   f"        }}")
        if "@@TMASTORE@@" in store:
            op_ = self.oplan
            o_ncalls = 1 << len(op_["iter_pos"])
            o_koff = " | ".join(f"((u64)((k >> {j}) & 1) << {b})" for j, b in enumerate(op_["iter_pos"])) or "0ull"
            o_coords = ["0" if bx else f"(int)((b >> {lo}) & {(1 << nb) - 1}ull)" for lo, nb, bx in op_["dims"]]
            o_coords += ["0"] * (5 - len(o_coords))
            o_bytes = op_["box_amps"] * (16 if self.dtype == nat.QSB_C128 else 8)
            # in place: the loads' map (over src = dst); out of place: a map over dst
            o_map = "tmap" if (op_ is tp and not self.ext_perm) else "tmap_o"
            store = store.replace("@@TMASTORE@@", (
                f"    if (tid < 32) {{\n"
                f"      for (int k = tid; k < {o_ncalls}; k += 32) {{\n"
                f"        const u64 b = obase | {o_koff};\n"
                f"        const int co[5] = {{{', '.join(o_coords)}}};\n"
                f"        tma5_store(&{o_map}, co, reinterpret_cast<const char*>(&sm.tbuf[0]) + (u64)k * {o_bytes}u);\n"
                f"      }}\n"
                f"      bulk_commit();\n"
                f"    }}"))
        pr = "double" if (self.dtype == nat.QSB_C128 or self.expect) else "float"
        defs = (f"#define QSB_F32X2 {1 if self.dtype == nat.QSB_C64 else 0}\n#define R {real}\n#define PR {pr}\n#define C {real}2\n#define KB {K}\n#define HBB {self.HB}\n#define SBB {self.SB}\n#define GB {self.G}\n#define STAGES {self.stages}\n#define ALIAS {1 if self.alias else 0}\n#define TBUF {"sm.stage[s]" if self.alias else "sm.tbuf"}\n"
                f"#define CONSUMERS {self.consumers}\n#define CONSUMERS_ALL {self.consumers * self.groups}\n"
                f"#define PINGPONG {1 if self.pingpong else 0}\n#define MAXPIV {MAX_PIV}\n#define NPIV {self.npiv}\n"
                f"#define NCOEF {max(1, len(self.coeffs))}\n#define NTAB {len(self.tables)}\n"
                f"#define TPC {self.sched[0]}\n#define DYN {self.sched[1]}\n")
        issue = f"""      {{ // producer warp: fetch tile c into stage s (tile number tno)
        const u64 base = {base_expr};
{self.ep_code}
        __syncwarp();
        if (lane == 0) {{
          sm.base[s][0] = base;
          sm.base[s][1] = {out_expr};
          mbar_expect_tx(&sm.full[s], (u32)((1u << KB) * sizeof(C)));
        }}
        __syncwarp();
        char* d = reinterpret_cast<char*>(&sm.stage[s][0]);
{produce}
      }}"""
        if self.halves:
            # both stages hold one tile: half h (tile bit K-1 = h) in stage h
            halves_code = []
            for h in (0, 1):
                halves_code.append(f"""      {{ // producer warp: half {h} of tile c -> stage {h}
        const int s = {h};
        if (it >= 1) mbar_wait(&sm.empty[{h}], (it & 1) ^ 1);""")
                if h == 0:
                    halves_code.append(f"""        const u64 base = {base_expr};
{self.ep_code}
        __syncwarp();
        if (lane == 0) {{ sm.base[0][0] = base; sm.base[0][1] = {out_expr}; }}""")
                else:
                    halves_code.append(f"""        const u64 base = {base_expr};""")
                halves_code.append(f"""        if (lane == 0) mbar_expect_tx(&sm.full[{h}], (u32)((1u << HBB) * sizeof(C)));
        __syncwarp();
        char* d = reinterpret_cast<char*>(&sm.stage[{h}][0]);
        constexpr u64 HALF = {h};
{produce}
      }}""")
            issue = "\n".join(halves_code)
        if self.pingpong:
            body = body.replace("@@REFILL@@", "    pp_sync(grp);  // my turn for the gate math")
            body += "\n    pp_arrive(1 - grp);  // the other group's turn"
        else:
            body = body.replace("@@REFILL@@", "")
        if self.alias:
            body = body.replace("@@RELEASE@@", "")
            body += "\n    csync();  // every thread is done with the stage (loads and transposes)\n" \
                    "    fence_async();\n    mbar_arrive(&sm.empty[s]);"
        if self.halves:
            head = """    mbar_wait(&sm.full[0], it & 1);
    const u64 base = sm.base[0][0];
    const u64 obase = sm.base[0][1];"""
        else:
            head = """    mbar_wait(&sm.full[s], ph);
    const u64 base = sm.base[s][0];
#if DYN || PINGPONG
    if (base == ~0ull) break;
#endif
    const u64 obase = sm.base[s][1];
    C* buf = sm.stage[s];"""
        return defs + _PRELUDE + f"""
// {self.consumers} consumer threads + one producer warpgroup (one active warp: TMA tile fetches and
// per-tile pivot factors, STAGES tiles ahead); setmaxnreg moves the producers' registers to the
// consumers, which hold the tile in registers.
extern "C" __global__ void __launch_bounds__({self.consumers * self.groups + 128}, {self.ctas})
{name}(const C* __restrict__ src, C* __restrict__ dst, const __grid_constant__ TMap tmap,
       const __grid_constant__ TMap tmap_o, const double* __restrict__ cf, unsigned long long* __restrict__ sched,
       const __grid_constant__ CP cp) {{
  extern __shared__ __align__(128) unsigned char smem_raw[];
  Smem& sm = *reinterpret_cast<Smem*>(smem_raw);
  double* scf = reinterpret_cast<double*>(smem_raw + sizeof(Smem));  // pivot tables
  const int tid = threadIdx.x;
  for (int i = tid; i < NTAB; i += {self.consumers * self.groups + 128}) scf[i] = cf[i];
  if (tid == 0) {{
    for (int s = 0; s < STAGES; ++s) {{ mbar_init(&sm.full[s], 1); mbar_init(&sm.empty[s], CONSUMERS); }}
    sm.zero = 0;
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }}
  __syncthreads();
  const u64 n_tiles = {1 << (n - K)}ull;
  // tiles of this CTA: TPC consecutive tiles per CTA with the grid covering the state once, so
  // the hardware block scheduler balances the SMs (a persistent grid with a static tile split
  // runs ~10% slower: every SM waits for the slowest one); TPC = 0: persistent grid-stride
#if TPC
  const u64 c_begin = (u64)blockIdx.x * TPC;
  const u64 c_end = c_begin + TPC < n_tiles ? c_begin + TPC : n_tiles;
  const u64 c_step = 1;
#else
  const u64 c_begin = blockIdx.x, c_end = n_tiles, c_step = gridDim.x;
#endif
  if (tid >= CONSUMERS_ALL) {{
    asm volatile("setmaxnreg.dec.sync.aligned.u32 {self.regs[1]};" ::: "memory");
    if (tid >= CONSUMERS_ALL + 32) return;
    const int lane = tid - CONSUMERS_ALL;
    int it = 0;
#if DYN
    // persistent: DYN consecutive tiles per grab from the launch's counter; a sentinel base
    // tells the consumers to stop; the last producer to finish re-arms the counter
    u64 c = 0, c_stop = 0;
    for (;; ++it) {{
      const int s = it % STAGES;
      const u32 ph = (it / STAGES) & 1;
      if (it >= STAGES) mbar_wait(&sm.empty[s], ph ^ 1);
      if (c == c_stop) {{
        u64 k = 0;
        if (lane == 0) k = atomicAdd(sched, 1ull);
        k = __shfl_sync(0xffffffffu, k, 0);
        c = k * DYN;
        c_stop = c + DYN < n_tiles ? c + DYN : n_tiles;
      }}
      if (c >= n_tiles) {{
        if (lane == 0) {{ sm.base[s][0] = ~0ull; mbar_arrive(&sm.full[s]); }}
#if PINGPONG
        {{  // the other consumer group's next stage gets a sentinel too
          const int s2 = (it + 1) % STAGES;
          if (it + 1 >= STAGES) mbar_wait(&sm.empty[s2], (((it + 1) / STAGES) & 1) ^ 1);
          if (lane == 0) {{ sm.base[s2][0] = ~0ull; mbar_arrive(&sm.full[s2]); }}
        }}
#endif
        break;
      }}
      const int tno = it;
{issue}
      ++c;
    }}
    if (lane == 0) {{
      __threadfence();
      if (atomicAdd(sched + 1, 1ull) == (u64)gridDim.x - 1) {{
        sched[0] = 0;
        sched[1] = 0;
        __threadfence();
      }}
    }}
#else
    for (u64 c = c_begin; c < c_end; c += c_step, ++it) {{
      const int s = it % STAGES;
      const u32 ph = (it / STAGES) & 1;
{"" if self.halves else "      if (it >= STAGES) mbar_wait(&sm.empty[s], ph ^ 1);"}
      const int tno = it;
{issue}
    }}
#if PINGPONG
    for (int e = 0; e < 2; ++e, ++it) {{  // both consumer groups stop on a sentinel
      const int s = it % STAGES;
      if (it >= STAGES) mbar_wait(&sm.empty[s], ((it / STAGES) & 1) ^ 1);
      if (lane == 0) {{ sm.base[s][0] = ~0ull; mbar_arrive(&sm.full[s]); }}
    }}
#endif
#endif
    return;
  }}
  asm volatile("setmaxnreg.inc.sync.aligned.u32 {self.regs[0]};" ::: "memory");
  double ea = 0.0;  // expectation passes: this thread's sum of Re <x|M|x>
#if PINGPONG
  {{
  const int grp = threadIdx.x / CONSUMERS;  // consumer group: takes producer iterations it = grp (mod 2)
  const int tid = threadIdx.x % CONSUMERS;
  if (grp == 1) pp_arrive(0);  // group 0 has the first gate-math turn
  for (int it = grp;; it += 2) {{
#else
  int it = 0;
#if DYN
  for (;; ++it) {{
#else
  for (u64 c = c_begin; c < c_end; c += c_step, ++it) {{
#endif
#endif
    const int s = it % STAGES;
    const u32 ph = (it / STAGES) & 1;
{head}
{body}
{store}
  }}
#if PINGPONG
  }}
#endif
{self._expect_epilogue() if self.expect else "  (void)ea;"}
{"  if (tid < 32) bulk_wait0();  // the last bulk stores are done before the CTA retires" if self.uses_tma_store else ""}
}}
"""

    def _expect_epilogue(self):
        """Deterministic CTA reduction of the per-thread sums -> dst[blockIdx.x] (double)."""
        return f"""  for (int o = 16; o > 0; o >>= 1) ea += __shfl_xor_sync(0xffffffffu, ea, o);
  csync();
  double* red = reinterpret_cast<double*>(&sm.ep[0][0]);
  if ((tid & 31) == 0) red[tid >> 5] = ea;
  csync();
  if (tid == 0) {{
    double t = 0.0;
    for (int w = 0; w < CONSUMERS / 32; ++w) t += red[w];
    reinterpret_cast<double*>(dst)[blockIdx.x] = t;
  }}"""


class _Compiled:
    __slots__ = ("func", "name", "smem", "tdesc", "tdesc_out", "n_tiles", "threads", "ctas", "tpc")

    def grid(self) -> int:
        """CTAs of one launch (one-shot tiles-per-CTA grid, or SMs x resident CTAs)."""
        if self.tpc:
            return pass_grid(self.n_tiles, self.threads - 128, self.tpc, _sm_count())
        return min(self.n_tiles, _sm_count() * self.ctas)


_SMS = None


def _sm_count() -> int:
    global _SMS
    if _SMS is None:
        torch = nat.torch_mod()
        _SMS = int(torch.cuda.get_device_properties(torch.cuda.current_device()).multi_processor_count)
    return _SMS


_cache: dict = {}
_lock = threading.Lock()
_disabled = os.environ.get("QSB_JIT", "1") == "0"
# QSB_JIT_PROBE=nogates|notransposes|nostores: timing experiments only (kernels compute wrong results)
_PROBE = os.environ.get("QSB_JIT_PROBE", "")
_MINIMAL = os.environ.get("QSB_MINIMAL_LAYOUT", "0") == "1"  # predicated transposes (fusion.MINIMAL_LAYOUT_CHANGES)
_avail = None


def _nvrtc_path():
    for p in ("/usr/local/cuda/lib64/libnvrtc.so.12",):
        if os.path.exists(p):
            return p
    try:
        import nvidia.cuda_nvrtc as m

        base = list(m.__path__)[0]
        p = os.path.join(base, "lib", "libnvrtc.so.12")
        if os.path.exists(p):
            return p
    except Exception:
        pass
    return ""


def available() -> bool:
    global _avail
    if _disabled:
        return False
    if _avail is None:
        try:
            _avail = bool(nat.lib().qsb_jit_available(_nvrtc_path().encode()))
        except Exception:
            _avail = False
    return _avail


def generate_full(words, dtype):
    """(source, kernel name, parameter coefficients, table coefficients, TMA plan) for a pass
    program (CPU-only)."""
    src, name, coeffs, tables, tplan, _key = _generate(words, dtype)
    return src, name, coeffs, tables, tplan


def _structure_key(g, words, dtype):
    masked = np.array(words, dtype=np.int64)
    if g.dpos:
        masked[np.fromiter(g.dpos, dtype=np.int64)] = 0
    return (int(dtype), masked.tobytes(), tuple(g.trace))


def _generate(words, dtype):
    g = _Gen(words, dtype)
    body_probe = g.generate("KNAME")
    name = "qsb_pass_" + hashlib.sha1(body_probe.encode()).hexdigest()[:16]
    src = body_probe.replace("KNAME", name)
    tplan = dict(g.tplan)
    # tensor map of the bulk stores when it differs from the loads' (out-of-place passes)
    tplan["tdesc_out"] = g.oplan["tdesc"] if (g.oplan is not None and (g.oplan is not g.tplan or g.ext_perm)) else None
    return (src, name, np.array(g.coeffs, dtype=np.float64), np.array(g.tables, dtype=np.float64), tplan,
            _structure_key(g, words, dtype))


def coefficients_only(words, dtype):
    """(structure key, parameter coefficients, table coefficients) without generating source:
    two programs with the same key compile to the same kernel (the key holds every word that is
    not a coefficient plus every value-dependent structure decision), so a pass whose structure
    was seen before -- every step of a time-dependent Trotter evolution -- only needs these."""
    g = _Gen(words, dtype)
    g.quiet = True
    g.generate("KNAME")
    return _structure_key(g, words, dtype), np.array(g.coeffs, dtype=np.float64), np.array(g.tables, dtype=np.float64)


# Coefficient recipes: for a structure seen before, the parameter and table vectors are plain
# reads of the program's coefficient words (plus structural constants), so a recipe -- the word
# position of every coefficient -- replaces the coefficient-only generator run (which walks the
# whole program: ~0.5 ms per pass).  A recipe is recorded with position-tagged reads and kept
# only if it reproduces a quiet generator run on a perturbed copy of the program (any derived
# value would differ); it matches a program with the same words outside the coefficient
# positions whose coefficients keep their value classes (0, +-1, +-1/sqrt 2, rounding noise,
# other), except that recorded noise may be an exact 0 now.  QSB_COEFF_RECIPES=0 disables.
RECIPES = os.environ.get("QSB_COEFF_RECIPES", "1") != "0"
_RECIPES: dict = {}
_RECIPES_MAX = 4096
_HH = 0.7071067811865475
RECIPE_STATS = {"hits": 0, "built": 0, "refused": 0}


def _value_classes(v) -> np.ndarray:
    """0, 1, -1, 1/sqrt 2, -1/sqrt 2 -> 0..4, anything else 5 (the values the generator's
    structure decisions test)."""
    out = np.full(v.shape[0], 5, np.uint8)
    out[np.abs(v) <= 1e-12] = 6  # rounding noise
    out[v == 0.0] = 0
    out[v == 1.0] = 1
    out[v == -1.0] = 2
    out[v == _HH] = 3
    out[v == -_HH] = 4
    return out


class _Recipe:
    __slots__ = ("dpos", "masked", "cls", "p_src", "p_const", "t_src", "t_const", "skey")


def _recipe_prekey(w, dtype):
    return (int(dtype), int(w.shape[0]), w[:H_TILEPOS + int(w[2])].tobytes())


def _recipe_lookup(w, dtype):
    with _lock:
        cands = list(_RECIPES.get(_recipe_prekey(w, dtype), ()))
    for r in cands:
        m = w.copy()
        m[r.dpos] = 0
        if m.tobytes() != r.masked:
            continue
        # every coefficient keeps its class (the kernel specialised on 0, +-1, ...), except that
        # rounding noise in the recorded program may be an exact 0 now (multiplied as a value)
        cls = _value_classes(w[r.dpos].view(np.float64))
        if np.all((cls == r.cls) | ((r.cls == 6) & (cls == 0))):
            return r
    return None


def _recipe_apply(r, w):
    v = w.view(np.float64)
    p = r.p_const.copy()
    sel = r.p_src >= 0
    p[sel] = v[r.p_src[sel]]
    t = r.t_const.copy()
    sel = r.t_src >= 0
    t[sel] = v[r.t_src[sel]]
    return p, t


def _recipe_build(words, dtype):
    """Record and check the recipe of a program (None when its coefficients are not plain
    reads, e.g. expectation passes)."""
    w = np.array(words, dtype=np.int64)
    if int(w[7]) & 2:
        return None
    g = _Gen(w, dtype)
    g.quiet = True
    g.record = True
    g.generate("KNAME")
    r = _Recipe()
    r.dpos = np.array(sorted(g.dpos), dtype=np.int64)
    m = w.copy()
    m[r.dpos] = 0
    r.masked = m.tobytes()
    vals = w[r.dpos].view(np.float64)
    r.cls = _value_classes(vals)
    r.p_src = np.array(g.csrc, dtype=np.int64)
    r.p_const = np.array(g.coeffs, dtype=np.float64)
    r.t_src = np.array(g.tsrc, dtype=np.int64)
    r.t_const = np.array(g.tables, dtype=np.float64)
    r.skey = _structure_key(g, w, dtype)
    # check on a perturbed program: every coefficient of class "other" scaled by (1 + 2^-20)
    w2 = w.copy()
    f = w2.view(np.float64)
    other = (r.cls == 5) | (r.cls == 6)
    f[r.dpos[other]] *= 1.0 + 2.0 ** -20
    g2 = _Gen(w2, dtype)
    g2.quiet = True
    g2.generate("KNAME")
    p2, t2 = _recipe_apply(r, w2)
    p1, t1 = _recipe_apply(r, w)
    ok = (_structure_key(g2, w2, dtype) == r.skey and np.array_equal(p2, np.array(g2.coeffs, dtype=np.float64))
          and np.array_equal(t2, np.array(g2.tables, dtype=np.float64))
          and np.array_equal(p1, r.p_const) and np.array_equal(t1, r.t_const))
    with _lock:
        if not ok:
            RECIPE_STATS["refused"] += 1
            return None
        RECIPE_STATS["built"] += 1
        if sum(len(v) for v in _RECIPES.values()) >= _RECIPES_MAX:
            _RECIPES.clear()
        _RECIPES.setdefault(_recipe_prekey(w, dtype), []).append(r)
    return r


def fast_coefficients(words, dtype):
    """coefficients_only through a matching recipe when there is one."""
    if RECIPES:
        w = np.asarray(words, dtype=np.int64)
        r = _recipe_lookup(w, dtype)
        if r is not None:
            RECIPE_STATS["hits"] += 1
            p, t = _recipe_apply(r, w)
            return r.skey, p, t
    return coefficients_only(words, dtype)


def generate(words, dtype):
    """(source, kernel name, parameter coefficients) for a pass program (CPU-only, tests)."""
    return generate_full(words, dtype)[:3]


MAX_COEFFS = 3072  # 24 KB of pivot tables staged in shared memory
MAX_PARAM_BYTES = 31616  # kernel parameter space: 32764 B minus the pointers and the two tensor maps


def split_stages(consumers: int) -> int:
    return 1 if ctas_per_sm(consumers) == 2 else 3


def smem_bytes(stage_bytes: int, n_coeffs=MAX_COEFFS, alias: bool = False, split: bool = False,
               consumers: int = 128, pingpong: bool = False) -> int:
    # STAGES stages + one transpose buffer of stage_bytes (a whole tile, or half of a 128 KB
    # tile); `alias`: a single stage that doubles as the transpose buffer (two CTAs per SM);
    # `split`: split_stages() stages + a half-size transpose buffer
    if pingpong:
        buf_bytes = 2 * stage_bytes  # one stage per consumer group, each its group's transpose buffer
    elif split:
        buf_bytes = split_stages(consumers) * stage_bytes + stage_bytes // 2
    else:
        buf_bytes = (1 if alias else STAGES + 1) * stage_bytes
    struct_bytes = buf_bytes + 4 * MAX_PIV * 16 + 8 * 3 * 4 + 16 + 16
    return struct_bytes + 8 * n_coeffs + 128


def _disk_cache_dir():
    """On-disk cubin cache (QSB_JIT_CACHE_DIR; default ~/.cache/qsb200; QSB_JIT_CACHE_DIR= (empty)
    disables).  Purely an optimisation: every read is checked and a miss recompiles."""
    d = os.environ.get("QSB_JIT_CACHE_DIR")
    if d is None:
        d = os.path.join(os.path.expanduser("~"), ".cache", "qsb200")
    if not d:
        return None
    tag = f"abi{int(nat.lib().qsb_abi_version())}-{os.path.basename(_nvrtc_path())}-sm100a"
    return os.path.join(d, "jit-" + tag)


def _load_or_compile(src: str, name: str) -> int:
    """CUfunction of `name` from the source: the disk cache when it holds this exact source's
    cubin, else NVRTC (and the cubin is stored for the next process)."""
    lib = nat.lib()
    fn = ctypes.c_void_p()
    digest = hashlib.sha256(src.encode()).hexdigest()
    ddir = _disk_cache_dir()
    path = os.path.join(ddir, f"{name}-{digest[:32]}.cubin") if ddir else None
    if path and os.path.exists(path):
        try:
            with open(path, "rb") as f:
                blob = f.read()
            if blob and lib.qsb_jit_load(blob, name.encode(), ctypes.byref(fn)) == 0:
                return fn.value
        except OSError:
            pass
    log = ctypes.create_string_buffer(1 << 16)
    cap = 8 << 20
    cubin = ctypes.create_string_buffer(cap) if path else None
    size = ctypes.c_size_t(0)
    rc = lib.qsb_jit_compile_cubin(src.encode(), name.encode(), _nvrtc_path().encode(), ctypes.byref(fn), log,
                                   len(log), cubin, cap if path else 0, ctypes.byref(size))
    if rc != 0:
        raise RuntimeError(f"NVRTC failed: {log.value.decode(errors='replace')[:2000]}")
    if path and 0 < size.value <= cap:
        try:
            os.makedirs(ddir, exist_ok=True)
            tmp = f"{path}.{os.getpid()}.{threading.get_ident()}.tmp"
            with open(tmp, "wb") as f:
                f.write(cubin.raw[:size.value])
            os.replace(tmp, path)
        except OSError:
            pass
    return fn.value


_WORDS_CACHE: dict = {}  # (dtype, program bytes) -> compile_words result: rebuilt identical circuits skip codegen
_WORDS_CACHE_MAX = 256


# compiled kernels by structure key (coefficients_only): a program whose structure was seen
# before only needs its coefficient vectors, not its source (time-dependent evolutions: every
# step has new coefficients, the same structure)
_STRUCT_CACHE: dict = {}


def _param_bytes(params, words, dtype):
    expect = bool(int(words[7]) & 2)
    pbytes = params.astype(np.float64 if (dtype == nat.QSB_C128 or expect) else np.float32)
    if pbytes.nbytes > MAX_PARAM_BYTES:
        raise RuntimeError(f"{pbytes.nbytes} bytes of gate coefficients exceed the kernel parameter space")
    if len(pbytes) == 0:
        pbytes = np.zeros(1, dtype=pbytes.dtype)
    return np.ascontiguousarray(pbytes)


def compile_words(words, dtype):
    wkey = (int(dtype), np.asarray(words, dtype=np.int64).tobytes())
    with _lock:
        done = _WORDS_CACHE.get(wkey)
    if done is not None:
        return done
    out = None
    if _STRUCT_CACHE:
        key, params, tables = fast_coefficients(words, dtype)
        with _lock:
            hit = _STRUCT_CACHE.get(key)
        if hit is not None and len(tables) <= MAX_COEFFS:
            out = (hit, (_param_bytes(params, words, dtype), tables))
    if out is None:
        out = _compile_words(words, dtype)
    with _lock:
        if len(_WORDS_CACHE) >= _WORDS_CACHE_MAX:
            _WORDS_CACHE.pop(next(iter(_WORDS_CACHE)))
        _WORDS_CACHE[wkey] = out
    return out


def _compile_words(words, dtype):
    src, name, params, tables, tplan, skey = _generate(words, dtype)
    if len(tables) > MAX_COEFFS:
        raise RuntimeError(f"{len(tables)} table entries exceed the shared-memory budget")
    pbytes = _param_bytes(params, words, dtype)
    expect = bool(int(words[7]) & 2)
    with _lock:
        hit = _cache.get(src)
    if hit is None:
        # NVRTC + module load outside the lock: passes of one plan compile concurrently
        fn = _load_or_compile(src, name)
        K, nreg = int(words[2]), int(words[3])
        amp = 16 if dtype == nat.QSB_C128 else 8
        stage_amps = 1 << (K - 1 if (1 << K) * amp > 65536 else K)
        fresh = _Compiled()
        fresh.func = fn
        fresh.name = name
        split = bool(int(words[7]) & 4) and (1 << K) * amp <= 65536
        pingpong = bool(int(words[7]) & 8) and (1 << K) * amp == 65536 and not split
        two = (ctas_per_sm(1 << (K - nreg)) == 2 or bool(int(words[7]) & 16)) and not pingpong
        alias = (1 << K) * amp == 65536 and two and not split
        fresh.smem = smem_bytes(stage_amps * amp, len(tables), alias, split, 1 << (K - nreg), pingpong)
        fresh.ctas = 2 if two else 1
        fresh.tdesc = np.array(tplan["tdesc"], dtype=np.int64)
        fresh.tdesc_out = None if tplan.get("tdesc_out") is None else np.array(tplan["tdesc_out"], dtype=np.int64)
        fresh.n_tiles = 1 << (int(words[4]) - K)
        fresh.threads = (1 << (K - nreg)) * (2 if pingpong else 1) + 128
        fresh.tpc = pass_schedule(int(words[4]) - K, 1 << (K - nreg), expect, (1 << K) * amp > 65536)[0]
        with _lock:
            hit = _cache.setdefault(src, fresh)
    with _lock:
        if len(_STRUCT_CACHE) >= 4096:
            _STRUCT_CACHE.pop(next(iter(_STRUCT_CACHE)))
        _STRUCT_CACHE[skey] = hit
    if RECIPES:
        try:
            _recipe_build(words, dtype)
        except Exception:  # an optimisation only
            pass
    return hit, (pbytes, tables)


def precompile(steps, dtype, device: int | None = None) -> None:
    """Specialise the passes of a plan concurrently (NVRTC runs outside the GIL and the cache
    lock); each worker binds the caller's CUDA device before loading its module.  Steps that
    fail keep `jit = None` and are retried (then fall back) when they run."""
    todo = [s for s in steps if getattr(s, "jit", None) is None and not getattr(s, "no_jit", False)]
    if len(todo) < 2 or not available():
        return
    if _STRUCT_CACHE:
        # passes whose structure is compiled already only need their coefficients: inline
        # (a thread pool per call costs more than that), the rest compile concurrently
        rest = []
        for st in todo:
            try:
                key, params, tables = fast_coefficients(st.words, dtype)
            except Exception:
                rest.append(st)
                continue
            with _lock:
                hit = _STRUCT_CACHE.get(key)
            if hit is not None and len(tables) <= MAX_COEFFS:
                st.jit = (hit, (_param_bytes(params, st.words, dtype), tables))
            else:
                rest.append(st)
        todo = rest
        if len(todo) < 2:
            return
    torch = nat.torch_mod()
    dev = torch.cuda.current_device() if device is None else device

    def work(step):
        try:
            torch.cuda.set_device(dev)
            step.jit = compile_words(step.words, dtype)
        except Exception:
            pass

    from concurrent.futures import ThreadPoolExecutor

    with ThreadPoolExecutor(max_workers=min(len(todo), max(1, min(16, os.cpu_count() or 1)))) as ex:
        list(ex.map(work, todo))


def run(words, dtype, src_ptr, dst_ptr, n_qubits, stream_ptr, compiled=None, coeffs=None, dev_tables=None):
    """Launch a specialised pass.  The pivot tables are staged through the library's host ring,
    or -- `dev_tables`, a device tensor holding them (CUDA-graph capture) -- read in place."""
    if compiled is None:
        compiled, coeffs = compile_words(words, dtype)
    params, tables = coeffs
    lib = nat.lib()
    tdo = None if compiled.tdesc_out is None else compiled.tdesc_out.ctypes.data
    if dev_tables is not None and len(tables):
        nat.check(
            lib.qsb_jit_run_pass_dev(compiled.func, src_ptr, dst_ptr, compiled.tdesc.ctypes.data, tdo, compiled.n_tiles,
                                     dev_tables.data_ptr(), len(tables), params.ctypes.data, params.nbytes,
                                     compiled.threads, compiled.smem, compiled.grid(), stream_ptr),
            "jit_run_pass_dev",
        )
        return
    nat.check(
        lib.qsb_jit_run_pass(compiled.func, src_ptr, dst_ptr, compiled.tdesc.ctypes.data, tdo, compiled.n_tiles,
                             tables.ctypes.data if len(tables) else None, len(tables),
                             params.ctypes.data, params.nbytes, compiled.threads, compiled.smem, compiled.grid(),
                             stream_ptr),
        "jit_run_pass",
    )
