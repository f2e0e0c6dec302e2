/*
 * qsb200 -- C ABI of the B200 (sm_100a) state-vector engine.
 *
 * This is the drop-in boundary for the hot path of the reference simulator `qsim`
 * (/root/reference/pkg/src/qsim).  Every entry point takes plain device pointers, sizes and a
 * caller-owned cudaStream_t (passed as void*), enqueues work asynchronously on that stream and
 * returns a qsb_status.  No torch / numpy types cross this boundary.  On a non-zero status,
 * qsb_last_error() returns a human-readable message (thread-local).
 *
 * Concurrency: entry points may be called from several host threads (host-side caches are
 * locked or thread-local).  The small device scratch buffers of the reductions and the pass
 * program ring are per device and per process, so work that uses them (norm / vdot / expect /
 * sampling / interpreted passes) must not run concurrently on two streams of one device --
 * the reference's contract of one stream per state, serialised calls (gates.py:389-394).
 *
 * Conventions (identical to the reference):
 *   - the state is 2**n complex numbers, interleaved (re, im), complex64 (dtype QSB_C64) or
 *     complex128 (QSB_C128);
 *   - qubit q lives at bit position n-1-q (qubit 0 is the MSB) -- state.py:1-6, 34-36.  This ABI
 *     takes BIT positions; the Python layer converts qubits to bits;
 *   - gate matrices are row-major 2**t x 2**t complex128 (numpy complex128 memory layout), and
 *     target_bits[0] is the most significant bit of the matrix index -- gates.py:128-131.
 *     For complex64 states the matrix is rounded to complex64 before use, as the reference's
 *     `mat64.astype(amplitudes.dtype)` does (gates.py:434, 447, 462).
 */
#ifndef QSB200_H
#define QSB200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define QSB_ABI_VERSION 5

typedef enum { QSB_C64 = 0, QSB_C128 = 1 } qsb_dtype;

/* Kernel classes of the reference (gates.py:334-352, KernelClass). */
typedef enum {
  QSB_KERNEL_AUTO = -1,
  QSB_KERNEL_GENERAL = 0,
  QSB_KERNEL_DIAGONAL = 1,
  QSB_KERNEL_PERMUTATION = 2
} qsb_kernel;

typedef enum {
  QSB_OK = 0,
  QSB_ERR_ARG = 1,      /* bad argument (maps to ValueError) */
  QSB_ERR_SHAPE = 2,    /* index / layout problem (maps to ShapeError) */
  QSB_ERR_CAPACITY = 3, /* size cap exceeded (maps to CapacityError) */
  QSB_ERR_CUDA = 4      /* CUDA runtime error (maps to SimulationError) */
} qsb_status;

/* ---- library ---------------------------------------------------------------------------- */
int qsb_abi_version(void);
const char* qsb_last_error(void);

/* ---- state allocator / initial states (state.py:67-75 zero_state, hamiltonians.py:115-117
 *      _plus_state).  The caller owns the 2**n-element device buffer. ------------------------- */
/* |basis_index>: all zeros, amplitude 1 at basis_index.  zero_state == basis_index 0. */
int qsb_init_basis(void* amps, int n_qubits, int dtype, uint64_t basis_index, void* stream);
/* every amplitude = (re, im); |+>^n is re = 2**(-n/2). */
int qsb_init_uniform(void* amps, int n_qubits, int dtype, double re, double im, void* stream);

/* ---- single-gate kernels: the reference's apply_matrix (gates.py:380-469) ---------------- */
/* Classify a 2**t x 2**t complex128 matrix exactly like classify_kernel (gates.py:340-352):
 * returns QSB_KERNEL_DIAGONAL / _PERMUTATION / _GENERAL. */
int qsb_classify(const double* matrix, int n_targets);
/* In-place application of `matrix` on `target_bits` (t = 1 to 5; 3-5 targets run a generic
 * one-group-per-thread kernel with the matrix as a kernel parameter), restricted to the basis
 * states whose `control_bits` are all 1.  `kernel` = QSB_KERNEL_AUTO classifies first;
 * an explicit class forces that body, with the reference's semantics (diagonal body reads only
 * the diagonal and skips rows equal to 1.0; permutation body takes the first non-zero of each
 * row and multiplies only phases != 1.0). */
int qsb_apply_matrix(void* amps, int n_qubits, int dtype, int n_targets, const int* target_bits,
                     int n_controls, const int* control_bits, const double* matrix, int kernel,
                     void* stream);
/* A gate list on a small or mid-size state in one launch per 64 gates (Circuit.execute without
 * pass planning, circuit.py:96-125 -> gates.py:472-487 per gate).  States up to
 * QSB_BATCH_MAX_STATE_BYTES (13 qubits complex128, 14 complex64) are held in one CTA's shared
 * memory; states up to QSB_GRID_BATCH_MAX_STATE_BYTES (26 / 27 qubits) are walked by a
 * cooperative grid with a grid barrier between gates (L2-resident up to ~64 MB).  The gates run in queue order with
 * the bodies and semantics of qsb_apply_matrix, so the result equals n_gates qsb_apply_matrix
 * calls bit for bit.  Gate i: n_targets[i] target bits at target_bits[2i..], n_controls[i]
 * control bits taken consecutively from control_bits, its 2**t x 2**t complex128 matrix
 * row-major at matrices[32i..] (interleaved re, im) and its kernel class in kernels[i].  The
 * whole list is validated before any work is enqueued. */
#define QSB_BATCH_MAX_STATE_BYTES 131072
#define QSB_GRID_BATCH_MAX_STATE_BYTES 1073741824
int qsb_apply_batch(void* amps, int n_qubits, int dtype, int n_gates, const int* n_targets,
                    const int* target_bits, const int* n_controls, const int* control_bits,
                    const double* matrices, const int* kernels, void* stream);
/* Multiply every amplitude of [amps, amps + n_amps) by (re, im) -- the all-global phase of the
 * sharded executor (sharding.py:281-283) and from_amplitudes(normalize=True) (state.py:101-105). */
int qsb_scale(void* amps, uint64_t n_amps, int dtype, double re, double im, void* stream);
/* Projective collapse (extension: the reference has no mid-circuit measurement):
 * amplitudes with (index & mask) == value are multiplied by `scale` (1/sqrt(p) of the outcome),
 * every other amplitude is set to zero. */
int qsb_collapse(void* amps, uint64_t n_amps, int dtype, uint64_t mask, uint64_t value, double scale,
                 void* stream);

/* ---- fused multi-gate pass (one HBM sweep for a run of gates) --- */
/* `program` is a flat little-endian int64 word stream produced by the host planner
 * (paper_2009_01845_b200/fusion.py); `n_words` its length.  src may equal dst when the pass
 * carries no tile-external bit permutation. */
int qsb_run_pass(const void* src, void* dst, int n_qubits, int dtype, const int64_t* program,
                 int64_t n_words, void* stream);
/* Bytes of shared memory the pass kernel needs for a tile of 2**tile_bits amplitudes. */
int qsb_pass_max_tile_bits(int dtype);

/* ---- pass specialisation (NVRTC): a straight-line kernel per pass structure -------------- */
/* 1 when NVRTC (dlopen'ed from `nvrtc_path` or the default search path) and the driver API
 * entry points are usable. */
int qsb_jit_available(const char* nvrtc_path);
/* Compile CUDA C++ `source` for sm_100a and return the CUfunction `name` in *func_out. */
int qsb_jit_compile(const char* source, const char* name, const char* nvrtc_path, void** func_out,
                    char* log_out, size_t log_cap);
/* qsb_jit_compile that also copies the compiled cubin into cubin_out (when it fits cubin_cap;
 * *cubin_size gets its size either way), for an on-disk kernel cache. */
int qsb_jit_compile_cubin(const char* source, const char* name, const char* nvrtc_path, void** func_out,
                          char* log_out, size_t log_cap, void* cubin_out, size_t cubin_cap, size_t* cubin_size);
/* Load a cubin produced by qsb_jit_compile_cubin (same library build) and return `name`. */
int qsb_jit_load(const void* cubin, const char* name, void** func_out);
/* Launch a specialised pass kernel over `n_tiles` tiles.  `tma_desc` describes the state as the
 * rank-5 tensor the kernel's tile loads address (15 words: rank, global dims[5], byte strides of
 * dims 1..4, box dims[5]; jit.py tma_plan); `tma_desc_out` (NULL: the same) the tensor the bulk
 * tile stores address over `dst` (out-of-place passes whose output tile bits sit elsewhere).  `tables` (doubles, staged to the device) are the
 * per-thread pivot tables; `params` (`param_bytes`, passed by value as the kernel's last
 * parameter) are the uniform gate coefficients; `grid` CTAs are launched (1 <= grid <= n_tiles:
 * one-shot CTAs of a few tiles each, or a persistent grid, as the kernel was generated for). */
int qsb_jit_run_pass(void* func, const void* src, void* dst, const int64_t* tma_desc, const int64_t* tma_desc_out,
                     uint64_t n_tiles,
                     const double* tables, int64_t n_tables, const void* params, int64_t param_bytes,
                     int threads, int smem_bytes, int grid, void* stream);
/* qsb_jit_run_pass with the pivot tables already in device memory (`dev_tables`, owned by the
 * caller and alive until the launch completes): nothing is staged through the library's host
 * ring, so the launch can be captured into a CUDA graph and replayed.  (qsb_jit_run_pass and
 * qsb_run_pass refuse to stage while their stream is capturing.) */
int qsb_jit_run_pass_dev(void* func, const void* src, void* dst, const int64_t* tma_desc,
                         const int64_t* tma_desc_out, uint64_t n_tiles,
                         const double* dev_tables, int64_t n_tables, const void* params, int64_t param_bytes,
                         int threads, int smem_bytes, int grid, void* stream);

/* ---- reductions (state.py:109-122 norm / overlap) ---------------------------------------- */
/* out[0] = sum |a_i|^2 (double, device pointer).  Deterministic two-level tree. */
int qsb_norm2(const void* amps, uint64_t n_amps, int dtype, double* out, void* stream);
/* out[0..1] = <a|b> (conjugate-linear in a), complex128 on device.  Deterministic. */
int qsb_vdot(const void* a, const void* b, uint64_t n_amps, int dtype, double* out, void* stream);

/* out[0..1] = sum_t <psi| M_t |psi> over n_terms 1- or 2-qubit terms (hamiltonians.py:192-207
 * `expectation`): ks[t] in {1, 2}, bits[2t] = bit of targets[0] (matrix MSB), bits[2t+1] = bit of
 * targets[1]; mats = 32 doubles per term (row-major complex 2^k x 2^k).  One read-only sweep per
 * term, no state copy; deterministic. */
int qsb_expect_terms(const void* amps, int n_qubits, int dtype, int n_terms, const int* ks, const int* bits,
                     const double* mats, double* out, void* stream);

/* ---- measurement (measurement.py:36-87) -------------------------------------------------- */
/* probs[i] = |a_i|^2 computed exactly as numpy's np.abs(a.astype(complex128))**2
 * (SURVEY.md Appendix B.1), float64 on device. */
int qsb_probabilities(const void* amps, uint64_t n_amps, int dtype, double* probs, void* stream);
/* Marginal over the bits NOT listed in `kept`, reproducing numpy's
 * `probs.reshape([2]*n).sum(axis=other)` followed by the transpose to the requested order, bit
 * for bit (pairwise inner sums, sequential outer accumulation)
 * -- measurement.py:50-58.  kept[0] is the most significant bit of the output index.
 * `scratch` holds qsb_marginal_scratch_doubles(n_bits, k) doubles. */
int qsb_marginal(const double* probs, int n_bits, int k, const int* kept, double* out,
                 double* scratch, void* stream);
/* qsb_marginal computed straight from the amplitudes (no 2^n probability array): available when
 * the 8 lowest bit positions are all reduced (numpy's 128-element leaves are then whole runs);
 * otherwise QSB_ERR_ARG.  Same bits as qsb_probabilities + qsb_marginal. */
int qsb_marginal_amps(const void* amps, int dtype, int n_bits, int k, const int* kept, double* out, double* scratch,
                      void* stream);
uint64_t qsb_marginal_scratch_doubles(int n_bits, int k);
/* cum[i] = fl(cum[i-1] + p[i]) -- the exact result of numpy's strictly sequential np.cumsum,
 * computed in parallel (binade-integer scan), then cum /= cum[n-1]
 * (measurement.py:81-82).  Synchronises `stream` once (data-dependent serial-point count). */
int qsb_cumsum_normalized(const double* probs, uint64_t n, double* cum, void* scratch,
                          size_t scratch_bytes, void* stream);
size_t qsb_cumsum_scratch_bytes(uint64_t n);
/* The same exact sequential cumsum; normalize = 0 leaves cum[i] = fl(cum[i-1] + p[i]) undivided
 * (the sharded sampler chains shards by prepending the previous shard's last value). */
int qsb_cumsum(const double* probs, uint64_t n, double* cum, void* scratch, size_t scratch_bytes, int normalize,
               void* stream);
/* The strictly sequential fl(c + p) chain on one device thread (no normalisation): the
 * cross-check for qsb_cumsum_normalized in the GPU tests. */
int qsb_cumsum_serial(const double* probs, uint64_t n, double* cum, void* stream);
/* PCG64 (XSL-RR 128/64, numpy.random.PCG64) draws u_k = (raw_k >> 11) * 2^-53 from the 128-bit
 * (state, inc) of numpy's bit_generator.state, then samples[k] = clip(#{i : cum[i] <= u_k},
 * 0, n-1) -- np.searchsorted(cum, u, side="right") (measurement.py:83-86). */
int qsb_sample(const double* cum, uint64_t n, uint64_t state_hi, uint64_t state_lo,
               uint64_t inc_hi, uint64_t inc_lo, uint64_t n_shots, int64_t* samples, void* stream);
/* The same draws; counts[k] = #{i : cum[i] <= u_k} without the clip, so that the counts of the
 * pieces of a distribution split across shards (in index order) add up to the global
 * searchsorted index (sharded sampling). */
int qsb_sample_counts(const double* cum, uint64_t n, uint64_t state_hi, uint64_t state_lo,
                      uint64_t inc_hi, uint64_t inc_lo, uint64_t n_shots, int64_t* counts, void* stream);
/* qsb_cumsum_normalized + qsb_sample in one call without materialising the CDF: each draw
 * finds its 4096-element block from the exact block boundaries of the scan; only the blocks
 * that hold a draw get the exact cumulative value before each of their 16-element rows
 * (written into `cum`, which needs ceil(n / 4096) * 256 doubles), and each draw walks its row
 * with fl(c + p) from that value.  Samples are bit-identical to the two-call path.
 * `scratch`: qsb_sample_exact_scratch_bytes(n, n_shots) bytes; n_shots < 2^32. */
size_t qsb_sample_exact_scratch_bytes(uint64_t n, uint64_t n_shots);
int qsb_sample_exact(const double* probs, uint64_t n, double* cum, void* scratch, size_t scratch_bytes,
                     uint64_t state_hi, uint64_t state_lo, uint64_t inc_hi, uint64_t inc_lo, uint64_t n_shots,
                     int64_t* samples, void* stream);
/* The same with the approximate 4096-element block sums supplied (qsb_probabilities_block_sums
 * computes them with the probabilities, in one read of the amplitudes). */
int qsb_sample_exact_bsums(const double* probs, const double* block_sums, uint64_t n, double* cum, void* scratch,
                           size_t scratch_bytes, uint64_t state_hi, uint64_t state_lo, uint64_t inc_hi,
                           uint64_t inc_lo, uint64_t n_shots, int64_t* samples, void* stream);
/* qsb_probabilities plus block_sums[b] = the sum of probs[4096 b .. 4096 b + 4095] in the order
 * qsb_sample_exact forms it (ceil(n / 4096) doubles). */
int qsb_probabilities_block_sums(const void* amps, uint64_t n, int dtype, double* probs, double* block_sums,
                                 void* stream);

/* ---- sharded execution helpers (sharding.py:53-111 partition / gather / _exchange_halves) - */
/* dst[i'] = src[i] where bit b of i moves to bit dst_bit[b] of i' (moveaxis of partition /
 * transpose of gather, sharding.py:65-70, 76-80). */
int qsb_permute_qubits(const void* src, void* dst, int n_bits, int dtype, const int* dst_bit,
                       void* stream);
/* In-process exchange: swap a's half with local `bit` = 1 and b's half with `bit` = 0
 * (sharding.py:100-111). */
int qsb_exchange_halves(void* a, void* b, int n_local_bits, int dtype, int bit, void* stream);
/* Copy the `half` (0 or 1) of a shard selected by local bit `bit` into / out of a contiguous
 * staging buffer, for elements [first, first + count) of that half in index order. */
int qsb_pack_half(const void* shard, int n_local_bits, int dtype, int bit, int half,
                  uint64_t first, uint64_t count, void* staging, void* stream);
int qsb_unpack_half(void* shard, int n_local_bits, int dtype, int bit, int half, uint64_t first,
                    uint64_t count, const void* staging, void* stream);
/* Batched global<->local exchange of k qubits (one all-to-all instead of k pairwise
 * reshuffles; the k-qubit generalisation of sharding.py:84-111).  A *part* of a shard is the
 * set of amplitudes whose local bits `bits[0..k)` hold the pattern `part_bits` (a mask already
 * placed at those bit positions); element e of a part is its e-th amplitude in index order.
 * pack/unpack copy elements [first, first + count) of a part to / from a contiguous staging
 * buffer (the per-peer send / receive chunks of the all-to-all). */
int qsb_pack_part(const void* shard, int n_local_bits, int dtype, int k, const int* bits, uint64_t part_bits,
                  uint64_t first, uint64_t count, void* staging, void* stream);
int qsb_unpack_part(void* shard, int n_local_bits, int dtype, int k, const int* bits, uint64_t part_bits,
                    uint64_t first, uint64_t count, const void* staging, void* stream);
/* In-process form: swap part `a_bits` of shard a with part `b_bits` of shard b (a != b). */
int qsb_exchange_parts(void* a, void* b, int n_local_bits, int dtype, int k, const int* bits, uint64_t a_bits,
                       uint64_t b_bits, void* stream);
/* Reduced density matrix of a qubit subset (entanglement_entropy, evolution.py:154-173):
 * rho[i][j] = sum_b psi(i, b) conj(psi(j, b)) in complex128, i = the k state bits
 * `partition_bits` (partition_bits[0] = MSB of i), b = every other bit.  Replaces the
 * reference's moveaxis + reshape + SVD (whose squared singular values are rho's eigenvalues).
 * 1 <= k <= 12.  `partials`: n_split * 4^k complex128 of device scratch (n_split a power of
 * two, n_split * 32 <= 2^(n-k)); `rho`: 4^k complex128 (device), row-major. */
int qsb_reduced_density(const void* amps, int n, int dtype, int k, const int* partition_bits, int n_split,
                        void* partials, void* rho, void* stream);

#ifdef __cplusplus
}
#endif

#endif /* QSB200_H */
