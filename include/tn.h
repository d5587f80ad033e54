/*
 * tn.h — C ABI of the B200 (sm_100a) sliced tensor-network contraction library
 * for arXiv 2310.03978 ("Efficient Quantum Circuit Simulation by Tensor Network
 * Methods on Modern GPUs").  Citations are PAPER.md lines (L<n>) of
 * /root/reference/PAPER.md; DESIGN.md lists every reading of the paper.
 *
 * What the library computes (the north-star hot path, SURVEY.md §8 a):
 *   Given a tensor network (the tensors of a quantum circuit, §2.1), a
 *   contraction path (§3.1), a slice set (§3.2) and a
 *   sparse-state boundary (§3.3, App. A.1), it executes every
 *   pairwise einsum (Eq. 3) as (optional) index permutation + complex
 *   GEMM on the GPU — sparse merges as gather-batched GEMMs (Eq. 7;
 *   L354) — sums the per-slice results in fp64 (L497 "the final outcome was the
 *   sum of the resulting tensors") and returns the amplitudes of the requested
 *   bitstrings.  No CPU fallback exists: every step of a contraction runs in
 *   this library's CUDA kernels.
 *
 * Conventions
 *   - All host arrays are owned by the caller and copied before a call returns.
 *   - Device memory is obtained through the tn_allocator given to tn_create (the
 *     Python binding passes torch's caching allocator, so the plan's arena, operand
 *     scratch and fp64 accumulator are torch-managed memory; SURVEY.md §8 b) and is
 *     owned by the context until tn_destroy / re-planning returns it; with a NULL
 *     allocator the library uses cudaMalloc / cudaFree.  The `out` buffer of
 *     tn_sum_slices is the caller's.
 *   - All GPU work is enqueued on the stream given to tn_create; calls that
 *     return device results do not synchronise unless stated.
 *   - Errors: every call returns a tn_status; on failure tn_last_error() returns
 *     a thread-local message.  No C++ exception crosses the ABI.
 *   - Call order: tn_create -> tn_load_network -> tn_set_path -> tn_set_slices
 *     -> tn_contract* -> tn_sum_slices.  tn_set_path invalidates the slice set
 *     and plan; tn_set_slices (re)builds the plan (TN_ERR_USAGE otherwise).
 */
#ifndef TN_B200_H
#define TN_B200_H

#include <stddef.h>
#include <stdint.h>

#if defined(__GNUC__)
#define TN_API __attribute__((visibility("default")))
#else
#define TN_API
#endif

#ifdef __cplusplus
extern "C" {
#endif

typedef struct tn_ctx tn_ctx;

typedef enum {
  TN_OK = 0,
  TN_ERR_USAGE = 1,     /* wrong call order / bad argument (SPEC L623 exit-code table) */
  TN_ERR_DATA = 2,      /* inconsistent network / path / slices / samples            */
  TN_ERR_RESOURCE = 3,  /* plan does not fit device memory                           */
  TN_ERR_CUDA = 4,      /* CUDA runtime / driver failure                              */
  TN_ERR_INTERNAL = 5
} tn_status;

typedef enum {
  /* Every tensor-core step uses the 3-pass hi/lo fp16 split (the 3xFP16 scheme of
   * §4.2 L383-386 with the power-of-two rescaling of L403/L594).                  */
  TN_PREC_EXTENDED = 0,
  /* The `mixed_topk` tensor-core steps with the largest T_cc run 1-pass fp16, the
   * rest 3-pass (mixed precision, §4.3, Table 3).                   */
  TN_PREC_MIXED = 1
} tn_precision;

/* Device-memory source of a context (SURVEY.md §8 b "torch caching allocator").
 *   alloc(bytes, device, cuda_stream, user) returns a device pointer (>= 256-B
 *     aligned) valid for work on `cuda_stream`, or NULL on failure (the calling
 *     tn_* function then fails with TN_ERR_RESOURCE);
 *   free(ptr, bytes, device, cuda_stream, user) returns a block obtained from alloc;
 *     work already enqueued on cuda_stream may still use it (stream-ordered release,
 *     as torch's caching allocator provides).
 * Both may be called from any tn_* call that (re)plans, loads or destroys. */
typedef struct {
  void* (*alloc)(size_t bytes, int device, void* cuda_stream, void* user);
  void (*free)(void* ptr, size_t bytes, int device, void* cuda_stream, void* user);
  void* user;
} tn_allocator;

/* Create a context bound to CUDA `device`, enqueuing on `cuda_stream` (a
 * cudaStream_t; NULL = legacy default stream).  One context per GPU / rank: "each
 * A100 GPU executed partial sub-tasks independently".  `allocator`
 * (copied; NULL = cudaMalloc) supplies every device allocation of the context.
 * device = -1 creates a host-only planner (bookkeeping and tn_plan_json only).
 * *out receives the handle.  TN_ERR_USAGE: out NULL, bad device index, an allocator
 * missing alloc or free; TN_ERR_CUDA: the device is not sm_100. */
TN_API tn_status tn_create(tn_ctx** out, int device, const tn_allocator* allocator, void* cuda_stream);

/* Load a tensor network (§2.1) and its sparse-state boundary.
 *   n_tensors       number of tensors N (>= 1)
 *   ranks[N]        number of indices of each tensor
 *   labels[Σranks]  bond id of every index, tensors concatenated; the data of
 *                   tensor t is row-major over its labels in this order
 *   dims[Σranks]    extent of every index (must agree for a shared bond)
 *   data            complex128 values, interleaved (re, im), tensors concatenated
 *                   row-major; rounded to complex64 on the device
 *   n_open, open_labels[n_open]
 *                   the open bonds, in qubit order: open_labels[q] is qubit q,
 *                   qubit 0 = most significant bit of a bitstring (DESIGN R4)
 *   n_samples, samples[n_samples*n_open]
 *                   the sparse state: one 0/1 byte per open bond per sample (the
 *                   bitstrings whose amplitudes are wanted, App. A.1).  samples =
 *                   NULL requests the full state (all 2^n_open bitstrings in index
 *                   order; n_open <= 24).  Duplicate samples are allowed.
 * Errors (TN_ERR_DATA): a closed bond not on exactly two tensors, an open bond not
 * on exactly one, a bond repeated inside a tensor, a dim mismatch, an open bond
 * with dim != 2, a sample byte not 0/1, n_open > 64, n_samples < 1. */
TN_API tn_status tn_load_network(tn_ctx* ctx, int32_t n_tensors, const int32_t* ranks,
                          const int64_t* labels, const int64_t* dims, const double* data,
                          int32_t n_open, const int64_t* open_labels,
                          int64_t n_samples, const uint8_t* samples);

/* Replace the tensor values of the loaded network (§2.1: gates and states
 * as tensors; same layout as `data` above, host pointer) without re-planning:
 * host->device copy on the context stream.  If any leaf's max |Re|,|Im| changes by
 * more than 2x (up or down), the fp16-plane delayed-scaling history restarts and
 * the next slice runs unfused; otherwise the history and the captured
 * CUDA graph are kept.  TN_ERR_USAGE before tn_load_network or on a host-only
 * context. */
TN_API tn_status tn_upload_tensors(tn_ctx* ctx, const double* data);

/* Set the contraction path (§3.1): n_steps = N-1 pairs (i, j) of tensor
 * ids; the result of step (i, j) takes id i ("indexed by the first tensor") and
 * id j retires.  TN_ERR_DATA if a pair references a retired/unknown id, i == j,
 * or n_steps != N-1. */
TN_API tn_status tn_set_path(tn_ctx* ctx, int32_t n_steps, const int32_t* pairs);

/* Slice the listed closed bonds (§3.2) and build the execution plan.
 * Slice index t in [0, Π dims) decodes in mixed radix over sliced_labels in the
 * given order, the LAST label fastest (DESIGN R7).  n_sliced = 0 = no slicing.
 * *n_slices_out receives Π dims.  TN_ERR_DATA for an open, unknown or repeated
 * label; TN_ERR_RESOURCE if the plan's device memory does not fit. */
TN_API tn_status tn_set_slices(tn_ctx* ctx, int32_t n_sliced, const int64_t* sliced_labels,
                        int64_t* n_slices_out);

/* Contract slices t = slice_begin .. slice_end-1 (each one full pass over the
 * path, every step the pairwise einsum of Eq. 3, sparse merges per Eq. 7
 * L306-308; the slices are the independent sub-tasks of L293) and ADD each slice's
 * root tensor into the context's fp64 accumulator (fused slice-accumulate, L497).  Repeating a range double-counts it.  Asynchronous.
 * precision / mixed_topk: see tn_precision.  TN_ERR_DATA if the range is not
 * inside [0, n_slices).  The first slice a context executes runs every kernel
 * launch directly (it tunes the SIMT kernel variants and seeds the delayed
 * scaling of fused fp16 operand planes); later slices replay one captured CUDA
 * graph of the per-slice launch sequence (not while profiling). */
TN_API tn_status tn_contract(tn_ctx* ctx, int64_t slice_begin, int64_t slice_end,
                      tn_precision precision, int32_t mixed_topk);

/* Zero the fp64 accumulator of the slice sum (L497) and the fused-plane overflow
 * flag (asynchronous).  TN_ERR_USAGE before tn_set_slices. */
TN_API tn_status tn_reset_accumulator(tn_ctx* ctx);

/* Write the accumulated amplitudes — "the sum of the resulting tensors" (L497) of the
 * slices contracted so far, i.e. "the amplitudes of sampled bitstrings" (L256) — in
 * the caller's sample order (full state: index order), as complex128 (re, im) into
 * the DEVICE buffer out[2*n_out] (caller-owned, >= 16-B aligned).
 * n_out must equal n_samples (or 2^n_open for the full state; 1 when n_open = 0).
 * Asynchronous on the context stream.  The fused-plane overflow flag (a producer
 * epilogue's delayed-scaling margin exceeded, so the sum may contain saturated fp16
 * operands) is checked by the gather kernel itself: when it is set, out is filled
 * with NaN instead of amplitudes, and tn_last_overflow() reports it after a sync
 * (rerun with TN_FUSE_PLANES=0); tn_reset_accumulator clears the flag.
 * TN_ERR_USAGE: n_out mismatch, out NULL, before tn_set_slices. */
TN_API tn_status tn_sum_slices(tn_ctx* ctx, double* out, int64_t n_out);

/* Same as tn_sum_slices but into a HOST buffer; synchronises the stream and fails
 * with TN_ERR_DATA (no output) when the fused-plane overflow flag is set. */
TN_API tn_status tn_sum_slices_host(tn_ctx* ctx, double* out_host, int64_t n_out);

/* Plan facts for reports: T_cc (Eq. 4, ops_per_element = 8) and T_mc
 * (Eq. 5, sizeof_data = 8) summed over the path of one slice. */
typedef struct {
  int64_t n_slices;          /* Π dims of the sliced bonds                               */
  int64_t n_out;             /* amplitudes returned by tn_sum_slices                     */
  int32_t n_steps;           /* N-1                                                     */
  int32_t n_tc_steps;        /* steps routed to the tcgen05 GEMM                         */
  double flops_per_slice;    /* Σ_steps T_cc (Eq. 4, 8 flop per complex MAC)             */
  double tc_flops_per_slice; /* the part of it executed on tensor cores                  */
  double bytes_per_slice;    /* Σ_steps T_mc (Eq. 5, 8 B per complex element)            */
  double peak_elements;      /* largest intermediate (elements)                          */
  int64_t device_bytes;      /* device memory held by the plan                           */
  int64_t arena_bytes;       /* liveness-planned intermediate arena                      */
  int64_t scratch_bytes;     /* fp16 operand-plane scratch of the largest tensor-core step */
  int64_t graph_replays;     /* slices executed by replaying the captured per-slice CUDA
                                graph (every slice after the first; TN_GRAPHS=0 disables) */
} tn_info;
/* TN_ERR_USAGE before tn_set_slices. */
TN_API tn_status tn_get_info(tn_ctx* ctx, tn_info* info);

/* Bit-exact bookkeeping dump (JSON): per step the pair (L259-262), J/m/n/k from the
 * Eq. 3 set rule (L225-228), T_cc (Eq. 4), T_mc (Eq. 5), routing, and the sparse-
 * merge gather tables (Eq. 7); root table; slice decode (L292-295).
 * Writes at most cap bytes (NUL-terminated if room) and the full length to *len. */
TN_API tn_status tn_plan_json(tn_ctx* ctx, char* buf, size_t cap, size_t* len);

/* Kernel-family timing inside tn_contract, for the roofline report (SURVEY.md §8 d:
 * achieved = algorithmic T_cc (Eq. 4) or bytes (Eq. 5) / measured device time).
 * When enabled, CUDA events bracket every launch of each kernel family on the
 * context stream; stats accumulate until reset.  family: 0 = tcgen05 GEMM,
 * 1 = operand prep (permute + scale + hi/lo split), 2 = SIMT einsum, 3 = slice
 * select + misc.  ms = summed event durations, flops = algorithmic T_cc of those
 * launches, bytes = algorithmic bytes (Eq. 5 operands + result; prep: read 8 B +
 * write 2 B per plane element). */
TN_API tn_status tn_set_profiling(tn_ctx* ctx, int enabled);
typedef struct { int64_t launches; double ms; double flops; double bytes; } tn_kernel_stats;
TN_API tn_status tn_get_kernel_stats(tn_ctx* ctx, int family, tn_kernel_stats* out);
/* Zero all kernel-family statistics (synchronises pending profiling events). */
TN_API tn_status tn_reset_kernel_stats(tn_ctx* ctx);
/* Per path step: device milliseconds accumulated while profiling is enabled, summed
 * over the slices contracted since the last reset, for kernel family `family` (0 GEMM,
 * 1 prep, 2 SIMT einsum, 3 misc) or all families (-1).  ms_out: host array of n
 * doubles (entries past the step count are 0).  Synchronises the context stream.
 * TN_ERR_USAGE on a null ctx, n < 0 or a bad family. */
TN_API tn_status tn_get_step_stats(tn_ctx* ctx, int family, int64_t n, double* ms_out);

/* Stand-alone complex GEMM through the same kernels (unit tests, accumulator
 * probes): one step of TTGT's GEMM (L248) in the 3xFP16 split of Eq. 8 (L367-377,
 * L383-386) or 1-pass (L442), batched with gathers as the sparse einsum (L354).  Device pointers, complex64 interleaved:
 *   A[ga][m][k], B[gb][n][k] (both K-contiguous), C[J][m][n];
 *   ia[J], ib[J] (device int32, may be NULL = slab 0) select the A / B slab of
 *   batch j (the gather of a sparse einsum, Eq. 7 / L354).
 *   passes = 3 (hi/lo split) or 1; force_simt != 0 runs the SIMT kernel instead.
 *   format = operand format of the tensor-core path (Fig. 4):
 *   0 fp16 (the product path), 1 bf16 (3xBF16 / 1xBF16), 2 tf32 (3xTF32 of Eq. 8 as
 *   printed / 1xTF32, kind::tf32); formats 1 and 2 run single-CTA tiles.
 * Synchronous on the context stream.  TN_ERR_USAGE on bad sizes, passes or format. */
TN_API tn_status tn_cgemm(tn_ctx* ctx, const float* A, const float* B, float* C,
                   int64_t J, int64_t m, int64_t n, int64_t k, int64_t ga, int64_t gb,
                   const int32_t* ia, const int32_t* ib, int passes, int force_simt, int format);

/* Thread-local message of the last failing call on this thread (never NULL). */
TN_API const char* tn_last_error(void);
/* Library version string (static storage). */
TN_API const char* tn_version(void);
/* 1 if a fused producer epilogue of this context saturated an fp16 plane since the
 * last tn_reset_accumulator (synchronises the context stream), 0 if not, -1 on a bad
 * or host-only context.  See tn_sum_slices. */
TN_API int tn_last_overflow(tn_ctx* ctx);
/* Release every device block (through the allocator) and the context; waits for
 * the context stream.  NULL is a no-op. */
TN_API void tn_destroy(tn_ctx* ctx);

#ifdef __cplusplus
}
#endif
#endif /* TN_B200_H */
