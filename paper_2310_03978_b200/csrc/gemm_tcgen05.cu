// tcgen05 / TMEM / TMA complex GEMM for sm_100a — the tensor-core hot loop of
// the sliced contraction.
//
//   C[j][m][n] = 2^-(sA+sB) * Σ_k  A[ia(j)][m][k] · B[ib(j)][n][k]     (complex)
//
// Operands arrive as K-contiguous fp16 planes (re_hi, im_hi[, re_lo, im_lo]) of
// the rescaled values x*2^s, written by the prep kernel.  The complex product
// is formed from real MMAs on the planes, using the instruction descriptor's
// negate-A bit for the -Ai·Bi term (no real embedding of B is materialised):
//   Cr += Ar·Br - Ai·Bi,   Ci += Ar·Bi + Ai·Br.
// Extended precision (3 passes) follows Eq. 8 with fp16
// in place of tf32 (the 3xFP16 variant, L383-386): per real product
//   x·y ≈ x_big·y_small + x_small·y_big + x_big·y_big   (small·small dropped,
// small terms issued first).  Mixed mode (1 pass) keeps only big·big (L442).
//
// Accumulator promotion.  tcgen05 kind::f16 truncates (RZ) its fp32 TMEM
// accumulator after every MMA (measured: tools/accum_probe.py, DESIGN.md
// "Numerics").  A truncating chain of T MMAs biases the result toward zero by
// ≈0.37·2^-24·T relative, so a K-loop of thousands of MMAs drifts by 1e-5..1e-3.
// The MMA warp therefore restarts the TMEM accumulator every `kchunk` k-blocks
// and the epilogue warps add each finished chunk into an fp32 register sum with
// round-to-nearest: the bias becomes ≈0.37·2^-24·(MMAs per chunk) independently
// of K, and the chunk sums combine without bias.
//
// Operand formats (template FMT, Fig. 4): fp16 planes (the product
// path), bf16 planes (3xBF16, L383) or tf32 in 32-bit containers (3xTF32, Eq. 8 as
// printed, kind::tf32).  A k-block is always 64 B of K per row (32 fp16/bf16 or 16
// tf32 elements) and an MMA consumes 32 B of it, so the smem layout, descriptors and
// issue order are the same for all three; only the instruction kind, the descriptor's
// operand-format fields and the TMA element type differ.
//
// Sparse einsum (Eq. 7) is the same kernel: batch j selects the A and
// B slabs through the gather tables ia/ib — the "separate pointers for each
// matrix of the batched GEMM" of L354 become TMA slab coordinates, so no
// gathered copies are materialised.
//
// Structure (one CTA per SM, persistent, 12 warps = 3 warpgroups):
//   warp 0      TMA producer: 4D tensor-map loads (K, rows, slab, plane), box
//               32x128, SWIZZLE_64B, into a STAGES-deep smem ring (mbarrier tx).
//   warp 1      TMEM allocator (512 cols) + single-thread tcgen05.mma issuer,
//               kind::f16, M=128 N=128 K=16; a chunk accumulator Cr|Ci is 256
//               TMEM columns, double-buffered; tcgen05.commit frees smem stages
//               and hands finished chunks to the epilogue.
//   warps 2-3   idle (they complete warpgroup 0, whose register budget is lowered
//               to 40 per thread with setmaxnreg so that the two epilogue
//               warpgroups can raise theirs to 232: the epilogue's 64+64 fp32
//               column sums and a 32+32-column TMEM load fit without spills)
//   warps 4-11  epilogue: warp (quadrant q, half h) owns TMEM lanes 32q..32q+31
//               and output columns 64h..64h+63 of both Cr and Ci; tcgen05.ld
//               32x32b.x32 -> fp32 RN register sums of the chunks scaled by
//               2^-(sA+sB) and store complex64 (or fused fp64 accumulate into the
//               slice sum, a8) + absmax of the result for the consumer's rescale.
#include "tn_internal.h"
#include <cstdio>

namespace tn {
namespace {

constexpr int BM = 128, BN = 128, BK = 32;          // BK in complex k (64 B fp16 rows)
enum { FMT_F16 = 0, FMT_BF16 = 1, FMT_TF32 = 2 };
// k elements per 64-B k-block row
template <int FMT> __host__ __device__ constexpr int bk_elems() { return FMT == FMT_TF32 ? 16 : 32; }
constexpr int PLANE_TILE = 128 * BK * 2;            // 8 KiB per plane tile
constexpr uint32_t TMEM_COLS = 512;

// PAIR = CTA pair (cta_group::2, cluster of 2): the MMA tile is 256 x 128; each CTA
// stages its own 128 rows of A and half (64 rows) of B, so a CTA's smem supplies
// 6 KiB per M=256 MMA instead of 8 KiB per M=128 MMA (smem bandwidth, not the
// tensor pipe, bounds the single-CTA kernel: DESIGN.md "GEMM structure").
template <int PASSES, bool PAIR = false>
struct Cfg {
  static constexpr int PLANES = PASSES == 3 ? 4 : 2;
  static constexpr int B_TILE = PAIR ? PLANE_TILE / 2 : PLANE_TILE;   // per-plane B tile
  static constexpr int STAGE_BYTES = PLANES * (PLANE_TILE + B_TILE);
  static constexpr int STAGES = PAIR ? (PASSES == 3 ? 4 : 8) : (PASSES == 3 ? 3 : 6);
  static constexpr int SMEM_BYTES =
      STAGES * STAGE_BYTES + 1024 /*align*/ + 256 /*barriers*/ + 2 * BN * 8 /*column offsets*/;
  static constexpr int TILE_M = PAIR ? 2 * BM : BM;
};
// per-warp staging tile for plane outputs whose unit-stride dim is a row dim
// (8 epilogue warps only: 16 would exceed the 227 KB shared-memory limit)
template <int EW>
constexpr int stage_bytes() { return EW == 8 ? EW * 32 * 10 * 8 : 0; }

// instruction descriptor: D=f32 (bits 4-5 = 1), A/B format at bits 7-9 / 10-12 (kind::f16:
// 0 = f16, 1 = bf16; kind::tf32: 2 = tf32), K-major, N>>3 at bits 17-22, M>>4 at bits
// 24-28; bit 13 = negate A.
template <bool PAIR, int FMT = FMT_F16>
struct Idesc {
  static constexpr uint32_t AB = FMT == FMT_F16 ? 0u : (FMT == FMT_BF16 ? 1u : 2u);
  static constexpr uint32_t POS = (1u << 4) | (AB << 7) | (AB << 10) | ((uint32_t)(BN >> 3) << 17) |
                                  ((uint32_t)((PAIR ? 2 * BM : BM) >> 4) << 24);
};

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}

__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
               "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n.reg .pred P1;\nTN_WAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n"
      "@!P1 bra TN_WAIT_%=;\n}" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}
// shared::cluster address of the same smem variable in CTA `rank` of the cluster
__device__ __forceinline__ uint32_t map_rank(const void* p, uint32_t rank) {
  uint32_t r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(smem_u32(p)), "r"(rank));
  return r;
}
// Arrive on a barrier of another CTA of the cluster.  Only TMEM reads are ordered
// by this arrive (tcgen05.wait::ld + fence::before_thread_sync precede it), so the
// default CTA-scope release suffices; a cluster-scope release compiles to a
// MEMBAR.ALL.GPU + ERRBAR per drained chunk (43 % of the epilogue's stall samples).
__device__ __forceinline__ void mbar_arrive_remote(uint32_t cluster_addr) {
  asm volatile("mbarrier.arrive.shared::cluster.b64 _, [%0];" ::"r"(cluster_addr) : "memory");
}
__device__ __forceinline__ uint32_t cluster_rank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
__device__ __forceinline__ void cluster_sync() {
  asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;" ::
                   : "memory");
}

__device__ __forceinline__ void tma_load_4d(const CUtensorMap* map, void* dst, uint64_t* bar, int c0,
                                            int c1, int c2, int c3) {
  asm volatile(
      "cp.async.bulk.tensor.4d.shared::cluster.global.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%3, %4, %5, %6}], [%2];" ::"r"(smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(smem_u32(bar)), "r"(c0), "r"(c1), "r"(c2), "r"(c3)
      : "memory");
}

// operand loads with an L2 eviction-priority hint (evict_last: the A / B panels are
// re-read by the other column / row tiles of their wave, while the output streams
// past them through L2)
__device__ __forceinline__ void tma_load_4d_hint(const CUtensorMap* map, void* dst, uint64_t* bar, int c0,
                                                 int c1, int c2, int c3, uint64_t pol) {
  asm volatile(
      "cp.async.bulk.tensor.4d.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint"
      " [%0], [%1, {%3, %4, %5, %6}], [%2], %7;" ::"r"(smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(smem_u32(bar)), "r"(c0), "r"(c1), "r"(c2), "r"(c3), "l"(pol)
      : "memory");
}
__device__ __forceinline__ void tma_load_4d_pair_hint(const CUtensorMap* map, void* dst, uint32_t bar_cluster,
                                                      int c0, int c1, int c2, int c3, uint64_t pol) {
  asm volatile(
      "cp.async.bulk.tensor.4d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint"
      " [%0], [%1, {%3, %4, %5, %6}], [%2], %7;" ::"r"(smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(bar_cluster), "r"(c0), "r"(c1), "r"(c2), "r"(c3), "l"(pol)
      : "memory");
}

// CTA-pair TMA: the destination is this CTA's smem, the completion goes to the
// leader CTA's barrier (bar_cluster = its shared::cluster address)
__device__ __forceinline__ void tma_load_4d_pair(const CUtensorMap* map, void* dst, uint32_t bar_cluster,
                                                 int c0, int c1, int c2, int c3) {
  asm volatile(
      "cp.async.bulk.tensor.4d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%3, %4, %5, %6}], [%2];" ::"r"(smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(bar_cluster), "r"(c0), "r"(c1), "r"(c2), "r"(c3)
      : "memory");
}

// UMMA shared-memory descriptor, K-major, SWIZZLE_64B: 8-row atoms of 64 B rows,
// SBO = 512 B between atoms, LBO unused (1), version 1 (sm_100), layout 4.
__device__ __forceinline__ uint64_t sdesc(uint32_t addr) {
  return (uint64_t)((addr >> 4) & 0x3FFFu) | ((uint64_t)1 << 16) | ((uint64_t)(512 >> 4) << 32) |
         ((uint64_t)1 << 46) | ((uint64_t)4 << 61);
}

// MMA issue: called by the whole (converged) MMA warp; one lane is elected inside
// the asm, so every operand stays warp-uniform (uniform registers, no per-MMA
// ELECT / R2UR.BROADCAST loop as when a single-lane branch issues it).
template <bool PAIR, int FMT = FMT_F16>
__device__ __forceinline__ void mma_t(uint32_t d, uint64_t a, uint64_t b, uint32_t idesc,
                                      uint32_t accumulate) {
  if constexpr (FMT == FMT_TF32) {
    if constexpr (PAIR)
      asm volatile(
          "{\n.reg .pred p, e;\nelect.sync _|e, 0xffffffff;\nsetp.ne.b32 p, %4, 0;\n"
          "@e tcgen05.mma.cta_group::2.kind::tf32 [%0], %1, %2, %3, p;\n}" ::"r"(d),
          "l"(a), "l"(b), "r"(idesc), "r"(accumulate));
    else
      asm volatile(
          "{\n.reg .pred p, e;\nelect.sync _|e, 0xffffffff;\nsetp.ne.b32 p, %4, 0;\n"
          "@e tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n}" ::"r"(d),
          "l"(a), "l"(b), "r"(idesc), "r"(accumulate));
  } else if constexpr (PAIR)
    asm volatile(
        "{\n.reg .pred p, e;\nelect.sync _|e, 0xffffffff;\nsetp.ne.b32 p, %4, 0;\n"
        "@e tcgen05.mma.cta_group::2.kind::f16 [%0], %1, %2, %3, p;\n}" ::"r"(d),
        "l"(a), "l"(b), "r"(idesc), "r"(accumulate));
  else
    asm volatile(
        "{\n.reg .pred p, e;\nelect.sync _|e, 0xffffffff;\nsetp.ne.b32 p, %4, 0;\n"
        "@e tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n}" ::"r"(d),
        "l"(a), "l"(b), "r"(idesc), "r"(accumulate));
}

// commit (elected lane of the converged MMA warp): arrive on `bar` when the issued
// MMAs retire (pair: on the barrier at the same offset in both CTAs)
template <bool PAIR>
__device__ __forceinline__ void mma_commit_t(uint64_t* bar) {
  if constexpr (PAIR)
    asm volatile(
        "{\n.reg .pred e;\nelect.sync _|e, 0xffffffff;\n"
        "@e tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64"
        " [%0], %1;\n}" ::"r"(smem_u32(bar)),
        "h"((uint16_t)3)
        : "memory");
  else
    asm volatile(
        "{\n.reg .pred e;\nelect.sync _|e, 0xffffffff;\n"
        "@e tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n}" ::"r"(
            smem_u32(bar))
        : "memory");
}

__device__ __forceinline__ void fence_before() {
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
}
__device__ __forceinline__ void fence_after() {
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
}

#define TN_LD32(r, taddr)                                                                        \
  asm volatile(                                                                                  \
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14," \
      "%15,%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"               \
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]),      \
        "=r"(r[7]), "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]),  \
        "=r"(r[14]), "=r"(r[15]), "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]),            \
        "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]), "=r"(r[24]), "=r"(r[25]),            \
        "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])             \
      : "r"(taddr))

__device__ __forceinline__ void tmem_wait_ld() {
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
}

// Row-contiguous output through a per-warp smem stage.  The TMEM layout gives each
// lane one row, so a direct store instruction touches 32 rows with 16 B each (32
// half-filled sectors: the LSU, not DRAM, bounds output-heavy GEMMs).  Here the warp
// writes 8 columns of its 32 rows into smem (64-B rows, 16-B units XOR-swizzled by
// bits 1-2 of the row: conflict-free both ways), then each store instruction writes
// 8 rows x 64 contiguous bytes.  The four row bases a lane stores to are fetched once
// (not per column group), the four reads of a group are issued before its stores, and
// padding rows are masked by predicated stores (no divergent branch per store).
// base = element offset of this lane's row start (column n0); valid = the row exists;
// ncols = columns to write (a multiple of 8, <= WC: narrow GEMMs write N < 64).
__device__ __forceinline__ void st_global_v4_pred(void* p, float4 v, bool ok) {
  asm volatile("{\n.reg .pred q;\nsetp.ne.b32 q, %5, 0;\n@q st.global.v4.f32 [%0], {%1,%2,%3,%4};\n}" ::"l"(p),
               "f"(v.x), "f"(v.y), "f"(v.z), "f"(v.w), "r"((int)ok)
               : "memory");
}
template <int WC>
__device__ __forceinline__ void store_rows_staged(float4* buf, const float* sr, const float* si,
                                                  float2* C, int64_t base, bool valid, int lane,
                                                  float& amax, int ncols = WC) {
  const unsigned vmask = __ballot_sync(0xffffffffu, valid);
  const int c = lane & 3;
  float2* rowp[4];
  bool ok[4];
  int slot[4];
#pragma unroll
  for (int q = 0; q < 4; ++q) {
    const int r = (lane >> 2) + 8 * q;
    rowp[q] = C + __shfl_sync(0xffffffffu, base, r) + 2 * c;
    ok[q] = (vmask >> r) & 1u;
    slot[q] = r * 4 + (c ^ ((r >> 1) & 3));
  }
#pragma unroll
  for (int i = 0; i < WC; i += 8) {
    if (i >= ncols) break;
#pragma unroll
    for (int cc = 0; cc < 4; ++cc) {
      const float r0 = sr[i + 2 * cc], i0 = si[i + 2 * cc], r1 = sr[i + 2 * cc + 1], i1 = si[i + 2 * cc + 1];
      buf[lane * 4 + (cc ^ ((lane >> 1) & 3))] = make_float4(r0, i0, r1, i1);
      if (valid) amax = fmaxf(amax, fmaxf(fmaxf(fabsf(r0), fabsf(i0)), fmaxf(fabsf(r1), fabsf(i1))));
    }
    __syncwarp();
    float4 v[4];
#pragma unroll
    for (int q = 0; q < 4; ++q) v[q] = buf[slot[q]];
#pragma unroll
    for (int q = 0; q < 4; ++q) st_global_v4_pred(rowp[q] + i, v[q], ok[q]);
    __syncwarp();
  }
}

// 256-bit global store (STG.256: one full 32-B sector per lane)
__device__ __forceinline__ void st_global_v8(void* p, const uint32_t* v) {
  asm volatile("st.global.v8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"l"(p), "r"(v[0]), "r"(v[1]), "r"(v[2]),
               "r"(v[3]), "r"(v[4]), "r"(v[5]), "r"(v[6]), "r"(v[7])
               : "memory");
}

// shared-memory load through an explicit ld.shared (the column table is reached through a
// pointer the compiler cannot prove shared, which costs a generic LD per column)
__device__ __forceinline__ int64_t lds64(const int64_t* p) {
  int64_t v;
  asm volatile("ld.shared.s64 %0, [%1];" : "=l"(v) : "r"(smem_u32(p)));
  return v;
}

// Tile index -> (j, mt, nt).  Tiles of one batch are visited in groups of
// `group_m` tile rows, column-major inside a group, so the ~148 tiles resident
// at once share few A and B panels in L2.
__device__ __forceinline__ void decode_tile(const GemmArgs& a, int64_t tile, int& j, int& mt, int& nt) {
  const int64_t per_j = (int64_t)a.tiles_m * a.tiles_n;
  j = (int)(tile / per_j);
  const int rem = (int)(tile % per_j);
  if (a.group_m > 1) {
    const int gsz = a.group_m * a.tiles_n;
    const int g = rem / gsz;
    const int first = g * a.group_m;
    const int gm = min(a.tiles_m - first, a.group_m);
    const int r = rem % gsz;
    mt = first + r % gm;
    nt = r / gm;
  } else {
    mt = rem / a.tiles_n;
    nt = rem % a.tiles_n;
  }
}

constexpr int EPI_WARP0 = 4;   // first epilogue warp (warpgroup 1)
constexpr int REG_LOW = 40, REG_HIGH = 232;   // setmaxnreg budgets: warpgroup 0 / epilogue

template <int PASSES, int EW, bool PAIR, int FMT = FMT_F16>
__global__ void __launch_bounds__(32 * EPI_WARP0 + 32 * EW, 1) cgemm_tcgen05_kernel(const __grid_constant__ GemmArgs args) {
  static_assert(EW == 8, "two epilogue warpgroups");
  using C = Cfg<PASSES, PAIR>;
  constexpr int BKE = bk_elems<FMT>();   // k elements per k-block
  constexpr int PLANES = C::PLANES, STAGES = C::STAGES;
  // narrow GEMMs (N <= 64): N = 64 MMAs (half the tensor work of the padded 128-wide
  // tile); the pair's B halves become 32 rows each
  const uint32_t IDESC = args.narrow ? ((Idesc<PAIR, FMT>::POS & ~(0x3Fu << 17)) | ((uint32_t)(64 >> 3) << 17))
                                     : Idesc<PAIR, FMT>::POS;
  const uint32_t IDESC_NEG = IDESC | (1u << 13);
  extern __shared__ uint8_t smem_raw[];
  // 1024-B aligned base by an offset into the shared array (not an integer round trip, which
  // would hide the address space and turn every smem access through it into a generic one)
  uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + STAGES * C::STAGE_BYTES);
  uint64_t* empty = full + STAGES;
  // chunk accumulators in TMEM: 2 buffers of 256 columns (Cr | Ci, N = 128), or for narrow
  // GEMMs (N <= 64) 4 buffers of 128 columns, two per epilogue half: the halves then
  // drain alternate tiles (both busy, 4 chunks in flight) instead of half of the
  // epilogue idling on the dead columns 64..127
  uint64_t* cfull = empty + STAGES;     // chunk accumulator ready (MMA -> epilogue)
  uint64_t* cempty = cfull + 4;         // chunk accumulator drained (epilogue -> MMA)
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(cempty + 4);
  // general output map: per-tile column offsets, double-buffered by tile parity
  int64_t* noff_tab = reinterpret_cast<int64_t*>(smem + STAGES * C::STAGE_BYTES + 256);
  float2* stage_buf = reinterpret_cast<float2*>(noff_tab + 2 * BN);   // [warp][32][9]

  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  const int kblocks = (args.K + BKE - 1) / BKE;
  const int kchunk = (args.kchunk > 0 && args.kchunk < kblocks) ? args.kchunk : kblocks;
  const int nchunks = (kblocks + kchunk - 1) / kchunk;
  // pair: CTA rank in the cluster; tiles are scheduled per pair
  const uint32_t rank = PAIR ? cluster_rank() : 0;
  const int64_t unit = PAIR ? (blockIdx.x >> 1) : blockIdx.x;
  const int64_t units = PAIR ? (gridDim.x >> 1) : gridDim.x;

  if (threadIdx.x == 0) {
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    for (int s = 0; s < 4; ++s) {
      mbar_init(&cfull[s], 1);
      // drained by every epilogue warp (narrow: by one half), of both CTAs for a pair
      const int drainers = args.narrow ? EW / 2 : EW;
      mbar_init(&cempty[s], PAIR ? 2 * drainers : drainers);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&args.mapA)) : "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(PAIR ? &args.mapB2 : &args.mapB))
                 : "memory");
  }
  if (warp == 1) {
    if constexpr (PAIR) {
      asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                       smem_u32(tmem_slot)),
                   "r"(TMEM_COLS));
      asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;");
    } else {
      asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                       smem_u32(tmem_slot)),
                   "r"(TMEM_COLS));
      asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
  }
  fence_before();
  if constexpr (PAIR) cluster_sync(); else __syncthreads();
  fence_after();
  const uint32_t tmem_base = *tmem_slot;

  // register split (per SM sub-partition: REG_LOW + 2 x REG_HIGH <= 512 per lane slot);
  // each role's code sits inside the branch that set its budget, so ptxas allocates it
  // under that budget
  if (warp < EPI_WARP0) {
  asm volatile("setmaxnreg.dec.sync.aligned.u32 %0;" ::"n"(REG_LOW));
  if (warp == 0) {
    if (lane == 0) {
      // ---------------------------------------------------------------- TMA producer
      // pair: each CTA loads its own A rows and its half of B into its own smem;
      // completion bytes of both CTAs go to the leader's full barrier
      int stage = 0;
      uint32_t phase = 0;
      unsigned long long target = 0;
      uint64_t pol = 0;
      if (args.l2hint) asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(pol));
      const int per_unit = PAIR ? 2 : 1;
      for (int64_t tile = unit; tile < args.n_tiles; tile += units) {
        if (args.wave_sync) {
          // wave w = tile / units: producers with a tile in it = per_unit * min(units, rest)
          const int64_t w0 = tile - unit;
          const int64_t rest = args.n_tiles - w0;
          target += (unsigned long long)(per_unit * (rest < units ? rest : units));
          atomicAdd(args.wave_ctr, 1ull);
          for (int spin = 0; spin < 20000; ++spin) {   // bounded: a locality hint, never a hang
            unsigned long long v;
            asm volatile("ld.acquire.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(args.wave_ctr) : "memory");
            if (v >= target) break;
            __nanosleep(64);
          }
        }
        int j, mt, nt;
        decode_tile(args, tile, j, mt, nt);
        const int sa = args.ia ? args.ia[j] : 0;
        const int sb = args.blk_slab_b ? args.blk_slab_b[mt] : (args.ib ? args.ib[j] : 0);
        const int arow = mt * C::TILE_M + (int)rank * BM;
        const int brow = nt * BN + (int)rank * (args.narrow ? 32 : BN / 2);
        for (int kb = 0; kb < kblocks; ++kb) {
          mbar_wait(&empty[stage], phase ^ 1);
          uint8_t* st = smem + stage * C::STAGE_BYTES;
          if constexpr (PAIR) {
            const uint32_t fb = map_rank(&full[stage], 0);
            if (rank == 0) mbar_expect_tx(&full[stage], 2 * C::STAGE_BYTES);
            if (args.l2hint) {
#pragma unroll
              for (int p = 0; p < PLANES; ++p)
                tma_load_4d_pair_hint(&args.mapA, st + p * PLANE_TILE, fb, kb * BKE, arow, sa, p, pol);
#pragma unroll
              for (int p = 0; p < PLANES; ++p)
                tma_load_4d_pair_hint(&args.mapB2, st + PLANES * PLANE_TILE + p * C::B_TILE, fb, kb * BKE,
                                      brow, sb, p, pol);
            } else {
#pragma unroll
              for (int p = 0; p < PLANES; ++p)
                tma_load_4d_pair(&args.mapA, st + p * PLANE_TILE, fb, kb * BKE, arow, sa, p);
#pragma unroll
              for (int p = 0; p < PLANES; ++p)
                tma_load_4d_pair(&args.mapB2, st + PLANES * PLANE_TILE + p * C::B_TILE, fb, kb * BKE,
                                 brow, sb, p);
            }
          } else {
            mbar_expect_tx(&full[stage], C::STAGE_BYTES);
            if (args.l2hint) {
#pragma unroll
              for (int p = 0; p < PLANES; ++p)
                tma_load_4d_hint(&args.mapA, st + p * PLANE_TILE, &full[stage], kb * BKE, arow, sa, p, pol);
#pragma unroll
              for (int p = 0; p < PLANES; ++p)
                tma_load_4d_hint(&args.mapB, st + PLANES * PLANE_TILE + p * C::B_TILE, &full[stage],
                                 kb * BKE, brow, sb, p, pol);
            } else {
#pragma unroll
              for (int p = 0; p < PLANES; ++p)
                tma_load_4d(&args.mapA, st + p * PLANE_TILE, &full[stage], kb * BKE, arow, sa, p);
#pragma unroll
              for (int p = 0; p < PLANES; ++p)
                tma_load_4d(&args.mapB, st + PLANES * PLANE_TILE + p * C::B_TILE, &full[stage],
                            kb * BKE, brow, sb, p);
            }
          }
          if (++stage == STAGES) {
            stage = 0;
            phase ^= 1;
          }
        }
      }
    }
  } else if (warp == 1) {
    if (rank == 0) {
      // ---------------------------------------------------------------- MMA issuer
      // (whole warp, converged; one elected lane issues each tcgen05 instruction)
      int stage = 0;
      uint32_t phase = 0;
      int cb = 0;                 // wide: next chunk buffer (0/1)
      int hb = 0;                 // narrow: next buffer of each epilogue half's pair (bits 0, 1)
      uint32_t bph = 0;           // phase bit of each chunk buffer
      int b = 0;
      int titer = 0;
      for (int64_t tile = unit; tile < args.n_tiles; tile += units, ++titer) {
        for (int kb = 0; kb < kblocks; ++kb) {
          const int kin = kb % kchunk;
          if (kin == 0) {
            b = args.narrow ? 2 * (titer & 1) + ((hb >> (titer & 1)) & 1) : cb;
            // chunk buffer drained by the epilogue (pair: by both CTAs')
            mbar_wait(&cempty[b], ((bph >> b) & 1u) ^ 1u);
            fence_after();
          }
          const uint32_t d_re = tmem_base + (args.narrow ? b * 128 : b * 256);
          const uint32_t d_im = d_re + (args.narrow ? 64 : 128);
          mbar_wait(&full[stage], phase);
          fence_after();
          const uint32_t st = smem_u32(smem + stage * C::STAGE_BYTES);
          const uint32_t sb0 = st + PLANES * PLANE_TILE;
          if (PASSES == 3) {
            // Eq. 8, small terms first: every hi·lo / lo·hi MMA of the stage is
            // issued while the chunk accumulator is still ~2^-11 of its final size,
            // so the per-MMA RZ truncation only bites on the big·big MMAs.
#pragma unroll
            for (int kk = 0; kk < 2; ++kk) {   // 2 x 32 B of K per 64-B row
              const uint32_t koff = kk * 32;   // 16 fp16 / 8 tf32 = 32 B along K inside the swizzle row
              const uint64_t ar = sdesc(st + 0 * PLANE_TILE + koff);
              const uint64_t ai = sdesc(st + 1 * PLANE_TILE + koff);
              const uint64_t br = sdesc(sb0 + 0 * C::B_TILE + koff);
              const uint64_t bi = sdesc(sb0 + 1 * C::B_TILE + koff);
              const uint64_t arl = sdesc(st + 2 * PLANE_TILE + koff);
              const uint64_t ail = sdesc(st + 3 * PLANE_TILE + koff);
              const uint64_t brl = sdesc(sb0 + 2 * C::B_TILE + koff);
              const uint64_t bil = sdesc(sb0 + 3 * C::B_TILE + koff);
              const uint32_t acc0 = (kin | kk) != 0;
              // real part: Ar·Br - Ai·Bi (cross terms)
              mma_t<PAIR, FMT>(d_re, ar, brl, IDESC, acc0);
              mma_t<PAIR, FMT>(d_re, arl, br, IDESC, 1);
              mma_t<PAIR, FMT>(d_re, ail, bi, IDESC_NEG, 1);
              mma_t<PAIR, FMT>(d_re, ai, bil, IDESC_NEG, 1);
              // imaginary part: Ar·Bi + Ai·Br (cross terms)
              mma_t<PAIR, FMT>(d_im, ar, bil, IDESC, acc0);
              mma_t<PAIR, FMT>(d_im, arl, bi, IDESC, 1);
              mma_t<PAIR, FMT>(d_im, ai, brl, IDESC, 1);
              mma_t<PAIR, FMT>(d_im, ail, br, IDESC, 1);
            }
#pragma unroll
            for (int kk = 0; kk < 2; ++kk) {   // 2 x 32 B of K per 64-B row
              const uint32_t koff = kk * 32;
              const uint64_t ar = sdesc(st + 0 * PLANE_TILE + koff);
              const uint64_t ai = sdesc(st + 1 * PLANE_TILE + koff);
              const uint64_t br = sdesc(sb0 + 0 * C::B_TILE + koff);
              const uint64_t bi = sdesc(sb0 + 1 * C::B_TILE + koff);
              mma_t<PAIR, FMT>(d_re, ar, br, IDESC, 1);        // big·big last
              mma_t<PAIR, FMT>(d_re, ai, bi, IDESC_NEG, 1);
              mma_t<PAIR, FMT>(d_im, ar, bi, IDESC, 1);
              mma_t<PAIR, FMT>(d_im, ai, br, IDESC, 1);
            }
          } else {
#pragma unroll
            for (int kk = 0; kk < 2; ++kk) {   // 2 x 32 B of K per 64-B row
              const uint32_t koff = kk * 32;
              const uint64_t ar = sdesc(st + 0 * PLANE_TILE + koff);
              const uint64_t ai = sdesc(st + 1 * PLANE_TILE + koff);
              const uint64_t br = sdesc(sb0 + 0 * C::B_TILE + koff);
              const uint64_t bi = sdesc(sb0 + 1 * C::B_TILE + koff);
              const uint32_t acc0 = (kin | kk) != 0;
              mma_t<PAIR, FMT>(d_re, ar, br, IDESC, acc0);
              mma_t<PAIR, FMT>(d_re, ai, bi, IDESC_NEG, 1);
              mma_t<PAIR, FMT>(d_im, ar, bi, IDESC, acc0);
              mma_t<PAIR, FMT>(d_im, ai, br, IDESC, 1);
            }
          }
          mma_commit_t<PAIR>(&empty[stage]);   // frees the smem stage(s) when these MMAs retire
          if (++stage == STAGES) {
            stage = 0;
            phase ^= 1;
          }
          if (kin == kchunk - 1 || kb == kblocks - 1) {
            mma_commit_t<PAIR>(&cfull[b]);     // chunk accumulator ready for the epilogue(s)
            bph ^= 1u << b;
            if (args.narrow) hb ^= 1 << (titer & 1);
            else cb ^= 1;
          }
        }
      }
    }
  }
  } else {
    asm volatile("setmaxnreg.inc.sync.aligned.u32 %0;" ::"n"(REG_HIGH));
    // ---------------------------------------------------------------- epilogue (warps 4..11)
    // warp (quadrant q, sub s) owns TMEM lanes 32q..32q+31 and WC output columns
    // WC*s .. WC*s+WC-1 of both Cr and Ci (WC = 64 with 8 warps, 32 with 16)
    constexpr int WC = 512 / EW;
    const int quad = warp & 3;                  // TMEM lane quadrant this warp may access
    const int half = (warp - EPI_WARP0) >> 2;
    const int colh = args.narrow ? 0 : half;    // column half (narrow: the halves split tiles)
    const int row = quad * 32 + lane;
    // the operands carry 2^sA and 2^sB (|s| <= 120 each): 2^-(sA+sB) may leave the fp32
    // range, so 2^-sA is folded into the chunk promotion and 2^-sB applied once per tile
    // both exponents folded into the chunk scale when 2^-(sA+sB) is a normal fp32 (the
    // final per-tile multiply is then skipped)
    const int sab_all = *args.scaleA + *args.scaleB;
    const bool fold_ab = sab_all >= -100 && sab_all <= 100;
    const float scale = ldexpf(1.0f, fold_ab ? -sab_all : -*args.scaleA);
    const float scale_b = ldexpf(1.0f, -*args.scaleB);
    // fused plane output: consumer exponent sC = max(bound, delayed scaling); the planes
    // hold x * 2^sC = acc * 2^(sC - sA - sB)
    int plane_sc = 0;
    if (args.out_planes) {
      const int sab = *args.scaleA + *args.scaleB;
      plane_sc = min(120, max(-120, max(sab + args.plane_exp, *args.plane_pexp)));
      if (blockIdx.x == 0 && threadIdx.x == 32 * EPI_WARP0) *args.plane_scale_out = plane_sc;
    }
    bool plane_ovf = false;
    float amax = 0.f;
    int cb = 0, eb = 0;
    uint32_t bph = 0;                       // phase bit of each chunk buffer
    int titer = 0;
    int tab_nt = -1, tab_sel = 0;           // out_gen column table: tile column it holds
    // out_gen column offsets of tile column nt into the table buffer sel (all epilogue warps)
    auto col_table = [&](int nt_, int sel) {
      int64_t* tab = noff_tab + (sel & 1) * BN;
      const int et = threadIdx.x - 32 * EPI_WARP0;
      if (et < BN) {
        int64_t t = (int64_t)nt_ * BN + et, off = 0;
        for (int q = args.n_qo - 1; q >= 0; --q) {
          const int sh = args.qo_sh[q];
          off += (t & ((int64_t(1) << sh) - 1)) * args.qo_str[q];
          t >>= sh;
        }
        tab[et] = off;
      }
      asm volatile("bar.sync 1, %0;" ::"r"(32 * EW) : "memory");
    };
    if (args.narrow && args.out_gen) {      // one tile column: the table once, before the halves part
      tab_nt = 0;
      tab_sel = 1;
      col_table(0, tab_sel);
    }
    const int64_t t_first = unit + (args.narrow ? half * units : 0);
    const int64_t t_step = args.narrow ? 2 * units : units;
    for (int64_t tile = t_first; tile < args.n_tiles; tile += t_step, ++titer) {
      int j, mt, nt;
      decode_tile(args, tile, j, mt, nt);
      float sr[WC], si[WC];
#pragma unroll
      for (int i = 0; i < WC; ++i) { sr[i] = 0.f; si[i] = 0.f; }
      // column half entirely beyond N (narrow GEMMs): nothing to drain, only release
      const bool cols_live = (int)(nt * BN + colh * WC) < args.N;
      for (int ch = 0; ch < nchunks; ++ch) {
        const int b = args.narrow ? 2 * half + eb : cb;
        mbar_wait(&cfull[b], (bph >> b) & 1u);
        fence_after();
        const uint32_t tb = tmem_base + ((uint32_t)(quad * 32) << 16) +
                            (args.narrow ? b * 128 : b * 256 + half * WC);
        const uint32_t im_off = args.narrow ? 64 : 128;
        if (cols_live) {
#pragma unroll
          for (int c = 0; c < WC / 32; ++c) {
            if (c > 0 && nt * BN + colh * WC + c * 32 >= args.N) break;   // narrow: dead 32-column group
            uint32_t vr[32], vi[32];
            TN_LD32(vr, tb + c * 32);
            TN_LD32(vi, tb + im_off + c * 32);
            tmem_wait_ld();
#pragma unroll
            for (int i = 0; i < 32; ++i) {     // fp32 round-to-nearest promotion of the chunk,
              // with the power-of-two output scale folded in (exact: commutes with RN)
              sr[c * 32 + i] = fmaf(__uint_as_float(vr[i]), scale, sr[c * 32 + i]);
              si[c * 32 + i] = fmaf(__uint_as_float(vi[i]), scale, si[c * 32 + i]);
            }
          }
        }
        fence_before();
        __syncwarp();
        if (lane == 0) {
          if constexpr (PAIR) mbar_arrive_remote(map_rank(&cempty[b], 0));   // the leader's barrier
          else mbar_arrive(&cempty[b]);
        }
        bph ^= 1u << b;
        if (args.narrow) eb ^= 1;
        else cb ^= 1;
      }
      if (!fold_ab) {
#pragma unroll
        for (int i = 0; i < WC; ++i) { sr[i] *= scale_b; si[i] *= scale_b; }
      }
      int m = mt * C::TILE_M + (int)rank * BM + row;
      const int n0 = nt * BN + colh * WC;
      if (args.out_gen) {
        // ---- general output map: column offsets of this tile into smem (recomputed only
        // when the tile column changes; double-buffered), then stores
        if (nt != tab_nt) {
          tab_nt = nt;
          ++tab_sel;
          col_table(nt, tab_sel);
        }
        int64_t* tab = noff_tab + (tab_sel & 1) * BN;
        if (args.out_planes) {
          // ---- fused consumer prep: 8 destination-contiguous columns -> one 16-B vector
          // per fp16 plane (RN hi, RN lo = rn(x - hi), Eq. 8), scaled by 2^plane_exp
          if (n0 < args.N && (m < args.M || (EW == 8 && args.planes_rows))) {
            // rows mode: M is a multiple of 8 row groups, so a group is all-valid or all-padding
            int64_t t = m < args.M ? m : 0, moff = 0;
            for (int q = args.n_po - 1; q >= 0; --q) {
              const int sh = args.po_sh[q];
              moff += (t & ((int64_t(1) << sh) - 1)) * args.po_str[q];
              t >>= sh;
            }
            const int64_t rb = m < args.M ? (int64_t)j * args.M * (int64_t)args.N + moff : -1;
            const int64_t* tc = tab + colh * WC;
            __half* P = reinterpret_cast<__half*>(args.C);
            const int64_t pe = args.plane_elems;
            const float ps = ldexpf(1.0f, plane_sc);
            if (EW == 8 && args.planes_rows) {
              // unit-stride plane dim = the 8 lowest row bits: stage 8 columns of the
              // warp's 32 rows in smem, then lane (group g, column c) writes rows
              // 8g..8g+7 of column c as one 16-B vector per plane
              float2* buf = stage_buf + (warp - EPI_WARP0) * 32 * 10;
              const int g = lane >> 3, cc = lane & 7;
              const int64_t gb = __shfl_sync(0xffffffffu, rb, 8 * g);
#pragma unroll
              for (int i = 0; i < WC; i += 8) {
                if (n0 + i >= args.N) break;         // warp-uniform: narrow tiles stop early
#pragma unroll
                for (int jj = 0; jj < 8; ++jj) {
                  buf[lane * 9 + jj] = make_float2(sr[i + jj] * ps, si[i + jj] * ps);
                  if (rb >= 0 && n0 + i + jj < args.N)
                    amax = fmaxf(amax, fmaxf(fabsf(sr[i + jj]), fabsf(si[i + jj])));
                }
                __syncwarp();
                __align__(16) __half hr[8], hi[8], lr[8], li[8];
#pragma unroll
                for (int jj = 0; jj < 8; ++jj) {
                  const float2 x = buf[(8 * g + jj) * 9 + cc];
                  hr[jj] = __float2half_rn(x.x);
                  hi[jj] = __float2half_rn(x.y);
                  plane_ovf |= fmaxf(fabsf(x.x), fabsf(x.y)) >= 65504.f;
                  lr[jj] = __float2half_rn(x.x - __half2float(hr[jj]));
                  li[jj] = __float2half_rn(x.y - __half2float(hi[jj]));
                }
                __syncwarp();
                if (gb >= 0 && n0 + i + cc < args.N) {
                  const int64_t a0 = gb + lds64(tc + i + cc);
                  *reinterpret_cast<uint4*>(P + a0) = *reinterpret_cast<const uint4*>(hr);
                  *reinterpret_cast<uint4*>(P + pe + a0) = *reinterpret_cast<const uint4*>(hi);
                  if (args.out_nplanes == 4) {
                    *reinterpret_cast<uint4*>(P + 2 * pe + a0) = *reinterpret_cast<const uint4*>(lr);
                    *reinterpret_cast<uint4*>(P + 3 * pe + a0) = *reinterpret_cast<const uint4*>(li);
                  }
                }
              }
              continue;
            }
            if (args.planes_v16) {
              // 16 plane-contiguous, 32-B aligned columns: one 256-bit store per plane, so
              // every lane fills a whole sector (the 16-B vectors below fill half of one)
#pragma unroll
              for (int i = 0; i < WC; i += 16) {
                if (n0 + i >= args.N) continue;
                const int64_t a0 = rb + lds64(tc + i);
                __align__(32) __half hr[16], hi[16], lr[16], li[16];
#pragma unroll
                for (int jj = 0; jj < 16; ++jj) {
                  const float xr = sr[i + jj] * ps, xi = si[i + jj] * ps;
                  amax = fmaxf(amax, fmaxf(fabsf(sr[i + jj]), fabsf(si[i + jj])));
                  plane_ovf |= fmaxf(fabsf(xr), fabsf(xi)) >= 65504.f;
                  hr[jj] = __float2half_rn(xr);
                  hi[jj] = __float2half_rn(xi);
                  lr[jj] = __float2half_rn(xr - __half2float(hr[jj]));
                  li[jj] = __float2half_rn(xi - __half2float(hi[jj]));
                }
                st_global_v8(P + a0, reinterpret_cast<const uint32_t*>(hr));
                st_global_v8(P + pe + a0, reinterpret_cast<const uint32_t*>(hi));
                if (args.out_nplanes == 4) {
                  st_global_v8(P + 2 * pe + a0, reinterpret_cast<const uint32_t*>(lr));
                  st_global_v8(P + 3 * pe + a0, reinterpret_cast<const uint32_t*>(li));
                }
              }
              continue;
            }
#pragma unroll
            for (int i = 0; i < WC; i += 8) {
              if (n0 + i >= args.N) continue;
              const int64_t a0 = rb + lds64(tc + i);
              __align__(16) __half hr[8], hi[8], lr[8], li[8];
#pragma unroll
              for (int jj = 0; jj < 8; ++jj) {
                const float xr = sr[i + jj] * ps, xi = si[i + jj] * ps;
                amax = fmaxf(amax, fmaxf(fabsf(sr[i + jj]), fabsf(si[i + jj])));
                plane_ovf |= fmaxf(fabsf(xr), fabsf(xi)) >= 65504.f;
                hr[jj] = __float2half_rn(xr);
                hi[jj] = __float2half_rn(xi);
                lr[jj] = __float2half_rn(xr - __half2float(hr[jj]));
                li[jj] = __float2half_rn(xi - __half2float(hi[jj]));
              }
              *reinterpret_cast<uint4*>(P + a0) = *reinterpret_cast<const uint4*>(hr);
              *reinterpret_cast<uint4*>(P + pe + a0) = *reinterpret_cast<const uint4*>(hi);
              if (args.out_nplanes == 4) {
                *reinterpret_cast<uint4*>(P + 2 * pe + a0) = *reinterpret_cast<const uint4*>(lr);
                *reinterpret_cast<uint4*>(P + 3 * pe + a0) = *reinterpret_cast<const uint4*>(li);
              }
            }
          }
          continue;
        }
        if (EW == 8 && args.cols_contig && n0 + WC <= args.N) {
          // the 64 columns of every row are one contiguous, 16-B aligned output run
          int64_t t = m < args.M ? m : 0, moff = 0;
          for (int q = args.n_po - 1; q >= 0; --q) {
            const int sh = args.po_sh[q];
            moff += (t & ((int64_t(1) << sh) - 1)) * args.po_str[q];
            t >>= sh;
          }
          const int64_t rb = (int64_t)j * args.M * (int64_t)args.N + moff + lds64(tab + colh * WC);
          store_rows_staged<WC>(reinterpret_cast<float4*>(stage_buf + (warp - EPI_WARP0) * 32 * 10), sr, si,
                                args.C, rb, m < args.M, lane, amax);
          continue;
        }
        if (m < args.M && n0 < args.N) {
          int64_t t = m, moff = 0;
          for (int q = args.n_po - 1; q >= 0; --q) {
            const int sh = args.po_sh[q];
            moff += (t & ((int64_t(1) << sh) - 1)) * args.po_str[q];
            t >>= sh;
          }
          const int64_t rb = (int64_t)j * args.M * (int64_t)args.N + moff;
          const int64_t* tc = tab + colh * WC;
          if (args.cols_stride > 1) {
            // one strided column dim (the consumer's unit-stride dim is a row dim): a
            // column's offset is n * stride, no table reads or contiguity tests
            const int64_t cs = args.cols_stride;
            float2* dst = args.C + rb + (int64_t)n0 * cs;
#pragma unroll
            for (int i = 0; i < WC; ++i) {
              if (n0 + i >= args.N) continue;
              dst[i * cs] = make_float2(sr[i], si[i]);
              amax = fmaxf(amax, fmaxf(fabsf(sr[i]), fabsf(si[i])));
            }
            continue;
          }
#pragma unroll
          for (int i = 0; i < WC; i += 2) {      // full unroll: sr/si stay in registers
            if (n0 + i >= args.N) continue;
            const float r0 = sr[i], i0 = si[i];
            const int64_t a0 = rb + lds64(tc + i);
            amax = fmaxf(amax, fmaxf(fabsf(r0), fabsf(i0)));
            if (n0 + i + 1 < args.N) {
              const float r1 = sr[i + 1], i1 = si[i + 1];
              const int64_t a1 = rb + lds64(tc + i + 1);
              amax = fmaxf(amax, fmaxf(fabsf(r1), fabsf(i1)));
              if (a1 == a0 + 1 && (a0 & 1) == 0) {
                *reinterpret_cast<float4*>(args.C + a0) = make_float4(r0, i0, r1, i1);
              } else {
                args.C[a0] = make_float2(r0, i0);
                args.C[a1] = make_float2(r1, i1);
              }
            } else {
              args.C[a0] = make_float2(r0, i0);
            }
          }
        }
        continue;
      }
      if (args.pair_map) {
        // ---- dense merge: keep the (slab a, slab b) blocks that are merged configurations
        if (m < args.M && n0 < args.N) {
          const int a = m >> args.pm_sh_m, p = m & ((1 << args.pm_sh_m) - 1);
          const int shn = args.pm_sh_n, R1 = 1 << shn;
          const int32_t* pm = args.pair_map + (int64_t)a * args.pm_g1;
          const int64_t prow = (int64_t)p << shn;
          int bprev = -1, jj = -1;
#pragma unroll
          for (int i = 0; i < WC; i += 2) {
            const int n = n0 + i;
            if (n >= args.N) continue;
            if (shn >= 1) {                 // columns n, n+1 belong to the same slab b
              const int b = n >> shn;
              if (b != bprev) { jj = pm[b]; bprev = b; }
              if (jj < 0) continue;
              const int64_t addr = ((int64_t)jj << (args.pm_sh_m + shn)) + prow + (n & (R1 - 1));
              const float r0 = sr[i], i0 = si[i], r1 = sr[i + 1], i1 = si[i + 1];
              *reinterpret_cast<float4*>(args.C + addr) = make_float4(r0, i0, r1, i1);
              amax = fmaxf(amax, fmaxf(fmaxf(fabsf(r0), fabsf(i0)), fmaxf(fabsf(r1), fabsf(i1))));
            } else {                        // one column per slab
#pragma unroll
              for (int u = 0; u < 2; ++u) {
                if (n + u >= args.N) continue;
                const int32_t ju = pm[n + u];
                if (ju < 0) continue;
                const int64_t addr = ((int64_t)ju << args.pm_sh_m) + p;
                args.C[addr] = make_float2(sr[i + u], si[i + u]);
                amax = fmaxf(amax, fmaxf(fabsf(sr[i + u]), fabsf(si[i + u])));
              }
            }
          }
        }
        continue;
      }
      int64_t orow = (int64_t)j * args.M + m;
      if (args.rowmap && m < args.M) orow = args.rowmap[m];   // grouped merge: -1 = padding row
      if (EW == 8 && !args.acc && (((args.N % 8) == 0 && n0 < args.N) || ((args.N % 2) == 0 && n0 + WC <= args.N))) {
        // whole 8-column groups (narrow GEMMs: N = 8 .. 56 columns of the 64)
        store_rows_staged<WC>(reinterpret_cast<float4*>(stage_buf + (warp - EPI_WARP0) * 32 * 10), sr, si,
                              args.C, orow * (int64_t)args.N + n0, m < args.M && orow >= 0, lane, amax,
                              min(WC, args.N - n0));
        continue;
      }
      if (m < args.M && n0 < args.N && orow >= 0) {
        const int64_t base = orow * (int64_t)args.N + n0;
        if (args.acc) {
#pragma unroll
          for (int i = 0; i < WC; ++i) {
            if (n0 + i < args.N) {
              const float re = sr[i], im = si[i];
              double2 o = args.acc[base + i];
              o.x += (double)re;
              o.y += (double)im;
              args.acc[base + i] = o;
              amax = fmaxf(amax, fmaxf(fabsf(re), fabsf(im)));
            }
          }
        } else if ((args.N % 2) == 0 && n0 + WC <= args.N) {
          float4* dst = reinterpret_cast<float4*>(args.C + base);
#pragma unroll
          for (int i = 0; i < WC / 2; ++i) {
            const float r0 = sr[2 * i], i0 = si[2 * i];
            const float r1 = sr[2 * i + 1], i1 = si[2 * i + 1];
            dst[i] = make_float4(r0, i0, r1, i1);
            amax = fmaxf(amax, fmaxf(fmaxf(fabsf(r0), fabsf(i0)), fmaxf(fabsf(r1), fabsf(i1))));
          }
        } else {
#pragma unroll
          for (int i = 0; i < WC; ++i) {
            if (n0 + i < args.N) {
              const float re = sr[i], im = si[i];
              args.C[base + i] = make_float2(re, im);
              amax = fmaxf(amax, fmaxf(fabsf(re), fabsf(im)));
            }
          }
        }
      }
    }
    if (args.out_planes) {
      if (__any_sync(0xffffffffu, plane_ovf) && lane == 0) atomicOr(args.overflow, 1);
    }
    if (args.absmax_out) {
      for (int o = 16; o > 0; o >>= 1) amax = fmaxf(amax, __shfl_xor_sync(0xffffffffu, amax, o));
      if (lane == 0 && amax > 0.f) atomicMax(args.absmax_out, __float_as_uint(amax));
    }
  }
  fence_before();
  if constexpr (PAIR) cluster_sync(); else __syncthreads();
  fence_after();
  if (warp == 1) {
    if constexpr (PAIR)
      asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(tmem_base),
                   "r"(TMEM_COLS));
    else
      asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem_base),
                   "r"(TMEM_COLS));
  }
}

template <int PASSES, int EW, bool PAIR, int FMT = FMT_F16>
cudaError_t launch_impl(const GemmArgs& a, int num_sms, cudaStream_t s) {
  const int smem = Cfg<PASSES, PAIR>::SMEM_BYTES + stage_bytes<EW>();
  const void* kern = reinterpret_cast<const void*>(cgemm_tcgen05_kernel<PASSES, EW, PAIR, FMT>);
  if (cudaError_t e = set_smem_attr(kern, smem)) return e;
  if constexpr (PAIR) {
    // tiles of 256 rows, one per CTA pair (cluster of 2); persistent over the SMs
    GemmArgs p = a;
    p.tiles_m = (a.M + 2 * BM - 1) / (2 * BM);
    p.n_tiles = (int64_t)p.tiles_m * p.tiles_n * a.J;
    int64_t pairs = p.n_tiles < num_sms / 2 ? p.n_tiles : num_sms / 2;
    // a persistent grid must be co-resident (the wave sync waits on every producer):
    // never launch more clusters than can be active at once
    int max_clusters;
    {
      cudaLaunchConfig_t q = {};
      q.gridDim = dim3((unsigned)num_sms);
      q.blockDim = dim3(32 * EPI_WARP0 + 32 * EW);
      q.dynamicSmemBytes = smem;
      cudaLaunchAttribute qa[1];
      qa[0].id = cudaLaunchAttributeClusterDimension;
      qa[0].val.clusterDim.x = 2;
      qa[0].val.clusterDim.y = 1;
      qa[0].val.clusterDim.z = 1;
      q.attrs = qa;
      q.numAttrs = 1;
      max_clusters = max_active_clusters(kern, q, num_sms / 2);
    }
    if (pairs > max_clusters) pairs = max_clusters;
    if (pairs < 1) pairs = 1;
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3((unsigned)(2 * pairs));
    cfg.blockDim = dim3(32 * EPI_WARP0 + 32 * EW);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = s;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = 2;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    return cudaLaunchKernelEx(&cfg, cgemm_tcgen05_kernel<PASSES, EW, PAIR, FMT>, p);
  } else {
    int64_t grid = a.n_tiles < num_sms ? a.n_tiles : num_sms;
    if (grid < 1) grid = 1;
    cgemm_tcgen05_kernel<PASSES, EW, PAIR, FMT><<<(unsigned)grid, 32 * EPI_WARP0 + 32 * EW, smem, s>>>(a);
    return cudaGetLastError();
  }
}

}  // namespace

namespace {

typedef CUresult (*EncodeTiledFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*,
                                  const cuuint64_t*, const cuuint64_t*, const cuuint32_t*,
                                  const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                                  CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

EncodeTiledFn get_encode() {
  static EncodeTiledFn fn = nullptr;
  if (!fn) {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<EncodeTiledFn>(p);
  }
  return fn;
}

}  // namespace

bool gemm_pair_ok(const GemmArgs& a, int min_m) {
  // the pair shares one B slab per 256-row tile: grouped merges (slab per 128-row
  // block) stay on the single-CTA kernel
  return min_m > 0 && a.M >= min_m && a.blk_slab_b == nullptr;
}

cudaError_t launch_gemm(const GemmArgs& a_in, int passes, int num_sms, cudaStream_t s, int format) {
  GemmArgs a = a_in;
  a.narrow = (g_knobs.narrow_mma && a.N <= 64) ? 1 : 0;
  a.l2hint = g_knobs.l2hint;
  if (a.wave_sync) {
    cudaError_t e = cudaMemsetAsync(a.wave_ctr, 0, sizeof(unsigned long long), s);
    if (e != cudaSuccess) return e;
  }
  if (format == FMT_BF16)   // precision study formats (tn_cgemm): single-CTA tiles
    return passes == 3 ? launch_impl<3, 8, false, FMT_BF16>(a, num_sms, s)
                       : launch_impl<1, 8, false, FMT_BF16>(a, num_sms, s);
  if (format == FMT_TF32)
    return passes == 3 ? launch_impl<3, 8, false, FMT_TF32>(a, num_sms, s)
                       : launch_impl<1, 8, false, FMT_TF32>(a, num_sms, s);
  if (a.use_pair)
    return passes == 3 ? launch_impl<3, 8, true>(a, num_sms, s) : launch_impl<1, 8, true>(a, num_sms, s);
  return passes == 3 ? launch_impl<3, 8, false>(a, num_sms, s) : launch_impl<1, 8, false>(a, num_sms, s);
}

bool encode_plane_map(CUtensorMap* map, const void* base, int64_t Kpad, int64_t R, int64_t G,
                      int planes, int box_rows, char* err, size_t errcap, int format) {
  const int esz = format == FMT_TF32 ? 4 : 2;
  const CUtensorMapDataType dt = format == FMT_TF32   ? CU_TENSOR_MAP_DATA_TYPE_FLOAT32
                                 : format == FMT_BF16 ? CU_TENSOR_MAP_DATA_TYPE_BFLOAT16
                                                      : CU_TENSOR_MAP_DATA_TYPE_FLOAT16;
  EncodeTiledFn enc = get_encode();
  if (!enc) {
    snprintf(err, errcap, "cuTensorMapEncodeTiled unavailable");
    return false;
  }
  cuuint64_t dims[4] = {(cuuint64_t)Kpad, (cuuint64_t)R, (cuuint64_t)G, (cuuint64_t)planes};
  cuuint64_t strides[3] = {(cuuint64_t)(Kpad * esz), (cuuint64_t)(Kpad * esz * R),
                           (cuuint64_t)(Kpad * esz * R * G)};
  cuuint32_t box[4] = {(cuuint32_t)(64 / esz), (cuuint32_t)box_rows, 1, 1};
  cuuint32_t es[4] = {1, 1, 1, 1};
  CUresult r = enc(map, dt, 4, const_cast<void*>(base), dims, strides,
                   box, es, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_64B,
                   CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) {
    snprintf(err, errcap, "cuTensorMapEncodeTiled failed (%d): Kpad=%lld R=%lld G=%lld", (int)r,
             (long long)Kpad, (long long)R, (long long)G);
    return false;
  }
  return true;
}

}  // namespace tn
