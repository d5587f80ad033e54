// Internal descriptors shared by the host planner and the sm_100a kernels.
// Device descriptors live in device memory (uploaded once per plan) so the
// per-slice launch sequence only passes pointers.
#pragma once
#include <cstdint>
#include <cuda.h>
#include <cuda_fp16.h>
#include <cuda_runtime.h>

#define TN_MAXD 40          // max coalesced dims per operand side after merging runs

namespace tn {

// ---------------------------------------------------------------- SIMT einsum
// C[j][m][n] (+)= Σ_k A[slabA(j), m, k] · B[slabB(j), n, k] over strided views.
struct EinsumDesc {
  const float2* A; const float2* B; float2* C;
  int64_t a_off, b_off;           // static element offsets
  int32_t a_leaf, b_leaf;         // index into the per-slice leaf offset array, or -1
  int64_t J;                      // batch (merged sparse configurations)
  const int32_t* ia; const int32_t* ib;   // slab tables (nullable -> slab 0)
  int64_t a_gs, b_gs;             // slab strides (elements)
  int64_t M, N, K;
  int32_t nm, nn, nk;
  int64_t m_ext[TN_MAXD], m_sa[TN_MAXD];
  int64_t n_ext[TN_MAXD], n_sb[TN_MAXD];
  int64_t k_ext[TN_MAXD], k_sa[TN_MAXD], k_sb[TN_MAXD];
  unsigned* absmax_out;           // nullable: atomicMax of |re|,|im| bits
  double2* acc;                   // nullable: acc[idx] += C instead of storing C
  // mode: 4 warp dot (batched merge, one warp per output row, N <= 32, lanes over K);
  // 0 general (one thread per output), 1 skinny (B = small operand staged in
  // smem, output layout [Mo][N][V] with V = A's smallest-stride free dim, which is
  // m_ext/m_sa[nm-1] here), 2 split-K dot (few outputs, long K; fp64 partials)
  int32_t mode, pow2;             // pow2: every m/n/k extent is a power of two (shift tables valid)
  uint8_t m_sh[TN_MAXD], n_sh[TN_MAXD], k_sh[TN_MAXD];   // log2 of the extents
  int64_t V;                      // mode 1: extent of the vector (lane) dim
  double* partial;                // mode 2: fp64 partial sums [2*J*M*N] (zeroed per launch)
  int64_t n_yslabs;               // mode 1 with J > 1: slabs of the small operand (all in smem)
  int64_t kchunk;                 // mode 2: k elements per block
  // mode 4, slab-staged variant (wd_ok = 1): the batches are grouped by B slab (CSR
  // wd_start[wd_nslabs + 1] / wd_list[J]); a block stages one contiguous part of a B slab
  // (2^wd_lb elements: the top wd_t bits of the slab offset are n bits) into shared memory
  // in [n_local][k] order, then its warps run that slab's batches with B from smem
  const int32_t* wd_start; const int32_t* wd_list;
  int64_t wd_nslabs;
  int32_t wd_ok, wd_t, wd_lb, wd_np;
  int32_t wd_contrib[16];         // part-offset bit b -> smem index weight (k: canonical k;
                                  // n: (1 << local n bit) * K)
  int32_t wd_nloc[32];            // local n index -> canonical output column
  int32_t wd_ptop[8];             // part index -> canonical output column offset
};

// ---------------------------------------------------------------- fused skinny chain
// A chain of skinny SIMT steps s1 -> s2 -> ... -> sL on the stem (each consumes the
// previous output as its big operand X and absorbs a small tensor Y) run as ONE pass:
// the index bits no step touches ("carry" bits) enumerate independent positions; for a
// tile of 32 carry positions (lanes = the 5 lowest-weight carry bits of the first input
// T0) a block loads T0's touched elements, runs every
// step in shared memory ([touched index][32 lanes] tensors) and writes TL.  Each output
// is the same fp32 k-ordered sum as einsum_skinny_kernel, so the result is bit-identical
// to running the steps one by one; the intermediates never reach HBM.
constexpr int TN_CHAIN_MAX = 8;
struct ChainStep {
  const float2* Y; int64_t y_off; int32_t y_leaf;
  int32_t N, K, P;                // outputs per o-position, k, touched o-positions
  int32_t tab;                    // int32 table offset: in_p[P], out_p[P], in_k[K], out_n[N], yoff[N*K]
  int32_t in_buf, pad_;           // smem buffer holding the step's input (0 = A, 1 = B)
};
struct ChainDesc {
  const float2* src; int64_t src_off; int32_t src_leaf, L;
  float2* dst; unsigned* absmax_out;
  int32_t a0, aL, nct, buf_a, buf_b, n_tab;   // log2 |W0|, log2 |WL|, outer carry bits, buffer elems
  int64_t n_tiles;
  int64_t ct_src[32], ct_dst[32];             // outer carry bit weights in T0 / TL
  int64_t lw_src[5], lw_dst[5];               // the 5 lane carry bits' weights in T0 / TL
  const int32_t* tab;                         // t0off[2^a0], tLoff[2^aL], then the step tables
  ChainStep st[TN_CHAIN_MAX];
};

// ---------------------------------------------------------------- operand prep
// Permute a strided complex64 view into K-contiguous fp16 planes with a
// per-tensor power-of-two scale: plane p of element (g, r, k) at
// dst[p*plane_elems + (g*R + r)*Kpad + k]; planes = re_hi, im_hi[, re_lo, im_lo].
struct PrepDesc {
  const float2* src; int64_t off; int32_t leaf;
  int64_t G, R, K, Kpad, g_stride;
  int32_t nr, nk;
  int64_t r_ext[TN_MAXD], r_s[TN_MAXD];
  int64_t k_ext[TN_MAXD], k_s[TN_MAXD];
  int32_t read_r_fast, pad_;      // 1: source stride of rows < of k (read along r)
  // general transposer (kind 2): the tile is the product of the dims t_* (which hold
  // both the source's and the destination's innermost contiguous runs); outer dims
  // c_*.  t dims are listed twice: in source-stride order (ts_*) and in destination-
  // stride order (td_*), with td_pos[i] = position of td dim i in the ts list.
  int32_t kind;                   // 0 transposer(r/k), 1 direct, 2 general transposer
  int32_t nt, nc;
  int32_t T, pad2_;
  int64_t nC;
  int64_t ts_ext[12], ts_src[12], ts_dst[12];   // source order, outer -> inner
  int64_t td_ext[12];
  int32_t td_pos[12];                           // destination order, outer -> inner
  int64_t c_ext[TN_MAXD], c_src[TN_MAXD], c_dst[TN_MAXD];
  uint8_t c_sh[TN_MAXD];          // log2 c_ext (general transposer requires power-of-two dims)
  const int64_t* gt_tab;          // plan-time tables: srcoff[T], dstoff[T], then int32 spos[T]
  const int64_t* rowoff;          // kind 3: source offset of each destination row (-1 = zeros)
  // bit-permutation transposer (kind 4): tile of 2^bp_t elements; outer bits in c_src /
  // c_dst (nc of them, nC = 2^nc tiles per slab); bp_tab = plan-time tile tables
  // [src lo/hi 128][dst T/8][slot T/4 words of u16][swizzle T/128 words of u8]
  int32_t bp_t, bp_vec;           // bp_vec: source pairs (e, e+1) are adjacent (16-B loads)
  const int64_t* bp_tab;
  // gate-folded prep (kind 5): the operand is the output of a skinny SIMT step
  // out[o][n][v] = sum_k Y[n][k] X[o, v, k] that is never materialised: src is X, the
  // tile holds X values (carry bits + k bits), each plane element applies Y on the fly.
  // bp_tab: [src lo/hi 128][dst T/8][cn: T int32 (carry pos | n << 16)]
  const float2* gy; int64_t gy_off; int32_t gy_leaf, g_N, g_K, g_cbits, g_ts, g_nn, g_nk, g_regroup;   // g_regroup: 1 = regrouped compute
  int64_t gy_n_ext[8], gy_n_s[8], gy_k_ext[8], gy_k_s[8];
  const unsigned* absmax_y;
  __half* dst; int64_t plane_elems;
  const unsigned* absmax_in;      // absmax of the source tensor (float bits)
  int* scale_out;                 // receives the exponent s (x * 2^s is split)
};

// ---------------------------------------------------------------- tcgen05 GEMM
struct GemmArgs {
  CUtensorMap mapA;               // 4D fp16 (Kpad, R, G, planes), box (32, 128, 1, 1), SW64
  CUtensorMap mapB;
  CUtensorMap mapB2;              // B with box (32, 64, 1, 1): per-CTA half of N for the CTA pair
  int32_t J, M, N, K;             // M = rows of A operand, N = rows of B operand (complex)
  const int32_t* ia; const int32_t* ib;
  float2* C;                      // [J][M][N] complex64
  const int* scaleA; const int* scaleB;
  unsigned* absmax_out;
  double2* acc;                   // nullable: fused fp64 slice-accumulate
  int32_t tiles_m, tiles_n;
  int64_t n_tiles;
  int32_t kchunk;                 // k-blocks per TMEM chunk promoted to the fp32 RN
                                  // register sum (0 = whole K in TMEM); see DESIGN.md
  int32_t group_m;                // tile rasterization: tile rows per group (L2 reuse)
  // grouped sparse merge (slab-regrouped Eq. 7): rows of A are gathered (j, q) rows
  // sorted by B's slab; blk_slab_b[mt] = B slab of 128-row block mt; rowmap[r] = output
  // row of gathered row r (-1 = padding); output C[rowmap[r]][n]
  const int32_t* blk_slab_b;
  const int32_t* rowmap;
  int32_t use_pair;               // 1: CTA-pair kernel (cta_group::2, 256-row tiles)
  // general output map (out_gen = 1): C[j·M·N + Σ digit_p(m)·po_str[p] + Σ digit_q(n)·qo_str[q]]
  // with row m / column n decomposed over power-of-two extents (log2 in po_sh / qo_sh,
  // outer -> inner).  Lets the producer write the consumer's preferred layout
  // ([P keep][Q keep][contracted, sorted]) so the consumer's operand is K-contiguous.
  int32_t out_gen, n_po, n_qo;
  int32_t cols_contig;            // out_gen: the 64 columns of a warp are one contiguous run
  int32_t cols_pad;
  int64_t cols_stride;            // out_gen: > 1 = the columns are one dim of this stride
  uint8_t po_sh[16], qo_sh[16];
  int64_t po_str[16], qo_str[16];
  // fused consumer prep (a3 + a6 in this epilogue): the output is written directly as the
  // consumer's K-contiguous fp16 planes (po/qo strides are plane-element strides; C is
  // the plane base, plane p at C + p*plane_elems halves).  Values are acc * 2^plane_exp
  // with plane_exp = -16 - ceil(log2 K): |acc| <= K 2^31 for operands scaled below 2^15,
  // so the planes stay below 2^15 without waiting for the output's absmax; the consumer's
  // exponent sA + sB + plane_exp goes to *plane_scale_out.
  int32_t l2hint;                 // 1: operand TMA loads carry an L2 evict_last policy
  int32_t out_planes, out_nplanes, plane_exp;
  int32_t planes_rows;            // 1: the unit-stride plane dim is the 8 lowest row bits
                                  // (staged through smem); 0: the 8 lowest column bits
  int64_t plane_elems;
  int* plane_scale_out;
  const int* plane_pexp;          // delayed-scaling exponent (SliceDesc.pexp[step])
  int* overflow;                  // set when a plane value reaches the fp16 range limit
  // wave synchronisation (locality hint): before each tile every producer arrives on a
  // global counter and waits (bounded spin) until all producers of the wave have
  // arrived, so the tiles that share A / B panels stream the same k-blocks together
  // and the panels are read from L2 instead of DRAM; zeroed per launch
  unsigned long long* wave_ctr;
  int32_t wave_sync, pad_w;
  // dense merge (pair-mapped epilogue): row = a*2^pm_sh_m + p, col = b*2^pm_sh_n + q,
  // j = pair_map[a*pm_g1 + b] (-1: not a merged configuration), out C[j][p][q]
  const int32_t* pair_map;
  int32_t pm_sh_m, pm_sh_n, pm_g1;
  int32_t narrow;                 // N <= 64: N = 64 MMA instructions (one column tile)
  int32_t planes_v16;             // plane mode, columns: 16 plane-contiguous columns, 32-B
                                  // aligned -> one 256-bit store per plane and 16 columns
};

// ---------------------------------------------------------------- slice select
struct SliceDesc {
  int32_t n_sliced;
  int64_t dims[64];
  int32_t n_terms;                // (leaf, sliced index, stride) terms
  const int32_t* term_leaf; const int32_t* term_p; const int64_t* term_stride;
  int32_t n_leaves;
  int64_t* leaf_off;              // out: per-leaf dynamic element offset
  int64_t* counter;               // in/out: current slice index (incremented)
  unsigned* absmax; int32_t absmax_first, absmax_count;  // zeroed per slice
  // delayed scaling of fused plane outputs: hist[s] = running max over finished slices
  // of step s's output absmax (merged here from the absmax slot before it is zeroed);
  // pexp[s] = 11 - e(hist[s]) puts the largest value seen so far near 2^11 (32x margin)
  unsigned* hist; int* pexp;
};

// Process-wide tuning and test-forcing knobs of the kernel launchers, re-read from the
// TN_* environment at every tn_create (DESIGN.md §10 lists every knob; planner knobs
// are read per plan in build_plan).  Defaults are the product settings.
struct Knobs {
  int gate_bps = 4;       // TN_GATE_BPS: gate-folded prep blocks per SM
  int skinny_rows = 0;    // TN_SKINNY_ROWS: force the skinny kernel's rows per thread (tests)
  int simt_old = 0;       // TN_SIMT_OLD: force the previous skinny design (A/B tests)
  int skinny_vec2 = 1;    // TN_SKINNY_VEC2=0: no paired-lane / k-pair 16-B accesses (tests)
  int gate_mma = 0;       // TN_GATE_MMA=1: gate-folded preps with K >= 4 on mma.sync (measured slower)
  int l2hint = 0;         // TN_GEMM_L2HINT=1: operand TMA loads with an evict_last policy (neutral)
  int narrow_mma = 1;     // TN_NARROW_MMA=0: N <= 64 GEMMs issue N = 128 MMAs (A/B tests)
  int prep_bp = 1;        // TN_PREP_BP=0: no bit-permutation transposer (A/B tests)
  int pair_min_m = 512;   // TN_GEMM_PAIR_MIN_M: CTA-pair GEMM from this M (0 = never)
};
extern Knobs g_knobs;
void refresh_knobs();

// cudaFuncSetAttribute(MaxDynamicSharedMemorySize) is per device context: applied once
// per (kernel, device), thread-safe; a later larger request raises it
cudaError_t set_smem_attr(const void* kernel, int bytes);
// cudaOccupancyMaxActiveClusters of a launch configuration, cached per (kernel, device)
int max_active_clusters(const void* kernel, const cudaLaunchConfig_t& cfg, int fallback);

// kernel launchers (kernels.cu / gemm_tcgen05.cu)
cudaError_t launch_slice_select(const SliceDesc* d_desc, cudaStream_t s);
cudaError_t launch_set_counter(int64_t* counter, int64_t value, cudaStream_t s);
cudaError_t launch_prep(const PrepDesc* d_desc, int64_t total, int planes, int kind, int tile_T,
                        const int64_t* leaf_off, cudaStream_t s, int gate_k = 0, int gate_n = 0);
// variant: kernel variant of the SIMT mode (0 = heuristic); einsum_variants() = how many
cudaError_t launch_einsum(const EinsumDesc* d_desc, const EinsumDesc& host_desc,
                          const int64_t* leaf_off, cudaStream_t s, int variant = 0);
int einsum_variants(const EinsumDesc& host_desc);
cudaError_t launch_chain(const ChainDesc* d_desc, const ChainDesc& host_desc, const int64_t* leaf_off,
                         cudaStream_t s);
size_t chain_smem_bytes(const ChainDesc& host_desc);
cudaError_t launch_gather_out(const double2* acc, const int32_t* pos, double2* out, int64_t n,
                              const int* flag, cudaStream_t s);
cudaError_t launch_absmax(const float2* x, int64_t n, unsigned* out, cudaStream_t s);
// precision-study operand prep (bf16 = 1 / tf32 = 2 planes) of a K-contiguous [rows][K] operand
cudaError_t launch_prep_fmt(const float2* src, void* dst, int64_t rows, int64_t K, int64_t Kpad,
                            int planes, int format, const unsigned* absmax, int* scale_out,
                            cudaStream_t s);
// format: 0 = fp16 planes (product path), 1 = bf16, 2 = tf32 (precision study, tn_cgemm)
cudaError_t launch_gemm(const GemmArgs& a, int passes, int num_sms, cudaStream_t s, int format = 0);
// CTA-pair eligibility: M >= min_m (g_knobs.pair_min_m, default 512; 0 = never) and
// one B slab per 256-row tile (not a grouped merge)
bool gemm_pair_ok(const GemmArgs& a, int min_m);
bool encode_plane_map(CUtensorMap* map, const void* base, int64_t Kpad, int64_t R, int64_t G,
                      int planes, int box_rows, char* err, size_t errcap, int format = 0);

}  // namespace tn
