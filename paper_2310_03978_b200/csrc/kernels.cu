// HBM-side kernels of the hot path (sm_100a):
//   slice_select  — a2: slice index -> mixed-radix digits -> per-leaf offsets
//                   (DESIGN R7: last sliced bond fastest)
//   prep          — a3 + a6: permutation of a strided complex64 view into the
//                   K-contiguous fp16 planes the tensor-core GEMM reads, with the
//                   per-tensor power-of-two rescale (L403, L594) and the RN hi/lo
//                   split of Eq. 8 (L367-377; 3xFP16 variant L383-386)
//   einsum_simt   — Eq. 3 (L219-229) on CUDA cores for small / skinny steps, with
//                   sparse-merge gather tables (Eq. 7) and fused fp64 accumulate
//   gather_out    — a9: merged-configuration order -> caller sample order
#include "tn_internal.h"
#include <cuda_bf16.h>

#include <algorithm>

namespace tn {

namespace {

template <typename T>
__device__ __forceinline__ void copy_desc_to_smem(T* dst, const T* src) {
  static_assert(sizeof(T) % 8 == 0, "desc size");
  const int n = sizeof(T) / 8;
  const uint64_t* s = reinterpret_cast<const uint64_t*>(src);
  uint64_t* d = reinterpret_cast<uint64_t*>(dst);
  for (int i = threadIdx.x; i < n; i += blockDim.x) d[i] = s[i];
  __syncthreads();
}

__device__ __forceinline__ float warp_max(float v) {
  for (int o = 16; o > 0; o >>= 1) v = fmaxf(v, __shfl_xor_sync(0xffffffffu, v, o));
  return v;
}

__device__ __forceinline__ void block_absmax(float v, unsigned* out) {
  __shared__ float red[32];
  v = warp_max(v);
  const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
  if (l == 0) red[w] = v;
  __syncthreads();
  if (w == 0) {
    float x = (l < (int)(blockDim.x >> 5)) ? red[l] : 0.f;
    x = warp_max(x);
    if (l == 0 && x > 0.f) atomicMax(out, __float_as_uint(x));
  }
}

// ---------------------------------------------------------------- slice select
__global__ void slice_select_kernel(const SliceDesc* __restrict__ d) {
  __shared__ int64_t digit[64];
  __shared__ int64_t t0;
  if (threadIdx.x == 0) {
    int64_t t = *d->counter;
    t0 = t;
    for (int p = d->n_sliced - 1; p >= 0; --p) {   // last sliced bond = fastest digit
      digit[p] = t % d->dims[p];
      t /= d->dims[p];
    }
  }
  __syncthreads();
  for (int l = threadIdx.x; l < d->n_leaves; l += blockDim.x) {
    int64_t off = 0;
    for (int q = 0; q < d->n_terms; ++q)
      if (d->term_leaf[q] == l) off += digit[d->term_p[q]] * d->term_stride[q];
    d->leaf_off[l] = off;
  }
  for (int a = threadIdx.x; a < d->absmax_count; a += blockDim.x) {
    const unsigned h = max(d->hist[a], d->absmax[d->absmax_first + a]);   // finished slice
    d->hist[a] = h;
    int e = 0;
    if (h) frexpf(__uint_as_float(h), &e);
    d->pexp[a] = h ? 11 - e : -100000;
    d->absmax[d->absmax_first + a] = 0u;
  }
  __syncthreads();
  if (threadIdx.x == 0) *d->counter = t0 + 1;
}

// first slice index of a tn_contract range, passed by value (a pinned-host copy
// would read the host word at execution time, after later calls overwrote it)
__global__ void set_counter_kernel(int64_t* counter, int64_t value) { *counter = value; }

// ---------------------------------------------------------------- operand prep
// Power-of-two exponent s with absmax·2^s in [2^14, 2^15) (inside the fp16 range,
// PAPER.md L403 "dynamic scaling"); block 0 publishes it for the GEMM epilogue.
__device__ __forceinline__ float prep_scale(const PrepDesc& d) {
  const float amax = __uint_as_float(*d.absmax_in);
  int s = 0;
  if (amax > 0.f) {
    int e;
    frexpf(amax, &e);            // amax = f * 2^e, f in [0.5, 1)
    s = 15 - e;
    s = max(-120, min(120, s));
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) *d.scale_out = s;
  return ldexpf(1.0f, s);
}

// RN hi/lo split of 8 consecutive k-values (Eq. 8: big = rn(x), small = rn(x - big))
// stored as one 16-byte vector per plane.
template <int PLANES>
__device__ __forceinline__ void split_store8(const PrepDesc& d, int64_t idx, const float2* v,
                                             float scale) {
  __align__(16) __half hr[8], hi[8], lr[8], li[8];
#pragma unroll
  for (int j = 0; j < 8; ++j) {
    const float xr = v[j].x * scale, xi = v[j].y * scale;
    hr[j] = __float2half_rn(xr);
    hi[j] = __float2half_rn(xi);
    if (PLANES == 4) {
      lr[j] = __float2half_rn(xr - __half2float(hr[j]));
      li[j] = __float2half_rn(xi - __half2float(hi[j]));
    }
  }
  const int64_t plane = d.plane_elems;
  *reinterpret_cast<uint4*>(d.dst + idx) = *reinterpret_cast<const uint4*>(hr);
  *reinterpret_cast<uint4*>(d.dst + plane + idx) = *reinterpret_cast<const uint4*>(hi);
  if (PLANES == 4) {
    *reinterpret_cast<uint4*>(d.dst + 2 * plane + idx) = *reinterpret_cast<const uint4*>(lr);
    *reinterpret_cast<uint4*>(d.dst + 3 * plane + idx) = *reinterpret_cast<const uint4*>(li);
  }
}

template <int PLANES>
__global__ void __launch_bounds__(256, 4) prep_kernel(const PrepDesc* __restrict__ gd,
                                                      const int64_t* __restrict__ leaf_off,
                                                      int64_t total) {
  __shared__ __align__(16) PrepDesc d;
  copy_desc_to_smem(&d, gd);
  const float2* src = d.src + d.off + (d.leaf >= 0 ? leaf_off[d.leaf] : 0);
  const float scale = prep_scale(d);
  const int64_t plane = d.plane_elems;
  // Tiled transpose: a tile is TR rows x TK k-values of one slab.  Row and column
  // source offsets are decomposed once per tile into smem, so each element costs
  // one add; the read phase walks whichever of (r, k) has the smaller source
  // stride (coalesced), the write phase walks k (K-contiguous planes).
  constexpr int TR = 32, TK = 64;
  __shared__ int64_t roff[TR];
  __shared__ int64_t koff[TK];
  __shared__ float2 tile[TR][TK + 1];
  const bool r_fast = d.read_r_fast != 0;
  const int64_t rtiles = (d.R + TR - 1) / TR, ktiles = (d.Kpad + TK - 1) / TK;
  const int64_t ntiles = d.G * rtiles * ktiles;
  for (int64_t t = blockIdx.x; t < ntiles; t += gridDim.x) {
    const int64_t kt = t % ktiles;
    const int64_t rt = (t / ktiles) % rtiles;
    const int64_t g = t / (ktiles * rtiles);
    const int64_t r0 = rt * TR, k0 = kt * TK;
    __syncthreads();   // previous tile fully consumed
    if (threadIdx.x < TR) {
      int64_t r = r0 + threadIdx.x, off = -1;
      if (r < d.R) {
        off = g * d.g_stride;
        for (int i = d.nr - 1; i >= 0; --i) { off += (r % d.r_ext[i]) * d.r_s[i]; r /= d.r_ext[i]; }
      }
      roff[threadIdx.x] = off;
    } else if (threadIdx.x < TR + TK) {
      int64_t k = k0 + threadIdx.x - TR, off = -1;
      if (k < d.K) {
        off = 0;
        for (int i = d.nk - 1; i >= 0; --i) { off += (k % d.k_ext[i]) * d.k_s[i]; k /= d.k_ext[i]; }
      }
      koff[threadIdx.x - TR] = off;
    }
    __syncthreads();
#pragma unroll
    for (int i = 0; i < TR * TK / 256; ++i) {
      const int e = threadIdx.x + i * 256;
      const int r = r_fast ? (e % TR) : (e / TK);
      const int k = r_fast ? (e / TR) : (e % TK);
      const int64_t ro = roff[r], ko = koff[k];
      tile[r][k] = (ro >= 0 && ko >= 0) ? src[ro + ko] : make_float2(0.f, 0.f);
    }
    __syncthreads();
#pragma unroll
    for (int i = 0; i < TR * TK / 512; ++i) {
      const int e = threadIdx.x + i * 256;          // pairs of k
      const int r = e / (TK / 2);
      const int k = (e % (TK / 2)) * 2;
      if (r0 + r >= d.R || k0 + k >= d.Kpad) continue;
      const float2 v0 = tile[r][k], v1 = tile[r][k + 1];
      const float xr0 = v0.x * scale, xi0 = v0.y * scale, xr1 = v1.x * scale, xi1 = v1.y * scale;
      const __half2 hr = __floats2half2_rn(xr0, xr1), hi = __floats2half2_rn(xi0, xi1);
      const int64_t idx = (g * d.R + r0 + r) * d.Kpad + k0 + k;   // Kpad even: half2-aligned
      reinterpret_cast<__half2*>(d.dst + idx)[0] = hr;
      reinterpret_cast<__half2*>(d.dst + plane + idx)[0] = hi;
      if (PLANES == 4) {   // residuals, RN (Eq. 8: small = rn(x - big))
        const float2 fr = __half22float2(hr), fi = __half22float2(hi);
        reinterpret_cast<__half2*>(d.dst + 2 * plane + idx)[0] =
            __floats2half2_rn(xr0 - fr.x, xr1 - fr.y);
        reinterpret_cast<__half2*>(d.dst + 3 * plane + idx)[0] =
            __floats2half2_rn(xi0 - fi.x, xi1 - fi.y);
      }
    }
  }
}

// Operand prep for the precision-study formats of tn_cgemm (Fig. 4, Eq. 8):
// a K-contiguous complex64 [G][R][K] operand -> planes re_big, im_big[, re_small,
// im_small] of [G][R][Kpad] in bf16 (format 1) or tf32 in 32-bit containers (format 2),
// big = rn(x·2^s), small = rn(x·2^s - big), both round-to-nearest-even (R11).
__device__ __forceinline__ float rn_tf32(float x) {
  uint32_t u = __float_as_uint(x);
  if ((u & 0x7f800000u) == 0x7f800000u) return x;            // inf / nan
  u += 0xfffu + ((u >> 13) & 1u);                            // RNE at bit 13
  return __uint_as_float(u & 0xffffe000u);
}

__global__ void __launch_bounds__(256) prep_fmt_kernel(const float2* __restrict__ src, void* dst,
                                                       int64_t rows, int64_t K, int64_t Kpad,
                                                       int planes, int format,
                                                       const unsigned* __restrict__ absmax,
                                                       int* scale_out) {
  const float amax = __uint_as_float(*absmax);
  int s = 0;
  if (amax > 0.f) {
    int e;
    frexpf(amax, &e);
    s = max(-120, min(120, 15 - e));
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) *scale_out = s;
  const float sc = ldexpf(1.0f, s);
  const int64_t plane = rows * Kpad;
  for (int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; idx < plane;
       idx += (int64_t)gridDim.x * blockDim.x) {
    const int64_t r = idx / Kpad, k = idx % Kpad;
    const float2 v = k < K ? src[r * K + k] : make_float2(0.f, 0.f);
    const float x[2] = {v.x * sc, v.y * sc};
#pragma unroll
    for (int c = 0; c < 2; ++c) {
      if (format == 2) {
        float* P = reinterpret_cast<float*>(dst);
        const float big = rn_tf32(x[c]);
        P[c * plane + idx] = big;
        if (planes == 4) P[(2 + c) * plane + idx] = rn_tf32(x[c] - big);
      } else {
        __nv_bfloat16* P = reinterpret_cast<__nv_bfloat16*>(dst);
        const __nv_bfloat16 big = __float2bfloat16_rn(x[c]);
        P[c * plane + idx] = big;
        if (planes == 4) P[(2 + c) * plane + idx] = __float2bfloat16_rn(x[c] - __bfloat162float(big));
      }
    }
  }
}

// Row-major digit decomposition of t over (ext[0..n-1]) -> Σ digit * stride.
// Circuit networks have power-of-two extents: those dims use shift/mask.
__device__ __forceinline__ int64_t decompose(int64_t t, int n, const int64_t* ext,
                                             const int64_t* stride) {
  int64_t off = 0;
  for (int i = n - 1; i >= 0; --i) {
    const int64_t e = ext[i];
    if ((e & (e - 1)) == 0) {
      off += (t & (e - 1)) * stride[i];
      t >>= (__ffsll(e) - 1);
    } else {
      off += (t % e) * stride[i];
      t /= e;
    }
  }
  return off;
}

// shift-table decomposition (all extents powers of two; sh = log2 extents)
__device__ __forceinline__ int64_t decompose_sh(int64_t t, int n, const uint8_t* sh,
                                                const int64_t* stride) {
  int64_t off = 0;
  for (int i = n - 1; i >= 0; --i) {
    const int s = sh[i];
    off += (t & ((int64_t(1) << s) - 1)) * stride[i];
    t >>= s;
  }
  return off;
}

__device__ __forceinline__ void store_out_f(const EinsumDesc& d, int64_t idx, float cr, float ci,
                                            float& amax) {
  if (d.acc) {
    double2 o = d.acc[idx];
    o.x += (double)cr;
    o.y += (double)ci;
    d.acc[idx] = o;
  } else {
    d.C[idx] = make_float2(cr, ci);
  }
  amax = fmaxf(amax, fmaxf(fabsf(cr), fabsf(ci)));
}

__device__ __forceinline__ void store_out(const EinsumDesc& d, int64_t idx, double cr, double ci,
                                          float& amax) {
  if (d.acc) {
    double2 o = d.acc[idx];
    o.x += cr;
    o.y += ci;
    d.acc[idx] = o;
  } else {
    d.C[idx] = make_float2((float)cr, (float)ci);
  }
  amax = fmaxf(amax, fmaxf(fabsf((float)cr), fabsf((float)ci)));
}

// ---------------------------------------------------------------- operand prep, direct
// Source walks k fastest (the common case once producers place the consumer's
// contracted bonds last): no smem transpose.  A thread owns 8 consecutive k of one
// row: 64 B of reads (16-B vectors when the innermost k dim is contiguous) and
// one 16-B store per plane; neighbouring threads take neighbouring k groups.
template <int PLANES>
__global__ void __launch_bounds__(256, 4) prep_direct_kernel(const PrepDesc* __restrict__ gd,
                                                             const int64_t* __restrict__ leaf_off) {
  __shared__ __align__(16) PrepDesc d;
  copy_desc_to_smem(&d, gd);
  const float2* src = d.src + d.off + (d.leaf >= 0 ? leaf_off[d.leaf] : 0);
  const float scale = prep_scale(d);
  const int64_t kgs = d.Kpad / 8;                      // Kpad is a multiple of 8
  const int64_t total = d.G * d.R * kgs;
  const bool kvec = d.nk > 0 && d.k_s[d.nk - 1] == 1 && (d.k_ext[d.nk - 1] % 8) == 0;
  for (int64_t w = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; w < total;
       w += (int64_t)gridDim.x * blockDim.x) {
    const int64_t kg = w % kgs, rg = w / kgs;
    const int64_t r = rg % d.R, g = rg / d.R;
    const int64_t k0 = kg * 8;
    float2 v[8];
    int64_t base;
    if (d.rowoff) {                  // kind 3: gathered rows (slab-grouped merge)
      base = d.rowoff[rg];
      if (base < 0) {                // padding row
#pragma unroll
        for (int j = 0; j < 8; ++j) v[j] = make_float2(0.f, 0.f);
        split_store8<PLANES>(d, rg * d.Kpad + k0, v, scale);
        continue;
      }
    } else {
      base = g * d.g_stride + decompose(r, d.nr, d.r_ext, d.r_s);
    }
    if (kvec && k0 + 8 <= d.K) {
      const float2* p = src + base + decompose(k0, d.nk, d.k_ext, d.k_s);
      if ((reinterpret_cast<uintptr_t>(p) & 15) == 0) {
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          const float4 q = reinterpret_cast<const float4*>(p)[j];
          v[2 * j] = make_float2(q.x, q.y);
          v[2 * j + 1] = make_float2(q.z, q.w);
        }
      } else {
#pragma unroll
        for (int j = 0; j < 8; ++j) v[j] = p[j];
      }
    } else {
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        const int64_t k = k0 + j;
        v[j] = k < d.K ? src[base + decompose(k, d.nk, d.k_ext, d.k_s)] : make_float2(0.f, 0.f);
      }
    }
    split_store8<PLANES>(d, rg * d.Kpad + k0, v, scale);
  }
}

// ---------------------------------------------------------------- operand prep, general
// Arbitrary permutation (cuTT-style): a tile is Bsz destination-contiguous
// elements (k-run of the plane rows) x Asz source-contiguous elements; block
// offset tables live in smem, so reads walk the source's innermost run and the
// half2 plane stores walk the destination's, whatever the interleaving.
template <int PLANES>
__global__ void __launch_bounds__(256, 3) prep_gt_kernel(const PrepDesc* __restrict__ gd,
                                                         const int64_t* __restrict__ leaf_off) {
  __shared__ __align__(16) PrepDesc d;
  copy_desc_to_smem(&d, gd);
  extern __shared__ __align__(16) uint8_t dyn[];
  const int T = d.T;
  int64_t* srcoff = reinterpret_cast<int64_t*>(dyn);            // [T] source order
  int64_t* dstoff = srcoff + T;                                  // [T] destination order
  float2* tile = reinterpret_cast<float2*>(dstoff + T);          // [T] source order
  int32_t* spos = reinterpret_cast<int32_t*>(tile + T);          // [T] dst order -> src index
  const float2* src = d.src + d.off + (d.leaf >= 0 ? leaf_off[d.leaf] : 0);
  const float scale = prep_scale(d);
  // tile tables (computed once at plan time), copied into smem
  const int32_t* gspos = reinterpret_cast<const int32_t*>(d.gt_tab + 2 * T);
  for (int e = threadIdx.x; e < T; e += blockDim.x) {
    srcoff[e] = d.gt_tab[e];
    dstoff[e] = d.gt_tab[T + e];
    spos[e] = gspos[e];
  }
  const int64_t plane = d.plane_elems;
  for (int64_t c = blockIdx.x; c < d.nC; c += gridDim.x) {
    // outer tile offsets: shift decomposition, evaluated by every thread (no serial step)
    int64_t sc = 0, dc = 0, t = c;
    for (int i = d.nc - 1; i >= 0; --i) {
      const int s = d.c_sh[i];
      const int64_t digit = t & ((int64_t(1) << s) - 1);
      t >>= s;
      sc += digit * d.c_src[i];
      dc += digit * d.c_dst[i];
    }
    __syncthreads();   // tables ready / previous tile consumed
    // tile slot of source-order element e is swizzled (e ^ ((e >> 5) & 31)) so the
    // strided destination-order reads spread over the banks
    for (int e = threadIdx.x; e < T; e += blockDim.x) tile[e ^ ((e >> 5) & 31)] = src[sc + srcoff[e]];
    __syncthreads();
    for (int f = 2 * threadIdx.x; f < T; f += 2 * blockDim.x) {
      const int p0 = spos[f], p1 = spos[f + 1];
      const float2 v0 = tile[p0 ^ ((p0 >> 5) & 31)], v1 = tile[p1 ^ ((p1 >> 5) & 31)];
      const float xr0 = v0.x * scale, xi0 = v0.y * scale, xr1 = v1.x * scale, xi1 = v1.y * scale;
      const __half2 hr = __floats2half2_rn(xr0, xr1), hi = __floats2half2_rn(xi0, xi1);
      const int64_t idx = dc + dstoff[f];             // dstoff[f+1] = dstoff[f] + 1, idx even
      reinterpret_cast<__half2*>(d.dst + idx)[0] = hr;
      reinterpret_cast<__half2*>(d.dst + plane + idx)[0] = hi;
      if (PLANES == 4) {
        const float2 fr = __half22float2(hr), fi = __half22float2(hi);
        reinterpret_cast<__half2*>(d.dst + 2 * plane + idx)[0] = __floats2half2_rn(xr0 - fr.x, xr1 - fr.y);
        reinterpret_cast<__half2*>(d.dst + 3 * plane + idx)[0] = __floats2half2_rn(xi0 - fi.x, xi1 - fi.y);
      }
    }
  }
}

// ---------------------------------------------------------------- operand prep, bit permutation
// Every extent of a circuit network is a power of two, so an operand permutation
// is a permutation of index bits: destination bit b carries source weight ws_b.
// A tile is 2^t elements spanned by t bits holding the destination's innermost
// bits (stored as 16-B plane vectors, walked in destination order) and the
// source's smallest-weight bits (read as 16-B pairs, walked in source order);
// the other bits enumerate tiles (outer weights in c_src / c_dst).  Tile offsets
// come from plan-time tables that are separable in the index bits, and the smem
// tile is XOR-swizzled per 16-slot row (mask chosen by the planner) so neither
// phase has bank conflicts.  All loads of a tile are issued before any use:
// 32 KB in flight per block, 4 blocks per SM.
// 16-B global -> shared copy without a register round trip (LDGSTS), L1 bypassed
__device__ __forceinline__ void cp_async16(void* smem, const void* gmem) {
  const uint32_t sa = (uint32_t)__cvta_generic_to_shared(smem);
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(sa), "l"(gmem) : "memory");
}
__device__ __forceinline__ void cp_async8(void* smem, const void* gmem) {
  const uint32_t sa = (uint32_t)__cvta_generic_to_shared(smem);
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(sa), "l"(gmem) : "memory");
}
__device__ __forceinline__ void cp_async_wait_all() {
  asm volatile("cp.async.commit_group;\ncp.async.wait_group 0;\n" ::: "memory");
}

// Outer tile offsets Σ_{bit i of c} (c_src[i], c_dst[i]) without a per-thread loop over
// the descriptor: lane i holds bit i's pair in registers (loaded once), the warp sums the
// set bits with a butterfly (every lane ends with the totals).  nc > 32: the plain loop.
struct TileBits {
  int64_t s0, d0;
};
__device__ __forceinline__ TileBits tile_bits_load(const int64_t* c_src, const int64_t* c_dst, int nc, int lane) {
  return TileBits{lane < nc ? c_src[lane] : 0, lane < nc ? c_dst[lane] : 0};
}
__device__ __forceinline__ void tile_bits_sum(const TileBits& t, uint64_t c, int lane, int nc, const int64_t* c_src,
                                              const int64_t* c_dst, int64_t& sc, int64_t& dc) {
  if (nc > 32) {
    sc = 0;
    dc = 0;
    for (int i = 0; i < nc; ++i)
      if ((c >> i) & 1) { sc += c_src[i]; dc += c_dst[i]; }
    return;
  }
  const bool b = (c >> lane) & 1u;
  int64_t s = b ? t.s0 : 0, d = b ? t.d0 : 0;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    s += __shfl_xor_sync(0xffffffffu, s, o);
    d += __shfl_xor_sync(0xffffffffu, d, o);
  }
  sc = s;
  dc = d;
}

constexpr int BP_TMAX = 4096;
constexpr size_t BP_SMEM = BP_TMAX * 8 + BP_TMAX / 8 * 8 + 128 * 8 + BP_TMAX * 2 + BP_TMAX / 16;

template <int PLANES>
__global__ void __launch_bounds__(256, 4) prep_bp_kernel(const PrepDesc* __restrict__ gd,
                                                         const int64_t* __restrict__ leaf_off) {
  __shared__ __align__(16) PrepDesc d;
  copy_desc_to_smem(&d, gd);
  extern __shared__ __align__(16) uint8_t dyn[];
  float2* tile = reinterpret_cast<float2*>(dyn);                          // [TMAX] swizzled
  int64_t* s_dst = reinterpret_cast<int64_t*>(tile + BP_TMAX);            // [TMAX/8]
  int64_t* s_src = s_dst + BP_TMAX / 8;                                   // [128] lo | hi
  uint16_t* s_slot = reinterpret_cast<uint16_t*>(s_src + 128);            // [TMAX]
  uint8_t* s_m = reinterpret_cast<uint8_t*>(s_slot + BP_TMAX);            // [TMAX/16]
  const int T = 1 << d.bp_t;
  {
    const int64_t* tab = d.bp_tab;
    for (int i = threadIdx.x; i < 128; i += blockDim.x) s_src[i] = tab[i];
    for (int i = threadIdx.x; i < T / 8; i += blockDim.x) s_dst[i] = tab[128 + i];
    const int64_t* ws = tab + 128 + T / 8;
    for (int i = threadIdx.x; i < T / 4; i += blockDim.x)
      reinterpret_cast<int64_t*>(s_slot)[i] = ws[i];
    const int64_t* wm = ws + T / 4;
    for (int i = threadIdx.x; i < (T / 16 + 7) / 8; i += blockDim.x)
      reinterpret_cast<int64_t*>(s_m)[i] = wm[i];
  }
  const float2* src = d.src + d.off + (d.leaf >= 0 ? leaf_off[d.leaf] : 0);
  const float scale = prep_scale(d);
  const bool vec = d.bp_vec && (reinterpret_cast<uintptr_t>(src) & 15) == 0;
  const int64_t tiles = d.G * d.nC;
  const int64_t rk = d.R * d.Kpad;
  const TileBits tb = tile_bits_load(d.c_src, d.c_dst, d.nc, threadIdx.x & 31);
  for (int64_t c = blockIdx.x; c < tiles; c += gridDim.x) {
    const int64_t g = c >> d.nc;                     // nC = 2^nc tiles per slab
    const int64_t cc = c - (g << d.nc);
    int64_t sc, dc;
    tile_bits_sum(tb, (uint64_t)cc, threadIdx.x & 31, d.nc, d.c_src, d.c_dst, sc, dc);
    sc += g * d.g_stride;
    dc += g * rk;
    __syncthreads();   // tables ready / previous tile consumed
    const float2* sp = src + sc;
    // every load of the tile in flight at once, straight to shared memory (LDGSTS)
    if (vec) {
#pragma unroll
      for (int i = 0; i < BP_TMAX / 512; ++i) {
        const int e = 2 * (threadIdx.x + i * 256);
        if (e < T) cp_async16(tile + (e ^ s_m[e >> 4]), sp + s_src[e & 63] + s_src[64 + (e >> 6)]);
      }
    } else {
#pragma unroll
      for (int i = 0; i < BP_TMAX / 256; ++i) {
        const int e = threadIdx.x + i * 256;
        if (e < T) cp_async8(tile + (e ^ s_m[e >> 4]), sp + s_src[e & 63] + s_src[64 + (e >> 6)]);
      }
    }
    cp_async_wait_all();
    __syncthreads();
#pragma unroll
    for (int i = 0; i < BP_TMAX / 2048; ++i) {
      const int q = threadIdx.x + i * 256;           // 8 destination-consecutive elements
      if (q < T / 8) {
        const uint4 sl = reinterpret_cast<const uint4*>(s_slot)[q];
        const uint32_t w[4] = {sl.x, sl.y, sl.z, sl.w};
        float2 v[8];
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          v[2 * j] = tile[w[j] & 0xFFFFu];
          v[2 * j + 1] = tile[w[j] >> 16];
        }
        split_store8<PLANES>(d, dc + s_dst[q], v, scale);
      }
    }
  }
}

// ---------------------------------------------------------------- operand prep, gate-folded
// The operand is out[o][n][v] = Σ_k Y[n][k] X[o, v, k] of a skinny SIMT step that is not
// run: a tile loads the X values of its carry bits (dest bits other than n) for every k,
// and each plane element applies the small matrix Y (staged in smem) while it is
// written.  Saves the skinny step's full pass over the big tensor.  Scale: |out| <=
// 2 K absmax(X) absmax(Y) per real component (bound, no absmax of out exists).
constexpr int GP_TMAX = 4096;
constexpr int GP_YMAX = 512, GP_NMAX = 256;

constexpr int GP_BUF = GP_TMAX + GP_TMAX / 32;     // X tile, then (aliased) the padded output tile
constexpr size_t GP_SMEM = GP_BUF * 8 + GP_YMAX * 8 + 128 * 8 /*src*/ + GP_TMAX / 8 * 8 /*dst*/ +
                           GP_TMAX * 2 /*fc*/ + GP_NMAX * 2 /*fn*/;

// output tile slot of destination-order element f: 16-B pairs (f >> 1) XOR-swizzled inside
// their 128-B row by bits 3-5 of the pair index, so the 8 lanes of a 128-bit read phase
// (pairs 4q + t, q = q0 .. q0 + 7) hit 8 different bank groups
__device__ __forceinline__ int gp_swz(int f) {
  const int u = f >> 1;
  return ((u ^ ((u >> 3) & 7)) << 1) | (f & 1);
}

__device__ __forceinline__ bool g_regroup_ok(int on, int TD, int N, int KT, int CB) {
  return on && TD == GP_TMAX && N % KT == 0 && CB % (16 / KT) == 0 &&
         (N / KT) * (CB / (16 / KT)) == 256;
}

// KT = K (gate inputs per output); a thread owns 16/KT carry positions, whose 16 X values
// it keeps in registers, so the X tile's smem is reused for the outputs (4 blocks/SM)
template <int PLANES, int KT>
__global__ void __launch_bounds__(256, 4) prep_gate_kernel(const PrepDesc* __restrict__ gd,
                                                           const int64_t* __restrict__ leaf_off) {
  __shared__ __align__(16) PrepDesc d;
  copy_desc_to_smem(&d, gd);
  extern __shared__ __align__(16) uint8_t dyn[];
  float2* buf = reinterpret_cast<float2*>(dyn);                      // [GP_BUF]
  float2* Ys = buf + GP_BUF;                                          // [N][KT]
  int64_t* s_src = reinterpret_cast<int64_t*>(Ys + GP_YMAX);          // [128]
  int64_t* s_dst = s_src + 128;                                       // [TD/8]
  uint16_t* s_fc = reinterpret_cast<uint16_t*>(s_dst + GP_TMAX / 8);  // [2^cb]
  uint16_t* s_fn = s_fc + GP_TMAX;                                    // [N]
  const int TD = 1 << d.bp_t, TS = 1 << d.g_ts, N = d.g_N, CB = 1 << d.g_cbits;
  {
    const int64_t* tab = d.bp_tab;
    for (int i = threadIdx.x; i < 128; i += blockDim.x) s_src[i] = tab[i];
    for (int i = threadIdx.x; i < TD / 8; i += blockDim.x) s_dst[i] = tab[128 + i];
    const uint16_t* fc = reinterpret_cast<const uint16_t*>(tab + 128 + TD / 8);
    for (int i = threadIdx.x; i < CB; i += blockDim.x) s_fc[i] = fc[i];
    for (int i = threadIdx.x; i < N; i += blockDim.x) s_fn[i] = fc[GP_TMAX + i];
    const float2* Y = d.gy + d.gy_off + (d.gy_leaf >= 0 ? leaf_off[d.gy_leaf] : 0);
    for (int e = threadIdx.x; e < N * KT; e += blockDim.x) {
      const int n = e / KT, k = e % KT;
      Ys[e] = Y[decompose(n, d.g_nn, d.gy_n_ext, d.gy_n_s) + decompose(k, d.g_nk, d.gy_k_ext, d.gy_k_s)];
    }
  }
  const float2* src = d.src + d.off + (d.leaf >= 0 ? leaf_off[d.leaf] : 0);
  float scale;
  {
    const float bound = 2.f * (float)KT * __uint_as_float(*d.absmax_in) * __uint_as_float(*d.absmax_y);
    int s = 0;
    if (bound > 0.f) {
      int e;
      frexpf(bound, &e);
      s = max(-120, min(120, 15 - e));
    }
    if (blockIdx.x == 0 && threadIdx.x == 0) *d.scale_out = s;
    scale = ldexpf(1.0f, s);
  }
  const bool vec = d.bp_vec && (reinterpret_cast<uintptr_t>(src) & 15) == 0;
  constexpr int CPT = 16 / KT;                    // carry positions per thread
  // regrouped compute (a full 4096-element tile, N a multiple of K): 256 threads x CPT
  // carry positions x KT outputs; Ys rows 16-B aligned for the paired loads
  const bool regroup = g_regroup_ok(d.g_regroup, TD, N, KT, CB);
  const TileBits tb = tile_bits_load(d.c_src, d.c_dst, d.nc, threadIdx.x & 31);
  for (int64_t c = blockIdx.x; c < d.nC; c += gridDim.x) {
    int64_t sc, dc;
    tile_bits_sum(tb, (uint64_t)c, threadIdx.x & 31, d.nc, d.c_src, d.c_dst, sc, dc);
    __syncthreads();   // tables / Y ready, previous tile's outputs consumed
    const float2* sp = src + sc;
    // every load of the tile in flight at once, straight to shared memory (LDGSTS)
    if (vec) {
#pragma unroll
      for (int i = 0; i < GP_TMAX / 512; ++i) {
        const int e = 2 * (threadIdx.x + i * 256);
        if (e < TS) cp_async16(buf + e, sp + s_src[e & 63] + s_src[64 + (e >> 6)]);
      }
    } else {
#pragma unroll
      for (int i = 0; i < GP_TMAX / 256; ++i) {
        const int e = threadIdx.x + i * 256;
        if (e < TS) cp_async8(buf + e, sp + s_src[e & 63] + s_src[64 + (e >> 6)]);
      }
    }
    cp_async_wait_all();
    __syncthreads();
    if (regroup) {
      // thread = (n group nq of KT outputs, carry group cg of CPT positions cg + r*CGN): every
      // Y row loaded (a warp-uniform broadcast) serves CPT outputs instead of one, and
      // consecutive lanes read consecutive carry positions of X (conflict-free)
      const int cgn = CB / CPT;
      const int nq = threadIdx.x / cgn, cg = threadIdx.x - nq * cgn;
      float2 xs[CPT][KT];
#pragma unroll
      for (int r = 0; r < CPT; ++r)
#pragma unroll
        for (int k = 0; k < KT; ++k) xs[r][k] = buf[cg + r * cgn + k * CB];
      __syncthreads();   // X tile read into registers: buf becomes the output tile
      // carry offsets cached in registers when each is reused KT >= 4 times (K <= 2: CPT >= 8
      // positions would not fit the 64-register budget next to the X values)
      constexpr bool FCR = KT >= 4;
      int fcs[FCR ? CPT : 1];
      if constexpr (FCR) {
#pragma unroll
        for (int r = 0; r < CPT; ++r) fcs[r] = s_fc[cg + r * cgn];
      }
#pragma unroll
      for (int jn = 0; jn < KT; ++jn) {
        const int n = nq * KT + jn;
        float2 y[KT];
        if constexpr (KT % 2 == 0) {
#pragma unroll
          for (int k = 0; k < KT; k += 2) {
            const float4 v = reinterpret_cast<const float4*>(Ys + n * KT)[k / 2];
            y[k] = make_float2(v.x, v.y);
            y[k + 1] = make_float2(v.z, v.w);
          }
        } else {
          y[0] = Ys[n];
        }
        const int fn = s_fn[n];
#pragma unroll
        for (int r = 0; r < CPT; ++r) {
          float ar = 0.f, ai = 0.f;
#pragma unroll
          for (int k = 0; k < KT; ++k) {
            ar = fmaf(xs[r][k].x, y[k].x, fmaf(-xs[r][k].y, y[k].y, ar));
            ai = fmaf(xs[r][k].x, y[k].y, fmaf(xs[r][k].y, y[k].x, ai));
          }
          const int f = (FCR ? fcs[FCR ? r : 0] : (int)s_fc[cg + r * cgn]) + fn;
          buf[gp_swz(f)] = make_float2(ar, ai);
        }
      }
      __syncthreads();
      for (int q = threadIdx.x; q < TD / 8; q += blockDim.x) {
        float2 o[8];
#pragma unroll
        for (int j = 0; j < 8; j += 2) {   // 16-B pairs, conflict-free under the swizzle
          const float4 v = reinterpret_cast<const float4*>(buf)[gp_swz(8 * q + j) >> 1];
          o[j] = make_float2(v.x, v.y);
          o[j + 1] = make_float2(v.z, v.w);
        }
        split_store8<PLANES>(d, dc + s_dst[q], o, scale);
      }
      continue;
    }
    float2 xs[CPT][KT];
#pragma unroll
    for (int i = 0; i < CPT; ++i) {
      const int cp = threadIdx.x + i * 256;
#pragma unroll
      for (int k = 0; k < KT; ++k) xs[i][k] = cp < CB ? buf[cp + k * CB] : make_float2(0.f, 0.f);
    }
    __syncthreads();   // X tile read into registers: buf becomes the output tile
#pragma unroll
    for (int i = 0; i < CPT; ++i) {
      const int cp = threadIdx.x + i * 256;
      if (cp >= CB) continue;
      const int fcp = s_fc[cp];
      for (int n = 0; n < N; ++n) {
        const float2* yr = Ys + n * KT;
        float ar = 0.f, ai = 0.f;
#pragma unroll
        for (int k = 0; k < KT; ++k) {
          const float2 y = yr[k];
          ar = fmaf(xs[i][k].x, y.x, fmaf(-xs[i][k].y, y.y, ar));
          ai = fmaf(xs[i][k].x, y.y, fmaf(xs[i][k].y, y.x, ai));
        }
        const int f = fcp + s_fn[n];
        buf[f + (f >> 5)] = make_float2(ar, ai);
      }
    }
    __syncthreads();
    for (int q = threadIdx.x; q < TD / 8; q += blockDim.x) {
      float2 o[8];
#pragma unroll
      for (int j = 0; j < 8; ++j) o[j] = buf[8 * q + j + ((8 * q) >> 5)];
      split_store8<PLANES>(d, dc + s_dst[q], o, scale);
    }
  }
}

// Tensor-core variant of the gate-folded prep (K = 4, 8, 16 and N <= 8 * NB): the small
// contraction out[carry][n] = Σ_k X[carry][k] Y[n][k] of a tile runs as warp-level
// m16n8k16 fp16 MMAs with fp32 accumulation in the 3-pass hi/lo split of Eq. 8
// (X and Y each carry their own power-of-two scale) and the complex
// product as four real ones (Cr = Xr Yr - Xi Yi, Ci = Xr Yi + Xi Yr).  The FFMA kernel
// above spends 4 K FFMA per output element (32 for K = 8): it is issue-bound on the
// 2^32-element stem operands; here a warp issues 12 MMAs per 16 x 8 outputs.  Y's
// fragments stay in registers for the whole kernel.
__device__ __forceinline__ uint32_t pack_h2(__half lo, __half hi) {
  return (uint32_t)__half_as_ushort(lo) | ((uint32_t)__half_as_ushort(hi) << 16);
}
__device__ __forceinline__ void split_h(float x, __half& h, __half& l) {
  h = __float2half_rn(x);
  l = __float2half_rn(x - __half2float(h));
}
__device__ __forceinline__ void mma16816(float* c, const uint32_t* a, const uint32_t* b) {
  asm volatile(
      "mma.sync.aligned.m16n8k16.row.col.f32.f16.f16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
      "{%0,%1,%2,%3};"
      : "+f"(c[0]), "+f"(c[1]), "+f"(c[2]), "+f"(c[3])
      : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b[0]), "r"(b[1]));
}

template <int PLANES, int KT, int NB>
__global__ void __launch_bounds__(256, 2) prep_gate_mma_kernel(const PrepDesc* __restrict__ gd,
                                                               const int64_t* __restrict__ leaf_off) {
  static_assert(KT == 4 || KT == 8 || KT == 16, "K padded to one m16n8k16 step");
  __shared__ __align__(16) PrepDesc d;
  copy_desc_to_smem(&d, gd);
  extern __shared__ __align__(16) uint8_t dyn[];
  float2* buf = reinterpret_cast<float2*>(dyn);                      // [GP_BUF] X tile
  float2* obuf = buf + GP_BUF;                                        // [GP_BUF] padded outputs
  float2* Ys = obuf + GP_BUF;                                         // [N][KT]
  int64_t* s_src = reinterpret_cast<int64_t*>(Ys + GP_YMAX);          // [128]
  int64_t* s_dst = s_src + 128;                                       // [TD/8]
  uint16_t* s_fc = reinterpret_cast<uint16_t*>(s_dst + GP_TMAX / 8);  // [2^cb]
  uint16_t* s_fn = s_fc + GP_TMAX;                                    // [N]
  const int TD = 1 << d.bp_t, TS = 1 << d.g_ts, N = d.g_N, CB = 1 << d.g_cbits;
  {
    const int64_t* tab = d.bp_tab;
    for (int i = threadIdx.x; i < 128; i += blockDim.x) s_src[i] = tab[i];
    for (int i = threadIdx.x; i < TD / 8; i += blockDim.x) s_dst[i] = tab[128 + i];
    const uint16_t* fc = reinterpret_cast<const uint16_t*>(tab + 128 + TD / 8);
    for (int i = threadIdx.x; i < CB; i += blockDim.x) s_fc[i] = fc[i];
    for (int i = threadIdx.x; i < N; i += blockDim.x) s_fn[i] = fc[GP_TMAX + i];
    const float2* Y = d.gy + d.gy_off + (d.gy_leaf >= 0 ? leaf_off[d.gy_leaf] : 0);
    for (int e = threadIdx.x; e < N * KT; e += blockDim.x) {
      const int n = e / KT, k = e % KT;
      Ys[e] = Y[decompose(n, d.g_nn, d.gy_n_ext, d.gy_n_s) + decompose(k, d.g_nk, d.gy_k_ext, d.gy_k_s)];
    }
  }
  const float2* src = d.src + d.off + (d.leaf >= 0 ? leaf_off[d.leaf] : 0);
  // scales: X and Y to the fp16 range (each |.| * 2^s < 2^15), the planes as the FFMA kernel
  const float ax = __uint_as_float(*d.absmax_in), ay = __uint_as_float(*d.absmax_y);
  auto exp15 = [](float a) {
    int e = 0;
    if (a > 0.f) frexpf(a, &e);
    return a > 0.f ? max(-120, min(120, 15 - e)) : 0;
  };
  const int sx = exp15(ax), sy = exp15(ay);
  float scale;
  {
    const float bound = 2.f * (float)KT * ax * ay;
    const int s = exp15(bound);
    if (blockIdx.x == 0 && threadIdx.x == 0) *d.scale_out = s;
    scale = ldexpf(1.0f, s);
  }
  const float fx = ldexpf(1.0f, sx), fy = ldexpf(1.0f, sy);
  const float ux = ldexpf(1.0f, -sx), uy = ldexpf(1.0f, -sy);
  __syncthreads();
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int g = lane >> 2, t = lane & 3;
  // B fragments (k x n, col): b0 = k {2t, 2t+1}, b1 = k {2t+8, 2t+9}, column n = 8 nb + g
  // of Yr, Yi and -Yi, each split hi / lo
  uint32_t bf[NB][6][2];
#pragma unroll
  for (int nb = 0; nb < NB; ++nb) {
    const int n = nb * 8 + g;
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      __half rh[2], rl[2], ih[2], il[2], nh[2], nl[2];
#pragma unroll
      for (int u = 0; u < 2; ++u) {
        const int k = 2 * t + 8 * h + u;
        const float2 y = (n < N && k < KT) ? Ys[n * KT + k] : make_float2(0.f, 0.f);
        split_h(y.x * fy, rh[u], rl[u]);
        split_h(y.y * fy, ih[u], il[u]);
        split_h(-y.y * fy, nh[u], nl[u]);
      }
      bf[nb][0][h] = pack_h2(rh[0], rh[1]);
      bf[nb][1][h] = pack_h2(rl[0], rl[1]);
      bf[nb][2][h] = pack_h2(ih[0], ih[1]);
      bf[nb][3][h] = pack_h2(il[0], il[1]);
      bf[nb][4][h] = pack_h2(nh[0], nh[1]);
      bf[nb][5][h] = pack_h2(nl[0], nl[1]);
    }
  }
  const bool vec = d.bp_vec && (reinterpret_cast<uintptr_t>(src) & 15) == 0;
  const int nrb = CB / 16;
  for (int64_t c = blockIdx.x; c < d.nC; c += gridDim.x) {
    int64_t sc = 0, dc = 0;
    for (int i = 0; i < d.nc; ++i)
      if ((c >> i) & 1) { sc += d.c_src[i]; dc += d.c_dst[i]; }
    __syncthreads();   // previous tile's outputs consumed
    const float2* sp = src + sc;
    if (vec) {
#pragma unroll
      for (int i = 0; i < GP_TMAX / 512; ++i) {
        const int e = 2 * (threadIdx.x + i * 256);
        if (e < TS) cp_async16(buf + e, sp + s_src[e & 63] + s_src[64 + (e >> 6)]);
      }
    } else {
#pragma unroll
      for (int i = 0; i < GP_TMAX / 256; ++i) {
        const int e = threadIdx.x + i * 256;
        if (e < TS) cp_async8(buf + e, sp + s_src[e & 63] + s_src[64 + (e >> 6)]);
      }
    }
    cp_async_wait_all();
    __syncthreads();
    // per 16-carry row block of this warp: A fragments from the X tile (element (carry, k)
    // at buf[carry + k*CB]; a0 = (g, k 2t..2t+1), a1 = (g+8, ..), a2 = (g, k+8), a3 = (g+8,
    // k+8)), 12 MMAs per 8 output columns, outputs into the padded output tile
    for (int rb = warp; rb < nrb; rb += 8) {
      uint32_t af[4][4];                        // [Xr_h, Xr_l, Xi_h, Xi_l][reg]
#pragma unroll
      for (int r = 0; r < 4; ++r) {
        const int row = rb * 16 + g + ((r & 1) ? 8 : 0);
        const int k0 = 2 * t + ((r & 2) ? 8 : 0);
        __half xrh[2], xrl[2], xih[2], xil[2];
#pragma unroll
        for (int u = 0; u < 2; ++u) {
          const int k = k0 + u;
          const float2 x = k < KT ? buf[row + k * CB] : make_float2(0.f, 0.f);
          split_h(x.x * fx, xrh[u], xrl[u]);
          split_h(x.y * fx, xih[u], xil[u]);
        }
        af[0][r] = pack_h2(xrh[0], xrh[1]);
        af[1][r] = pack_h2(xrl[0], xrl[1]);
        af[2][r] = pack_h2(xih[0], xih[1]);
        af[3][r] = pack_h2(xil[0], xil[1]);
      }
#pragma unroll
      for (int nb = 0; nb < NB; ++nb) {
        float cr[4] = {0.f, 0.f, 0.f, 0.f}, ci[4] = {0.f, 0.f, 0.f, 0.f};
        // small terms first, big x big last (Eq. 8)
        mma16816(cr, af[0], bf[nb][1]);   // Xr_h Yr_l
        mma16816(cr, af[1], bf[nb][0]);   // Xr_l Yr_h
        mma16816(cr, af[2], bf[nb][5]);   // Xi_h (-Yi)_l
        mma16816(cr, af[3], bf[nb][4]);   // Xi_l (-Yi)_h
        mma16816(ci, af[0], bf[nb][3]);   // Xr_h Yi_l
        mma16816(ci, af[1], bf[nb][2]);   // Xr_l Yi_h
        mma16816(ci, af[2], bf[nb][1]);   // Xi_h Yr_l
        mma16816(ci, af[3], bf[nb][0]);   // Xi_l Yr_h
        mma16816(cr, af[0], bf[nb][0]);   // Xr_h Yr_h
        mma16816(cr, af[2], bf[nb][4]);   // Xi_h (-Yi)_h
        mma16816(ci, af[0], bf[nb][2]);   // Xr_h Yi_h
        mma16816(ci, af[2], bf[nb][0]);   // Xi_h Yr_h
        // c0, c1: (row g, n 2t, 2t+1); c2, c3: (row g+8, ...)
#pragma unroll
        for (int r = 0; r < 4; ++r) {
          const int row = rb * 16 + g + ((r & 2) ? 8 : 0);
          const int n = nb * 8 + 2 * t + (r & 1);
          if (n < N) {
            const int f = s_fc[row] + s_fn[n];
            obuf[f + (f >> 5)] = make_float2(cr[r] * ux * uy, ci[r] * ux * uy);
          }
        }
      }
    }
    __syncthreads();
    for (int q = threadIdx.x; q < TD / 8; q += blockDim.x) {
      float2 o[8];
#pragma unroll
      for (int j = 0; j < 8; ++j) o[j] = obuf[8 * q + j + ((8 * q) >> 5)];
      split_store8<PLANES>(d, dc + s_dst[q], o, scale);
    }
  }
}

// ---------------------------------------------------------------- SIMT einsum, general
// One thread per output C[j][m][n]; fp64 accumulation (a long fp32 RN chain would
// cost ~2^-24·sqrt(K/2) relative).
__global__ void __launch_bounds__(256) einsum_kernel(const EinsumDesc* __restrict__ gd,
                                                     const int64_t* __restrict__ leaf_off,
                                                     int64_t total) {
  __shared__ __align__(16) EinsumDesc d;
  copy_desc_to_smem(&d, gd);
  const float2* A = d.A + d.a_off + (d.a_leaf >= 0 ? leaf_off[d.a_leaf] : 0);
  const float2* B = d.B + d.b_off + (d.b_leaf >= 0 ? leaf_off[d.b_leaf] : 0);
  const int nk = d.nk;
  const int64_t klast = nk > 0 ? d.k_ext[nk - 1] : 1;
  const int64_t ka_last = nk > 0 ? d.k_sa[nk - 1] : 0;
  const int64_t kb_last = nk > 0 ? d.k_sb[nk - 1] : 0;
  const int64_t kouter = nk > 0 ? d.K / klast : 1;
  float amax = 0.f;
  for (int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; idx < total;
       idx += (int64_t)gridDim.x * blockDim.x) {
    const int64_t n = idx % d.N;
    const int64_t t1 = idx / d.N;
    const int64_t m = t1 % d.M;
    const int64_t j = t1 / d.M;
    const int64_t ao = (d.ia ? (int64_t)d.ia[j] : 0) * d.a_gs + decompose(m, d.nm, d.m_ext, d.m_sa);
    const int64_t bo = (d.ib ? (int64_t)d.ib[j] : 0) * d.b_gs + decompose(n, d.nn, d.n_ext, d.n_sb);
    double cr = 0.0, ci = 0.0;
    for (int64_t ko = 0; ko < kouter; ++ko) {
      const int64_t ak = ao + decompose(ko, nk - 1, d.k_ext, d.k_sa);
      const int64_t bk = bo + decompose(ko, nk - 1, d.k_ext, d.k_sb);
      for (int64_t ki = 0; ki < klast; ++ki) {
        const float2 a = A[ak + ki * ka_last];
        const float2 b = B[bk + ki * kb_last];
        cr = fma((double)a.x, (double)b.x, cr);
        cr = fma(-(double)a.y, (double)b.y, cr);
        ci = fma((double)a.x, (double)b.y, ci);
        ci = fma((double)a.y, (double)b.x, ci);
      }
    }
    store_out(d, idx, cr, ci, amax);
  }
  if (d.absmax_out) block_absmax(amax, d.absmax_out);
}

// ---------------------------------------------------------------- SIMT einsum, skinny
// C[o][n][v] = Σ_k A[o, v, k] B[n, k] for a small B (N*K <= 8192 complex, staged
// in smem once per block, rows padded to an even N) and a big A streamed exactly
// once: lanes walk A's smallest-stride free dim v (coalesced reads), the output
// keeps v innermost (coalesced writes).  These are the HBM-bound "absorb a gate
// into the stem" steps (stage 1 dominates).  VEC = 2: a thread
// owns the pair (v, v+1) (unit-stride, even run): 16-B loads and stores.  The k
// loop issues KU loads before any use (memory-level parallelism), and B is read
// as 16-B pairs of n, so one shared-memory load feeds 8·VEC FMAs.  fp32
// accumulation (K <= 256 here).
template <int NMAX, int VEC, bool POW2, int KP, int R>
__global__ void __launch_bounds__(256) einsum_skinny_kernel(const EinsumDesc* __restrict__ gd,
                                                            const int64_t* __restrict__ leaf_off) {
  __shared__ __align__(16) EinsumDesc d;
  copy_desc_to_smem(&d, gd);
  extern __shared__ __align__(16) uint8_t dyn[];
  const int K = (int)d.K, N = (int)d.N, Np = (N + 1) & ~1;
  // batched merges (J > 1, R = 1): every slab of the small operand is staged, batch j
  // reads X slab ia[j] and Y slab ib[j]; the output is [J][Xo][N][V]
  const int GY = d.J > 1 ? (int)d.n_yslabs : 1;
  float2* Bs = reinterpret_cast<float2*>(dyn);                 // [GY][K][Np]
  int64_t* koff = reinterpret_cast<int64_t*>(dyn + sizeof(float2) * GY * K * Np);
  const float2* A = d.A + d.a_off + (d.a_leaf >= 0 ? leaf_off[d.a_leaf] : 0);
  const float2* B = d.B + d.b_off + (d.b_leaf >= 0 ? leaf_off[d.b_leaf] : 0);
  for (int e = threadIdx.x; e < GY * K * Np; e += blockDim.x) {
    const int sy = e / (K * Np), ee = e % (K * Np);
    const int k = ee / Np, n = ee % Np;
    Bs[e] = n < N ? B[sy * d.b_gs + decompose(n, d.nn, d.n_ext, d.n_sb) + decompose(k, d.nk, d.k_ext, d.k_sb)]
                  : make_float2(0.f, 0.f);
  }
  for (int k = threadIdx.x; k < K; k += blockDim.x) koff[k] = decompose(k, d.nk, d.k_ext, d.k_sa);
  __syncthreads();
  // k values loaded per row before any use; R rows per thread (grid-stride apart, so
  // every warp access stays lane-coalesced): R·KU·VEC·8 B in flight per thread
  constexpr int KU = R == 4 ? 4 : (R == 2 ? (VEC == 2 ? 4 : 8) : (NMAX <= 16 ? 8 : 4));
  const int64_t V = d.V, Vv = V / VEC, Mb = d.M / VEC, Mv = d.J * Mb;
  const bool vv_p2 = (Vv & (Vv - 1)) == 0, mb_p2 = (Mb & (Mb - 1)) == 0;
  const int lvv = __ffsll(Vv) - 1, lmb = __ffsll(Mb) - 1;
  const int64_t vstride = d.m_sa[d.nm - 1];
  const int64_t step = (int64_t)gridDim.x * blockDim.x;
  float amax = 0.f;
  for (int64_t m0 = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; m0 < Mv; m0 += R * step) {
    const float2* a_row[R];
    int64_t obase[R];
    bool live[R];
    int64_t bslab = 0;                 // J > 1 runs with R = 1
#pragma unroll
    for (int r = 0; r < R; ++r) {
      const int64_t m = m0 + r * step;
      live[r] = m < Mv;
      int64_t mm = live[r] ? m : m0, jb = 0;
      if (d.J > 1) {
        jb = mb_p2 ? (mm >> lmb) : mm / Mb;
        mm -= jb * Mb;
      }
      // power-of-two extents: shifts instead of 64-bit division (emulated, ~100 instructions)
      const int64_t vi = (vv_p2 ? (mm & (Vv - 1)) : (mm % Vv)) * VEC, o = vv_p2 ? (mm >> lvv) : mm / Vv;
      a_row[r] = A + (d.J > 1 ? (int64_t)d.ia[jb] * d.a_gs : 0) +
                 (POW2 ? decompose_sh(o, d.nm - 1, d.m_sh, d.m_sa) : decompose(o, d.nm - 1, d.m_ext, d.m_sa)) +
                 vi * vstride;
      obase[r] = jb * d.M * N + o * N * V + vi;
      if (r == 0 && d.J > 1) bslab = (int64_t)d.ib[jb] * K * Np;
    }
    float cr[R][VEC][NMAX], ci[R][VEC][NMAX];
#pragma unroll
    for (int r = 0; r < R; ++r)
#pragma unroll
      for (int u = 0; u < VEC; ++u)
#pragma unroll
        for (int n = 0; n < NMAX; ++n) { cr[r][u][n] = 0.f; ci[r][u][n] = 0.f; }
    for (int k0 = 0; k0 < K; k0 += KU) {
      float2 a[KU][R][VEC];
#pragma unroll
      for (int r = 0; r < R; ++r) {
        if (KP == 2) {     // (k, k+1) adjacent in A (innermost k dim unit-stride): 16-B loads
#pragma unroll
          for (int kk = 0; kk < KU; kk += 2) {
            if (k0 + kk < K) {
              const float4 q = __ldg(reinterpret_cast<const float4*>(a_row[r] + koff[k0 + kk]));
              a[kk][r][0] = make_float2(q.x, q.y);
              a[kk + 1][r][0] = make_float2(q.z, q.w);
            } else {
              a[kk][r][0] = make_float2(0.f, 0.f);
              a[kk + 1][r][0] = make_float2(0.f, 0.f);
            }
          }
        } else {
#pragma unroll
          for (int kk = 0; kk < KU; ++kk) {
            if (k0 + kk < K) {
              if (VEC == 2) {
                const float4 q = __ldg(reinterpret_cast<const float4*>(a_row[r] + koff[k0 + kk]));
                a[kk][r][0] = make_float2(q.x, q.y);
                a[kk][r][VEC - 1] = make_float2(q.z, q.w);
              } else {
                a[kk][r][0] = __ldg(a_row[r] + koff[k0 + kk]);
              }
            } else {
#pragma unroll
              for (int u = 0; u < VEC; ++u) a[kk][r][u] = make_float2(0.f, 0.f);
            }
          }
        }
      }
#pragma unroll
      for (int kk = 0; kk < KU; ++kk) {
        if (k0 + kk < K) {
          const float4* brow = reinterpret_cast<const float4*>(Bs + bslab + (k0 + kk) * Np);
#pragma unroll
          for (int n2 = 0; n2 < NMAX / 2; ++n2) {
            if (2 * n2 < N) {
              const float4 b = brow[n2];     // B[2n2] = (x, y), B[2n2+1] = (z, w)
#pragma unroll
              for (int r = 0; r < R; ++r)
#pragma unroll
                for (int u = 0; u < VEC; ++u) {
                  const float2 x = a[kk][r][u];
                  cr[r][u][2 * n2] = fmaf(x.x, b.x, fmaf(-x.y, b.y, cr[r][u][2 * n2]));
                  ci[r][u][2 * n2] = fmaf(x.x, b.y, fmaf(x.y, b.x, ci[r][u][2 * n2]));
                  cr[r][u][2 * n2 + 1] = fmaf(x.x, b.z, fmaf(-x.y, b.w, cr[r][u][2 * n2 + 1]));
                  ci[r][u][2 * n2 + 1] = fmaf(x.x, b.w, fmaf(x.y, b.z, ci[r][u][2 * n2 + 1]));
                }
            }
          }
        }
      }
    }
#pragma unroll
    for (int r = 0; r < R; ++r) {
      if (!live[r]) continue;
#pragma unroll
      for (int n = 0; n < NMAX; ++n) {
        if (n < N) {
          const int64_t idx = obase[r] + (int64_t)n * V;
          if (VEC == 2 && !d.acc) {
            *reinterpret_cast<float4*>(d.C + idx) =
                make_float4(cr[r][0][n], ci[r][0][n], cr[r][VEC - 1][n], ci[r][VEC - 1][n]);
            amax = fmaxf(amax, fmaxf(fmaxf(fabsf(cr[r][0][n]), fabsf(ci[r][0][n])),
                                     fmaxf(fabsf(cr[r][VEC - 1][n]), fabsf(ci[r][VEC - 1][n]))));
          } else {
#pragma unroll
            for (int u = 0; u < VEC; ++u) store_out_f(d, idx + u, cr[r][u][n], ci[r][u][n], amax);
          }
        }
      }
    }
  }
  if (d.absmax_out) block_absmax(amax, d.absmax_out);
}

// ---------------------------------------------------------------- SIMT einsum, wide skinny
// Same layout contract as einsum_skinny_kernel (out [Mo][N][V]) for outer-product-
// like steps: K <= KMAX (the big operand's row lives in registers), N up to 4096
// (small operand staged in smem as [N][Kp], Kp = even K, read as 16-B pairs of k),
// outputs streamed n by n with lanes along v; VEC = 2 as in the skinny kernel.
template <int KMAX, int VEC, int KP>
__global__ void __launch_bounds__(256) einsum_wide_kernel(const EinsumDesc* __restrict__ gd,
                                                          const int64_t* __restrict__ leaf_off) {
  __shared__ __align__(16) EinsumDesc d;
  copy_desc_to_smem(&d, gd);
  extern __shared__ __align__(16) uint8_t dyn[];
  const int K = (int)d.K, N = (int)d.N, Kp = (K + 1) & ~1;
  float2* Bs = reinterpret_cast<float2*>(dyn);                 // [N][Kp]
  const float2* A = d.A + d.a_off + (d.a_leaf >= 0 ? leaf_off[d.a_leaf] : 0);
  const float2* B = d.B + d.b_off + (d.b_leaf >= 0 ? leaf_off[d.b_leaf] : 0);
  for (int e = threadIdx.x; e < Kp * N; e += blockDim.x) {
    const int n = e / Kp, k = e % Kp;
    Bs[e] = k < K ? B[decompose(n, d.nn, d.n_ext, d.n_sb) + decompose(k, d.nk, d.k_ext, d.k_sb)]
                  : make_float2(0.f, 0.f);
  }
  __syncthreads();
  const int64_t V = d.V, Vv = V / VEC, Mv = d.M / VEC;
  const bool vv_p2 = (Vv & (Vv - 1)) == 0;
  const int lvv = __ffsll(Vv) - 1;
  const int64_t vstride = d.m_sa[d.nm - 1];
  float amax = 0.f;
  for (int64_t m = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; m < Mv;
       m += (int64_t)gridDim.x * blockDim.x) {
    const int64_t vi = (vv_p2 ? (m & (Vv - 1)) : (m % Vv)) * VEC, o = vv_p2 ? (m >> lvv) : m / Vv;
    const float2* a_row = A + decompose(o, d.nm - 1, d.m_ext, d.m_sa) + vi * vstride;
    float2 a[KMAX][VEC];
    if (KP == 2) {         // (k, k+1) adjacent in A: 16-B loads
#pragma unroll
      for (int k = 0; k < KMAX; k += 2) {
        if (k < K) {
          const float4 q = __ldg(reinterpret_cast<const float4*>(a_row + decompose(k, d.nk, d.k_ext, d.k_sa)));
          a[k][0] = make_float2(q.x, q.y);
          a[k + 1][0] = make_float2(q.z, q.w);
        } else {
          a[k][0] = make_float2(0.f, 0.f);
          a[k + 1][0] = make_float2(0.f, 0.f);
        }
      }
    } else
#pragma unroll
    for (int k = 0; k < KMAX; ++k) {
      if (k < K) {
        const float2* p = a_row + decompose(k, d.nk, d.k_ext, d.k_sa);
        if (VEC == 2) {
          const float4 q = __ldg(reinterpret_cast<const float4*>(p));
          a[k][0] = make_float2(q.x, q.y);
          a[k][VEC - 1] = make_float2(q.z, q.w);
        } else {
          a[k][0] = __ldg(p);
        }
      } else {
#pragma unroll
        for (int u = 0; u < VEC; ++u) a[k][u] = make_float2(0.f, 0.f);
      }
    }
    float2* crow = d.C + o * N * V + vi;
    for (int n = 0; n < N; ++n) {
      float cr[VEC], ci[VEC];
#pragma unroll
      for (int u = 0; u < VEC; ++u) { cr[u] = 0.f; ci[u] = 0.f; }
      const float4* brow = reinterpret_cast<const float4*>(Bs + n * Kp);
#pragma unroll
      for (int k2 = 0; k2 < KMAX / 2; ++k2) {
        if (2 * k2 < K) {
          const float4 b = brow[k2];         // B[n][2k2] = (x, y), B[n][2k2+1] = (z, w)
#pragma unroll
          for (int u = 0; u < VEC; ++u) {
            const float2 x0 = a[2 * k2][u], x1 = a[2 * k2 + 1][u];
            cr[u] = fmaf(x0.x, b.x, fmaf(-x0.y, b.y, fmaf(x1.x, b.z, fmaf(-x1.y, b.w, cr[u]))));
            ci[u] = fmaf(x0.x, b.y, fmaf(x0.y, b.x, fmaf(x1.x, b.w, fmaf(x1.y, b.z, ci[u]))));
          }
        }
      }
      if (VEC == 2 && !d.acc) {
        *reinterpret_cast<float4*>(crow + (int64_t)n * V) = make_float4(cr[0], ci[0], cr[VEC - 1], ci[VEC - 1]);
        amax = fmaxf(amax, fmaxf(fmaxf(fabsf(cr[0]), fabsf(ci[0])), fmaxf(fabsf(cr[VEC - 1]), fabsf(ci[VEC - 1]))));
      } else {
#pragma unroll
        for (int u = 0; u < VEC; ++u)
          store_out_f(d, (o * N + n) * V + vi + u, cr[u], ci[u], amax);
      }
    }
  }
  if (d.absmax_out) block_absmax(amax, d.absmax_out);
}

// ---------------------------------------------------------------- SIMT einsum, skinny (previous design, TN_SIMT_OLD=1 A/B)
// C[o][n][v] = Σ_k A[o, v, k] B[n, k] for a small B (N*K <= 8192 complex, staged
// in smem once per block) and a big A streamed exactly once: lanes walk A's
// smallest-stride free dim v (coalesced reads), the output keeps v innermost
// (coalesced writes).  These are the HBM-bound "absorb a gate into the stem"
// steps (stage 1 dominates).  fp32 accumulation (K <= 64 here).
template <int NMAX, bool POW2>
__global__ void __launch_bounds__(256) einsum_skinny_old_kernel(const EinsumDesc* __restrict__ gd,
                                                            const int64_t* __restrict__ leaf_off) {
  __shared__ __align__(16) EinsumDesc d;
  copy_desc_to_smem(&d, gd);
  extern __shared__ __align__(16) uint8_t dyn[];
  const int K = (int)d.K, N = (int)d.N;
  float2* Bs = reinterpret_cast<float2*>(dyn);                 // [K][N]
  int64_t* koff = reinterpret_cast<int64_t*>(dyn + sizeof(float2) * K * N);
  const float2* A = d.A + d.a_off + (d.a_leaf >= 0 ? leaf_off[d.a_leaf] : 0);
  const float2* B = d.B + d.b_off + (d.b_leaf >= 0 ? leaf_off[d.b_leaf] : 0);
  for (int e = threadIdx.x; e < K * N; e += blockDim.x) {
    const int k = e / N, n = e % N;
    Bs[e] = B[decompose(n, d.nn, d.n_ext, d.n_sb) + decompose(k, d.nk, d.k_ext, d.k_sb)];
  }
  for (int k = threadIdx.x; k < K; k += blockDim.x) koff[k] = decompose(k, d.nk, d.k_ext, d.k_sa);
  __syncthreads();
  const int64_t V = d.V;
  const bool vp2 = (V & (V - 1)) == 0;
  const int lv = __ffsll(V) - 1;
  const int64_t vstride = d.m_sa[d.nm - 1];
  // U rows per thread per iteration (independent loads in flight); U = 2 while
  // the accumulators fit comfortably in registers
  constexpr int U = NMAX <= 16 ? 2 : 1;
  const int64_t step = (int64_t)gridDim.x * blockDim.x;
  float amax = 0.f;
  for (int64_t m0 = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; m0 < d.M; m0 += U * step) {
    const float2* a_row[U];
    int64_t obase[U];
    bool live[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int64_t m = m0 + u * step;
      live[u] = m < d.M;
      const int64_t mm = live[u] ? m : m0;
      const int64_t vi = POW2 ? (mm & (V - 1)) : mm % V, o = POW2 ? (mm >> lv) : mm / V;
      a_row[u] = A + (POW2 ? decompose_sh(o, d.nm - 1, d.m_sh, d.m_sa)
                           : decompose(o, d.nm - 1, d.m_ext, d.m_sa)) + vi * vstride;
      obase[u] = o * N * V + vi;
    }
    float accr[U][NMAX], acci[U][NMAX];
#pragma unroll
    for (int u = 0; u < U; ++u)
#pragma unroll
      for (int n = 0; n < NMAX; ++n) { accr[u][n] = 0.f; acci[u][n] = 0.f; }
    for (int k = 0; k < K; ++k) {
      float2 a[U];
#pragma unroll
      for (int u = 0; u < U; ++u) a[u] = a_row[u][koff[k]];
#pragma unroll
      for (int n = 0; n < NMAX; ++n) {
        if (n < N) {
          const float2 b = Bs[k * N + n];
#pragma unroll
          for (int u = 0; u < U; ++u) {
            accr[u][n] = fmaf(a[u].x, b.x, accr[u][n]);
            accr[u][n] = fmaf(-a[u].y, b.y, accr[u][n]);
            acci[u][n] = fmaf(a[u].x, b.y, acci[u][n]);
            acci[u][n] = fmaf(a[u].y, b.x, acci[u][n]);
          }
        }
      }
    }
#pragma unroll
    for (int u = 0; u < U; ++u)
      if (live[u])
#pragma unroll
        for (int n = 0; n < NMAX; ++n)
          if (n < N) store_out_f(d, obase[u] + (int64_t)n * V, accr[u][n], acci[u][n], amax);
  }
  if (d.absmax_out) block_absmax(amax, d.absmax_out);
}

// Vectorised variant: the lane run v is unit-stride and even, so a thread owns the
// pair (v, v+1): one 16-byte load per k and one 16-byte store per n (pairs are
// adjacent in A and in C), half the instructions per byte of the scalar kernel.
template <int NMAX, bool POW2>
__global__ void __launch_bounds__(256) einsum_skinny2_old_kernel(const EinsumDesc* __restrict__ gd,
                                                             const int64_t* __restrict__ leaf_off) {
  __shared__ __align__(16) EinsumDesc d;
  copy_desc_to_smem(&d, gd);
  extern __shared__ __align__(16) uint8_t dyn[];
  const int K = (int)d.K, N = (int)d.N;
  float2* Bs = reinterpret_cast<float2*>(dyn);                 // [K][N]
  int64_t* koff = reinterpret_cast<int64_t*>(dyn + sizeof(float2) * K * N);
  const float2* A = d.A + d.a_off;
  const float2* B = d.B + d.b_off + (d.b_leaf >= 0 ? leaf_off[d.b_leaf] : 0);
  for (int e = threadIdx.x; e < K * N; e += blockDim.x) {
    const int k = e / N, n = e % N;
    Bs[e] = B[decompose(n, d.nn, d.n_ext, d.n_sb) + decompose(k, d.nk, d.k_ext, d.k_sb)];
  }
  for (int k = threadIdx.x; k < K; k += blockDim.x) koff[k] = decompose(k, d.nk, d.k_ext, d.k_sa);
  __syncthreads();
  const int64_t V = d.V, Vh = V / 2, Mh = d.M / 2;
  const int lvh = __ffsll(Vh) - 1;
  float amax = 0.f;
  for (int64_t m = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; m < Mh;
       m += (int64_t)gridDim.x * blockDim.x) {
    const int64_t vi = (POW2 ? (m & (Vh - 1)) : (m % Vh)) * 2, o = POW2 ? (m >> lvh) : m / Vh;
    const float2* a_row = A + (POW2 ? decompose_sh(o, d.nm - 1, d.m_sh, d.m_sa)
                                    : decompose(o, d.nm - 1, d.m_ext, d.m_sa)) + vi;
    float r0[NMAX], i0[NMAX], r1[NMAX], i1[NMAX];
#pragma unroll
    for (int n = 0; n < NMAX; ++n) { r0[n] = 0.f; i0[n] = 0.f; r1[n] = 0.f; i1[n] = 0.f; }
    for (int k = 0; k < K; ++k) {
      const float4 q = *reinterpret_cast<const float4*>(a_row + koff[k]);
#pragma unroll
      for (int n = 0; n < NMAX; ++n) {
        if (n < N) {
          const float2 b = Bs[k * N + n];
          r0[n] = fmaf(q.x, b.x, r0[n]); r0[n] = fmaf(-q.y, b.y, r0[n]);
          i0[n] = fmaf(q.x, b.y, i0[n]); i0[n] = fmaf(q.y, b.x, i0[n]);
          r1[n] = fmaf(q.z, b.x, r1[n]); r1[n] = fmaf(-q.w, b.y, r1[n]);
          i1[n] = fmaf(q.z, b.y, i1[n]); i1[n] = fmaf(q.w, b.x, i1[n]);
        }
      }
    }
    const int64_t base = o * N * V + vi;
#pragma unroll
    for (int n = 0; n < NMAX; ++n) {
      if (n < N) {
        const int64_t idx = base + (int64_t)n * V;
        if (d.acc) {
          store_out_f(d, idx, r0[n], i0[n], amax);
          store_out_f(d, idx + 1, r1[n], i1[n], amax);
        } else {
          *reinterpret_cast<float4*>(d.C + idx) = make_float4(r0[n], i0[n], r1[n], i1[n]);
          amax = fmaxf(amax, fmaxf(fmaxf(fabsf(r0[n]), fabsf(i0[n])), fmaxf(fabsf(r1[n]), fabsf(i1[n]))));
        }
      }
    }
  }
  if (d.absmax_out) block_absmax(amax, d.absmax_out);
}

// ---------------------------------------------------------------- SIMT einsum, wide skinny
// Same layout contract as einsum_skinny_old_kernel (out [Mo][N][V]) for outer-product-
// like steps: K <= KMAX (the big operand's row lives in registers), N up to 4096
// (small operand staged in smem), outputs streamed n by n with lanes along v.
template <int KMAX>
__global__ void __launch_bounds__(256) einsum_wide_old_kernel(const EinsumDesc* __restrict__ gd,
                                                          const int64_t* __restrict__ leaf_off) {
  __shared__ __align__(16) EinsumDesc d;
  copy_desc_to_smem(&d, gd);
  extern __shared__ __align__(16) uint8_t dyn[];
  const int K = (int)d.K, N = (int)d.N;
  float2* Bs = reinterpret_cast<float2*>(dyn);                 // [N][K]
  const float2* A = d.A + d.a_off + (d.a_leaf >= 0 ? leaf_off[d.a_leaf] : 0);
  const float2* B = d.B + d.b_off + (d.b_leaf >= 0 ? leaf_off[d.b_leaf] : 0);
  for (int e = threadIdx.x; e < K * N; e += blockDim.x) {
    const int n = e / K, k = e % K;
    Bs[e] = B[decompose(n, d.nn, d.n_ext, d.n_sb) + decompose(k, d.nk, d.k_ext, d.k_sb)];
  }
  __syncthreads();
  const int64_t V = d.V;
  const bool vp2 = (V & (V - 1)) == 0;
  const int lv = __ffsll(V) - 1;
  const int64_t vstride = d.m_sa[d.nm - 1];
  float amax = 0.f;
  for (int64_t m = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; m < d.M;
       m += (int64_t)gridDim.x * blockDim.x) {
    const int64_t vi = vp2 ? (m & (V - 1)) : m % V, o = vp2 ? (m >> lv) : m / V;
    const float2* a_row = A + decompose(o, d.nm - 1, d.m_ext, d.m_sa) + vi * vstride;
    float2 a[KMAX];
#pragma unroll
    for (int k = 0; k < KMAX; ++k)
      a[k] = k < K ? a_row[decompose(k, d.nk, d.k_ext, d.k_sa)] : make_float2(0.f, 0.f);
    for (int n = 0; n < N; ++n) {
      float cr = 0.f, ci = 0.f;
#pragma unroll
      for (int k = 0; k < KMAX; ++k) {
        if (k < K) {
          const float2 b = Bs[n * K + k];
          cr = fmaf(a[k].x, b.x, cr);
          cr = fmaf(-a[k].y, b.y, cr);
          ci = fmaf(a[k].x, b.y, ci);
          ci = fmaf(a[k].y, b.x, ci);
        }
      }
      store_out(d, (o * N + n) * V + vi, cr, ci, amax);
    }
  }
  if (d.absmax_out) block_absmax(amax, d.absmax_out);
}

// ---------------------------------------------------------------- SIMT einsum, warp dot
// Batched merges with tiny per-batch outputs and a long K (e.g. the last merges of a
// sparse-state path: J = 65 536 batches of 4 x 16 outputs, K = 2048): one warp per
// output row (j, m) computes all N <= 32 outputs, lanes striding K (coalesced along
// the operands' unit-stride k), fp32 lane sums reduced across the warp in fp64.
constexpr int WD_NMAX = 32;
__global__ void __launch_bounds__(256) einsum_wdot_kernel(const EinsumDesc* __restrict__ gd,
                                                          const int64_t* __restrict__ leaf_off) {
  __shared__ __align__(16) EinsumDesc d;
  copy_desc_to_smem(&d, gd);
  __shared__ int64_t boff[8][WD_NMAX];
  const float2* A = d.A + d.a_off + (d.a_leaf >= 0 ? leaf_off[d.a_leaf] : 0);
  const float2* B = d.B + d.b_off + (d.b_leaf >= 0 ? leaf_off[d.b_leaf] : 0);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int N = (int)d.N;
  const int64_t rows = d.J * d.M;
  float amax = 0.f;
  for (int64_t row = blockIdx.x * 8 + warp; row < rows; row += (int64_t)gridDim.x * 8) {
    const int64_t m = row % d.M, j = row / d.M;
    const int64_t ao = (d.ia ? (int64_t)d.ia[j] : 0) * d.a_gs + decompose(m, d.nm, d.m_ext, d.m_sa);
    if (lane < N)
      boff[warp][lane] = (d.ib ? (int64_t)d.ib[j] : 0) * d.b_gs + decompose(lane, d.nn, d.n_ext, d.n_sb);
    __syncwarp();
    float cr[WD_NMAX], ci[WD_NMAX];
#pragma unroll
    for (int n = 0; n < WD_NMAX; ++n) { cr[n] = 0.f; ci[n] = 0.f; }
    for (int64_t k = lane; k < d.K; k += 32) {
      int64_t ka = 0, kb = 0, t = k;
      if (d.pow2) {                    // shift tables: no 64-bit division per k
        for (int i = d.nk - 1; i >= 0; --i) {
          const int sh = d.k_sh[i];
          const int64_t dg = t & ((int64_t(1) << sh) - 1);
          t >>= sh;
          ka += dg * d.k_sa[i];
          kb += dg * d.k_sb[i];
        }
      } else {
        for (int i = d.nk - 1; i >= 0; --i) {
          const int64_t dg = t % d.k_ext[i];
          t /= d.k_ext[i];
          ka += dg * d.k_sa[i];
          kb += dg * d.k_sb[i];
        }
      }
      const float2 a = __ldg(A + ao + ka);
#pragma unroll
      for (int n = 0; n < WD_NMAX; ++n) {
        if (n < N) {
          const float2 b = __ldg(B + boff[warp][n] + kb);
          cr[n] = fmaf(a.x, b.x, fmaf(-a.y, b.y, cr[n]));
          ci[n] = fmaf(a.x, b.y, fmaf(a.y, b.x, ci[n]));
        }
      }
    }
    double outr = 0.0, outi = 0.0;
#pragma unroll
    for (int n = 0; n < WD_NMAX; ++n) {
      if (n < N) {
        double r = cr[n], i = ci[n];
        for (int o = 16; o > 0; o >>= 1) {
          r += __shfl_xor_sync(0xffffffffu, r, o);
          i += __shfl_xor_sync(0xffffffffu, i, o);
        }
        if (lane == n) { outr = r; outi = i; }
      }
    }
    if (lane < N) store_out(d, row * N + lane, outr, outi, amax);
    __syncwarp();
  }
  if (d.absmax_out) block_absmax(amax, d.absmax_out);
}

// Variant for batched merges whose per-batch output is tiny (M <= 4 rows, N <= 32; e.g.
// the final merge of a sparse-state path: J = 65 536 batches of 4 x 16 outputs, K = 2048):
// a warp computes all M rows x NN = 8 columns of one batch j (ceil(N/8) warps per batch),
// so each k of the B slab is read once per batch instead of once per output row and each
// A row is reused for 8 columns; lanes stride K, two k per lane per iteration with all
// loads issued before the FMAs; fp32 lane sums, fp64 warp reduction.
template <int MM, int NN>
__global__ void __launch_bounds__(128) einsum_wdotj_kernel(const EinsumDesc* __restrict__ gd,
                                                           const int64_t* __restrict__ leaf_off) {
  static_assert(MM * NN <= 32, "at most 32 outputs per warp (1 per lane)");
  __shared__ __align__(16) EinsumDesc d;
  copy_desc_to_smem(&d, gd);
  const float2* A = d.A + d.a_off + (d.a_leaf >= 0 ? leaf_off[d.a_leaf] : 0);
  const float2* B = d.B + d.b_off + (d.b_leaf >= 0 ? leaf_off[d.b_leaf] : 0);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int M = (int)d.M, N = (int)d.N;
  const int NH = (N + NN - 1) / NN;     // warps per batch
  float amax = 0.f;
  __shared__ int64_t am[MM], bn[32];    // row offsets (same for every batch)
  if (threadIdx.x < MM) am[threadIdx.x] = threadIdx.x < M ? decompose(threadIdx.x, d.nm, d.m_ext, d.m_sa) : 0;
  if (threadIdx.x < 32) bn[threadIdx.x] = threadIdx.x < N ? decompose(threadIdx.x, d.nn, d.n_ext, d.n_sb) : 0;
  __syncthreads();
  auto koffs = [&](int64_t k, int64_t& ka, int64_t& kb) {
    int64_t t = k;
    ka = 0;
    kb = 0;
    for (int i = d.nk - 1; i >= 0; --i) {
      const int sh = d.k_sh[i];
      const int64_t dg = d.pow2 ? (t & ((int64_t(1) << sh) - 1)) : t % d.k_ext[i];
      t = d.pow2 ? (t >> sh) : t / d.k_ext[i];
      ka += dg * d.k_sa[i];
      kb += dg * d.k_sb[i];
    }
  };
  const int64_t units = d.J * NH;
  for (int64_t u_ = blockIdx.x * 4 + warp; u_ < units; u_ += (int64_t)gridDim.x * 4) {
    const int64_t j = u_ / NH;
    const int n0 = (int)(u_ % NH) * NN;
    const int64_t ao = (d.ia ? (int64_t)d.ia[j] : 0) * d.a_gs;
    const int64_t bo = (d.ib ? (int64_t)d.ib[j] : 0) * d.b_gs;
    float cr[MM][NN], ci[MM][NN];
#pragma unroll
    for (int m = 0; m < MM; ++m)
#pragma unroll
      for (int n = 0; n < NN; ++n) { cr[m][n] = 0.f; ci[m][n] = 0.f; }
    for (int64_t k0 = lane; k0 < d.K; k0 += 64) {
      const bool two = k0 + 32 < d.K;
      int64_t ka0, kb0, ka1 = 0, kb1 = 0;
      koffs(k0, ka0, kb0);
      if (two) koffs(k0 + 32, ka1, kb1);
      float2 a[2][MM], b[2][NN];
#pragma unroll
      for (int u = 0; u < 2; ++u) {
        const bool ok = u == 0 || two;
        const int64_t ka = u ? ka1 : ka0, kb = u ? kb1 : kb0;
#pragma unroll
        for (int m = 0; m < MM; ++m)
          a[u][m] = (ok && m < M) ? __ldg(A + ao + am[m] + ka) : make_float2(0.f, 0.f);
#pragma unroll
        for (int n = 0; n < NN; ++n)
          b[u][n] = (ok && n0 + n < N) ? __ldg(B + bo + bn[n0 + n] + kb) : make_float2(0.f, 0.f);
      }
#pragma unroll
      for (int u = 0; u < 2; ++u)
#pragma unroll
        for (int n = 0; n < NN; ++n)
#pragma unroll
          for (int m = 0; m < MM; ++m) {
            cr[m][n] = fmaf(a[u][m].x, b[u][n].x, fmaf(-a[u][m].y, b[u][n].y, cr[m][n]));
            ci[m][n] = fmaf(a[u][m].x, b[u][n].y, fmaf(a[u][m].y, b[u][n].x, ci[m][n]));
          }
    }
    // output (m, n0 + n) is reduced onto lane m * NN + n
    double orr = 0.0, oi = 0.0;
#pragma unroll
    for (int m = 0; m < MM; ++m)
#pragma unroll
      for (int n = 0; n < NN; ++n) {
        if (m < M && n0 + n < N) {
          double r = cr[m][n], i = ci[m][n];
          for (int o = 16; o > 0; o >>= 1) {
            r += __shfl_xor_sync(0xffffffffu, r, o);
            i += __shfl_xor_sync(0xffffffffu, i, o);
          }
          if (lane == m * NN + n) { orr = r; oi = i; }
        }
      }
    const int m = lane / NN, n = n0 + lane % NN;
    if (m < M && n < N && lane < MM * NN) store_out(d, (j * M + m) * N + n, orr, oi, amax);
  }
  if (d.absmax_out) block_absmax(amax, d.absmax_out);
}

// Slab-staged variant of the warp dot (mode 4 variant 3, EinsumDesc.wd_*): the final
// merges of the sparse boundary share each B slab between many batches while B's k order
// is scattered (lanes over k would read 8 B per 32-B sector, 4x the bytes, once per
// batch).  A block takes one contiguous part of one B slab — all k of N >> wd_t columns —
// reads it once with coalesced loads into shared memory in [n_local][k] order (scatter
// through two bit tables), then its warps run every batch of that slab: lanes over k, A
// rows from global memory (per-k offsets from a smem table), B from smem without bank
// conflicts, fp32 lane sums and an fp64 warp reduction per output (as einsum_wdotj).
constexpr int WDS_WARPS = 16;
constexpr int WDS_MAX_PART = 16384;   // elements of a staged part (128 KiB)
__global__ void __launch_bounds__(32 * WDS_WARPS) einsum_wdots_kernel(const EinsumDesc* __restrict__ gd,
                                                                     const int64_t* __restrict__ leaf_off) {
  constexpr int MM = 4, NN = 8;
  __shared__ __align__(16) EinsumDesc d;
  __shared__ int32_t tlo[128], thi[128];
  __shared__ int64_t am[MM];
  extern __shared__ __align__(16) uint8_t wds_smem[];
  copy_desc_to_smem(&d, gd);
  float2* sB = reinterpret_cast<float2*>(wds_smem);                 // [np][K]
  int32_t* ka = reinterpret_cast<int32_t*>(sB + ((int64_t)1 << d.wd_lb));   // [K]
  const float2* A = d.A + d.a_off + (d.a_leaf >= 0 ? leaf_off[d.a_leaf] : 0);
  const float2* B = d.B + d.b_off + (d.b_leaf >= 0 ? leaf_off[d.b_leaf] : 0);
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int lb = d.wd_lb, llo = lb < 7 ? lb : 7, lhi = lb - llo;
  const int M = (int)d.M, N = (int)d.N, K = (int)d.K;
  for (int x = tid; x < (1 << llo); x += blockDim.x) {
    int v = 0;
    for (int b = 0; b < llo; ++b) if ((x >> b) & 1) v += d.wd_contrib[b];
    tlo[x] = v;
  }
  for (int x = tid; x < (1 << lhi); x += blockDim.x) {
    int v = 0;
    for (int b = 0; b < lhi; ++b) if ((x >> b) & 1) v += d.wd_contrib[llo + b];
    thi[x] = v;
  }
  if (tid < MM) am[tid] = tid < M ? decompose(tid, d.nm, d.m_ext, d.m_sa) : 0;
  for (int k = tid; k < K; k += blockDim.x) ka[k] = (int32_t)decompose_sh(k, d.nk, d.k_sh, d.k_sa);
  __syncthreads();
  const int T = 1 << d.wd_t, P = 1 << lb, NP = d.wd_np;
  const int NG = (NP + NN - 1) / NN;
  const int lomask = (1 << llo) - 1;
  float amax = 0.f;
  for (int64_t u = blockIdx.x; u < d.wd_nslabs * T; u += gridDim.x) {
    const int64_t slab = u / T;
    const int part = (int)(u % T);
    const int j0 = d.wd_start[slab], j1 = d.wd_start[slab + 1];
    if (j0 == j1) continue;                      // uniform over the block
    const float2* src = B + slab * d.b_gs + (int64_t)part * P;
    // every element of the part in flight at once (8-B LDGSTS into its scattered slot)
    for (int o = tid; o < P; o += blockDim.x) cp_async8(sB + tlo[o & lomask] + thi[o >> llo], src + o);
    cp_async_wait_all();
    __syncthreads();
    for (int task = warp; task < (j1 - j0) * NG; task += WDS_WARPS) {
      const int64_t j = d.wd_list[j0 + task / NG];
      const int nb0 = (task % NG) * NN;
      const float2* Aj = A + (d.ia ? (int64_t)d.ia[j] : 0) * d.a_gs;
      float cr[MM][NN], ci[MM][NN];
#pragma unroll
      for (int m = 0; m < MM; ++m)
#pragma unroll
        for (int n = 0; n < NN; ++n) { cr[m][n] = 0.f; ci[m][n] = 0.f; }
      for (int k0 = lane; k0 < K; k0 += 64) {
        const bool two = k0 + 32 < K;
        float2 a[2][MM], b[2][NN];
#pragma unroll
        for (int uu = 0; uu < 2; ++uu) {
          const bool ok = uu == 0 || two;
          const int k = k0 + 32 * uu;
          const int32_t kaa = ok ? ka[k] : 0;
#pragma unroll
          for (int m = 0; m < MM; ++m)
            a[uu][m] = (ok && m < M) ? __ldg(Aj + am[m] + kaa) : make_float2(0.f, 0.f);
#pragma unroll
          for (int n = 0; n < NN; ++n)
            b[uu][n] = (ok && nb0 + n < NP) ? sB[(nb0 + n) * K + k] : make_float2(0.f, 0.f);
        }
#pragma unroll
        for (int uu = 0; uu < 2; ++uu)
#pragma unroll
          for (int n = 0; n < NN; ++n)
#pragma unroll
            for (int m = 0; m < MM; ++m) {
              cr[m][n] = fmaf(a[uu][m].x, b[uu][n].x, fmaf(-a[uu][m].y, b[uu][n].y, cr[m][n]));
              ci[m][n] = fmaf(a[uu][m].x, b[uu][n].y, fmaf(a[uu][m].y, b[uu][n].x, ci[m][n]));
            }
      }
      double orr = 0.0, oi = 0.0;
#pragma unroll
      for (int m = 0; m < MM; ++m)
#pragma unroll
        for (int n = 0; n < NN; ++n) {
          if (m < M && nb0 + n < NP) {
            double r = cr[m][n], i = ci[m][n];
            for (int o = 16; o > 0; o >>= 1) {
              r += __shfl_xor_sync(0xffffffffu, r, o);
              i += __shfl_xor_sync(0xffffffffu, i, o);
            }
            if (lane == m * NN + n) { orr = r; oi = i; }
          }
        }
      const int m = lane / NN, nl = nb0 + lane % NN;
      if (m < M && nl < NP) {
        const int64_t n = (int64_t)d.wd_ptop[part] + d.wd_nloc[nl];
        store_out(d, (j * M + m) * N + n, orr, oi, amax);
      }
    }
    __syncthreads();
  }
  if (d.absmax_out) block_absmax(amax, d.absmax_out);
}

// ---------------------------------------------------------------- fused skinny chain
// tn::ChainDesc (tn_internal.h).  A block takes a tile of 32 carry positions
// (lane = carry position: unit stride in the chain's input T0 and output TL), loads T0's
// touched elements into smem W0[e][lane], runs the steps W_{i-1} -> W_i in smem (warp task =
// one o-position p and up to 8 outputs n: the K inputs of p in registers, Y rows broadcast
// from smem, the same fp32 k-ordered sums as einsum_skinny_kernel) and stores W_L.
constexpr int CH_THREADS = 256;

// one chain step W_{i-1} -> W_i for K inputs and NG outputs per warp task (templated so the
// k loop and the NG output chains unroll: NG independent FMA chains per task)
template <int K, int NG>
__device__ __forceinline__ void chain_step(const float2* __restrict__ W, float2* __restrict__ O,
                                           const float2* __restrict__ Ys, const int32_t* in_p,
                                           const int32_t* out_p, const int32_t* in_k, const int32_t* out_n,
                                           int P, int N, int warp, int lane) {
  const int ngr = N / NG;
  for (int task = warp; task < P * ngr; task += CH_THREADS / 32) {
    const int p = task / ngr, nb = (task - p * ngr) * NG;
    float2 x[K];
    const int ip = in_p[p];
#pragma unroll
    for (int k = 0; k < K; ++k) x[k] = W[(ip + in_k[k]) * 32 + lane];
    const int op = out_p[p];
    float ar[NG], ai[NG];
#pragma unroll
    for (int j = 0; j < NG; ++j) { ar[j] = 0.f; ai[j] = 0.f; }
#pragma unroll
    for (int k = 0; k < K; k += 2) {
#pragma unroll
      for (int j = 0; j < NG; ++j) {
        const float2* y = Ys + (nb + j) * K + k;
        float2 b0, b1 = make_float2(0.f, 0.f);
        if constexpr (K >= 2) {
          const float4 q = *reinterpret_cast<const float4*>(y);   // broadcast 16-B pair
          b0 = make_float2(q.x, q.y);
          b1 = make_float2(q.z, q.w);
        } else {
          b0 = y[0];
        }
        ar[j] = fmaf(x[k].x, b0.x, fmaf(-x[k].y, b0.y, ar[j]));
        ai[j] = fmaf(x[k].x, b0.y, fmaf(x[k].y, b0.x, ai[j]));
        if constexpr (K >= 2) {
          ar[j] = fmaf(x[k + 1].x, b1.x, fmaf(-x[k + 1].y, b1.y, ar[j]));
          ai[j] = fmaf(x[k + 1].x, b1.y, fmaf(x[k + 1].y, b1.x, ai[j]));
        }
      }
    }
#pragma unroll
    for (int j = 0; j < NG; ++j) O[(op + out_n[nb + j]) * 32 + lane] = make_float2(ar[j], ai[j]);
  }
}

template <int K>
__device__ __forceinline__ void chain_step_k(const float2* W, float2* O, const float2* Ys, const int32_t* in_p,
                                             const int32_t* out_p, const int32_t* in_k, const int32_t* out_n,
                                             int P, int N, int warp, int lane) {
  if (N >= 8) chain_step<K, 8>(W, O, Ys, in_p, out_p, in_k, out_n, P, N, warp, lane);
  else if (N == 4) chain_step<K, 4>(W, O, Ys, in_p, out_p, in_k, out_n, P, N, warp, lane);
  else if (N == 2) chain_step<K, 2>(W, O, Ys, in_p, out_p, in_k, out_n, P, N, warp, lane);
  else chain_step<K, 1>(W, O, Ys, in_p, out_p, in_k, out_n, P, N, warp, lane);
}

__global__ void __launch_bounds__(CH_THREADS) einsum_chain_kernel(const ChainDesc* __restrict__ gd,
                                                                 const int64_t* __restrict__ leaf_off) {
  __shared__ __align__(16) ChainDesc d;
  copy_desc_to_smem(&d, gd);
  extern __shared__ __align__(16) uint8_t ch_smem[];
  float2* bufA = reinterpret_cast<float2*>(ch_smem);
  float2* bufB = bufA + 32 * (size_t)d.buf_a;
  float2* Ys = bufB + 32 * (size_t)d.buf_b;
  int ysz = 0;
  for (int i = 0; i < d.L; ++i) ysz += (d.st[i].N * d.st[i].K + 1) & ~1;
  const size_t ysz_al = (size_t)ysz;
  int32_t* tab = reinterpret_cast<int32_t*>(Ys + ysz + 2 * 32 * ((size_t)1 << d.a0));
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  for (int i = tid; i < d.n_tab; i += CH_THREADS) tab[i] = d.tab[i];
  __syncthreads();
  {
    int yo = 0;
    for (int i = 0; i < d.L; ++i) {
      const ChainStep& st = d.st[i];
      const float2* Y = st.Y + st.y_off + (st.y_leaf >= 0 ? leaf_off[st.y_leaf] : 0);
      const int32_t* yoff = tab + st.tab + 2 * st.P + st.K + st.N;
      for (int e = tid; e < st.N * st.K; e += CH_THREADS) Ys[yo + e] = Y[yoff[e]];
      yo += (st.N * st.K + 1) & ~1;      // 16-B aligned regions (paired Y loads)
    }
  }
  const float2* src = d.src + d.src_off + (d.src_leaf >= 0 ? leaf_off[d.src_leaf] : 0);
  const TileBits tb = tile_bits_load(d.ct_src, d.ct_dst, d.nct, lane);
  int64_t ls = 0, ld = 0;                      // this lane's carry offsets in T0 / TL
#pragma unroll
  for (int b = 0; b < 5; ++b)
    if ((lane >> b) & 1) { ls += d.lw_src[b]; ld += d.lw_dst[b]; }
  const int n0 = 1 << d.a0, nL = 1 << d.aL;
  const int32_t* t0off = tab;
  const int32_t* tLoff = tab + n0;
  float amax = 0.f;
  // the input tile is double-buffered: tile t + grid is loaded (8-B LDGSTS, all in flight)
  // while tile t runs its steps; step 0 reads W0 straight from the load buffer
  float2* w0buf[2] = {Ys + ysz_al, Ys + ysz_al + 32 * (size_t)n0};
  auto issue = [&](int64_t t, float2* dst) {
    int64_t cs_, cd_;
    tile_bits_sum(tb, (uint64_t)t, lane, d.nct, d.ct_src, d.ct_dst, cs_, cd_);
    const float2* sp = src + cs_ + ls;
    for (int e = warp; e < n0; e += CH_THREADS / 32) cp_async8(dst + e * 32 + lane, sp + t0off[e]);
  };
  __syncthreads();                   // Y staged
  if (blockIdx.x < d.n_tiles) issue(blockIdx.x, w0buf[0]);
  asm volatile("cp.async.commit_group;" ::: "memory");
  int cur = 0;
  for (int64_t t = blockIdx.x; t < d.n_tiles; t += gridDim.x) {
    int64_t cs, cdst;
    tile_bits_sum(tb, (uint64_t)t, lane, d.nct, d.ct_src, d.ct_dst, cs, cdst);
    if (t + gridDim.x < d.n_tiles) issue(t + gridDim.x, w0buf[cur ^ 1]);
    asm volatile("cp.async.commit_group;\ncp.async.wait_group 1;" ::: "memory");
    __syncthreads();                 // tile t's input complete for every thread
    int yo = 0;
    for (int i = 0; i < d.L; ++i) {
      const ChainStep& st = d.st[i];
      const float2* W = i == 0 ? w0buf[cur] : (st.in_buf ? bufB : bufA);
      float2* O = st.in_buf ? bufA : bufB;
      const int32_t* in_p = tab + st.tab;
      const int32_t* out_p = in_p + st.P;
      const int32_t* in_k = out_p + st.P;
      const int32_t* out_n = in_k + st.K;
      const int K = st.K, N = st.N;
      const float2* Yst = Ys + yo;
      switch (K) {   // the planner admits K = 1, 2, 4, 8, 16 (powers of two <= 16)
        case 1: chain_step_k<1>(W, O, Yst, in_p, out_p, in_k, out_n, st.P, N, warp, lane); break;
        case 2: chain_step_k<2>(W, O, Yst, in_p, out_p, in_k, out_n, st.P, N, warp, lane); break;
        case 4: chain_step_k<4>(W, O, Yst, in_p, out_p, in_k, out_n, st.P, N, warp, lane); break;
        case 8: chain_step_k<8>(W, O, Yst, in_p, out_p, in_k, out_n, st.P, N, warp, lane); break;
        default: chain_step_k<16>(W, O, Yst, in_p, out_p, in_k, out_n, st.P, N, warp, lane); break;
      }
      yo += (N * K + 1) & ~1;
      __syncthreads();
    }
    const float2* WL = (d.L & 1) ? bufB : bufA;
    float2* dp = d.dst + cdst + ld;
    for (int e = warp; e < nL; e += CH_THREADS / 32) {
      const float2 v = WL[e * 32 + lane];
      dp[tLoff[e]] = v;
      amax = fmaxf(amax, fmaxf(fabsf(v.x), fabsf(v.y)));
    }
    cur ^= 1;
    __syncthreads();                 // W_L read before the next tile's steps overwrite it
  }
  asm volatile("cp.async.wait_group 0;" ::: "memory");
  if (d.absmax_out) block_absmax(amax, d.absmax_out);
}

// Variant for operands whose unit stride is the output dim n: lane = (k group, n), so
// each load instruction reads NL consecutive n of 32/NL k values; one fp32 partial per
// lane, reduced across the k groups in fp64.
__global__ void __launch_bounds__(256) einsum_wdot2_kernel(const EinsumDesc* __restrict__ gd,
                                                           const int64_t* __restrict__ leaf_off) {
  __shared__ __align__(16) EinsumDesc d;
  copy_desc_to_smem(&d, gd);
  const float2* A = d.A + d.a_off + (d.a_leaf >= 0 ? leaf_off[d.a_leaf] : 0);
  const float2* B = d.B + d.b_off + (d.b_leaf >= 0 ? leaf_off[d.b_leaf] : 0);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int N = (int)d.N;
  int lnl = 0;
  while ((1 << lnl) < N) ++lnl;
  const int NL = 1 << lnl, G = 32 / NL;            // N <= 32: NL lanes per k group
  const int n = lane & (NL - 1), kg = lane >> lnl;
  const int64_t rows = d.J * d.M;
  float amax = 0.f;
  for (int64_t row = blockIdx.x * 8 + warp; row < rows; row += (int64_t)gridDim.x * 8) {
    const int64_t m = row % d.M, j = row / d.M;
    const int64_t ao = (d.ia ? (int64_t)d.ia[j] : 0) * d.a_gs + decompose(m, d.nm, d.m_ext, d.m_sa);
    const int64_t bo = (d.ib ? (int64_t)d.ib[j] : 0) * d.b_gs + (n < N ? decompose(n, d.nn, d.n_ext, d.n_sb) : 0);
    float cr = 0.f, ci = 0.f;
    for (int64_t k = kg; k < d.K; k += G) {
      int64_t ka = 0, kb = 0, t = k;
      for (int i = d.nk - 1; i >= 0; --i) {
        const int sh = d.k_sh[i];
        const int64_t dg = d.pow2 ? (t & ((int64_t(1) << sh) - 1)) : t % d.k_ext[i];
        t = d.pow2 ? (t >> sh) : t / d.k_ext[i];
        ka += dg * d.k_sa[i];
        kb += dg * d.k_sb[i];
      }
      if (n < N) {
        const float2 a = __ldg(A + ao + ka), b = __ldg(B + bo + kb);
        cr = fmaf(a.x, b.x, fmaf(-a.y, b.y, cr));
        ci = fmaf(a.x, b.y, fmaf(a.y, b.x, ci));
      }
    }
    double r = cr, i = ci;
    for (int o = 16; o >= NL; o >>= 1) {
      r += __shfl_xor_sync(0xffffffffu, r, o);
      i += __shfl_xor_sync(0xffffffffu, i, o);
    }
    if (kg == 0 && n < N) store_out(d, row * N + n, r, i, amax);
  }
  if (d.absmax_out) block_absmax(amax, d.absmax_out);
}

// ---------------------------------------------------------------- SIMT einsum, split-K dot
// Few outputs, long K (e.g. the last step of a closed network, a 2^30-long dot):
// block b takes output p = b / nchunk and a kchunk range of k; fp64 block
// reduction, fp64 atomicAdd into d.partial (zeroed before the launch).
__global__ void __launch_bounds__(256) einsum_dot_kernel(const EinsumDesc* __restrict__ gd,
                                                         const int64_t* __restrict__ leaf_off,
                                                         int64_t nchunk) {
  __shared__ __align__(16) EinsumDesc d;
  copy_desc_to_smem(&d, gd);
  __shared__ double red[2][8];
  const float2* A = d.A + d.a_off + (d.a_leaf >= 0 ? leaf_off[d.a_leaf] : 0);
  const float2* B = d.B + d.b_off + (d.b_leaf >= 0 ? leaf_off[d.b_leaf] : 0);
  const int64_t P = d.J * d.M * d.N;
  for (int64_t blk = blockIdx.x; blk < P * nchunk; blk += gridDim.x) {
    const int64_t p = blk / nchunk, c = blk % nchunk;
    const int64_t n = p % d.N, t1 = p / d.N, m = t1 % d.M, j = t1 / d.M;
    const int64_t ao = (d.ia ? (int64_t)d.ia[j] : 0) * d.a_gs + decompose(m, d.nm, d.m_ext, d.m_sa);
    const int64_t bo = (d.ib ? (int64_t)d.ib[j] : 0) * d.b_gs + decompose(n, d.nn, d.n_ext, d.n_sb);
    const int64_t k0 = c * d.kchunk, k1 = min(d.K, k0 + d.kchunk);
    double cr = 0.0, ci = 0.0;
    for (int64_t k = k0 + threadIdx.x; k < k1; k += blockDim.x) {
      const float2 a = A[ao + decompose(k, d.nk, d.k_ext, d.k_sa)];
      const float2 b = B[bo + decompose(k, d.nk, d.k_ext, d.k_sb)];
      cr = fma((double)a.x, (double)b.x, cr);
      cr = fma(-(double)a.y, (double)b.y, cr);
      ci = fma((double)a.x, (double)b.y, ci);
      ci = fma((double)a.y, (double)b.x, ci);
    }
    for (int o = 16; o > 0; o >>= 1) {
      cr += __shfl_xor_sync(0xffffffffu, cr, o);
      ci += __shfl_xor_sync(0xffffffffu, ci, o);
    }
    const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
    __syncthreads();
    if (l == 0) { red[0][w] = cr; red[1][w] = ci; }
    __syncthreads();
    if (threadIdx.x == 0) {
      double sr = 0.0, si = 0.0;
      for (int i = 0; i < (int)(blockDim.x >> 5); ++i) { sr += red[0][i]; si += red[1][i]; }
      atomicAdd(&d.partial[2 * p], sr);
      atomicAdd(&d.partial[2 * p + 1], si);
    }
  }
}

__global__ void einsum_dot_finalize(const EinsumDesc* __restrict__ gd) {
  __shared__ __align__(16) EinsumDesc d;
  copy_desc_to_smem(&d, gd);
  const int64_t P = d.J * d.M * d.N;
  float amax = 0.f;
  for (int64_t p = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; p < P;
       p += (int64_t)gridDim.x * blockDim.x)
    store_out(d, p, d.partial[2 * p], d.partial[2 * p + 1], amax);
  if (d.absmax_out) block_absmax(amax, d.absmax_out);
}

// flag (nullable): the fused-plane overflow flag; when set the sum may hold saturated
// fp16 operands, so NaN is written instead (tn_sum_slices stays asynchronous)
__global__ void gather_out_kernel(const double2* __restrict__ acc, const int32_t* __restrict__ pos,
                                  double2* __restrict__ out, int64_t n, const int* __restrict__ flag) {
  const bool bad = flag && *flag;
  const double nan = __longlong_as_double(0x7ff8000000000000LL);
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    out[i] = bad ? make_double2(nan, nan) : acc[pos[i]];
}

int grid_for(int64_t total, int threads) {
  int64_t b = (total + threads - 1) / threads;
  const int64_t cap = 148 * 16;
  if (b > cap) b = cap;
  if (b < 1) b = 1;
  return (int)b;
}

}  // namespace

cudaError_t launch_prep_fmt(const float2* src, void* dst, int64_t rows, int64_t K, int64_t Kpad,
                            int planes, int format, const unsigned* absmax, int* scale_out,
                            cudaStream_t s) {
  const int64_t n = rows * Kpad;
  const int64_t blocks = std::min<int64_t>((n + 255) / 256, 148 * 16);
  prep_fmt_kernel<<<(unsigned)std::max<int64_t>(blocks, 1), 256, 0, s>>>(src, dst, rows, K, Kpad, planes,
                                                                       format, absmax, scale_out);
  return cudaGetLastError();
}

cudaError_t launch_set_counter(int64_t* counter, int64_t value, cudaStream_t s) {
  set_counter_kernel<<<1, 1, 0, s>>>(counter, value);
  return cudaGetLastError();
}

cudaError_t launch_slice_select(const SliceDesc* d_desc, cudaStream_t s) {
  slice_select_kernel<<<1, 256, 0, s>>>(d_desc);
  return cudaGetLastError();
}

template <int PLANES, int KT, int NB>
cudaError_t launch_gate_mma_t(const PrepDesc* d_desc, int g, const int64_t* leaf_off, cudaStream_t s) {
  const void* k = reinterpret_cast<const void*>(prep_gate_mma_kernel<PLANES, KT, NB>);
  constexpr size_t smem = GP_SMEM + GP_BUF * 8;     // + the separate output tile
  if (cudaError_t e = set_smem_attr(k, (int)smem)) return e;
  prep_gate_mma_kernel<PLANES, KT, NB><<<g, 256, smem, s>>>(d_desc, leaf_off);
  return cudaGetLastError();
}

template <int PLANES, int KT>
cudaError_t launch_gate_t(const PrepDesc* d_desc, int g, const int64_t* leaf_off, cudaStream_t s) {
  if (cudaError_t e = set_smem_attr(reinterpret_cast<const void*>(prep_gate_kernel<PLANES, KT>), (int)GP_SMEM))
    return e;
  prep_gate_kernel<PLANES, KT><<<g, 256, GP_SMEM, s>>>(d_desc, leaf_off);
  return cudaGetLastError();
}

cudaError_t launch_gate(const PrepDesc* d_desc, int planes, int k, int g, const int64_t* leaf_off,
                        cudaStream_t s) {
#define TN_GATE(P)                                                        \
  switch (k) {                                                            \
    case 1: return launch_gate_t<P, 1>(d_desc, g, leaf_off, s);           \
    case 2: return launch_gate_t<P, 2>(d_desc, g, leaf_off, s);           \
    case 4: return launch_gate_t<P, 4>(d_desc, g, leaf_off, s);           \
    case 8: return launch_gate_t<P, 8>(d_desc, g, leaf_off, s);           \
    case 16: return launch_gate_t<P, 16>(d_desc, g, leaf_off, s);         \
    default: return cudaErrorInvalidValue;                                \
  }
  if (planes == 4) { TN_GATE(4) } else { TN_GATE(2) }
#undef TN_GATE
}

cudaError_t launch_prep(const PrepDesc* d_desc, int64_t total, int planes, int kind, int tile_T,
                        const int64_t* leaf_off, cudaStream_t s, int gate_k, int gate_n) {
  const int th = 256;
  if (kind == 5) {   // gate-folded prep (K = 1, 2, 4, 8 or 16, carried in the descriptor)
    const int64_t tiles = total / std::max(tile_T, 1);
    const int bps = g_knobs.gate_bps;
    const int g = (int)std::min<int64_t>(std::max<int64_t>(tiles, 1), 148 * bps);
    // TN_GATE_MMA=1, K >= 4 and N <= 32: warp-level tensor-core MMAs (off by default: on
    // C4 it ran 33 ms where the FFMA kernel runs 24 ms)
    if (g_knobs.gate_mma && gate_k >= 4 && gate_n >= 1 && gate_n <= 32) {
      const int gm = (int)std::min<int64_t>(std::max<int64_t>(tiles, 1), 148 * 2);
#define TN_GMMA(P, KT)                                                                       \
  (gate_n <= 8 ? launch_gate_mma_t<P, KT, 1>(d_desc, gm, leaf_off, s)                        \
               : gate_n <= 16 ? launch_gate_mma_t<P, KT, 2>(d_desc, gm, leaf_off, s)         \
                              : launch_gate_mma_t<P, KT, 4>(d_desc, gm, leaf_off, s))
      if (planes == 4) {
        if (gate_k == 4) return TN_GMMA(4, 4);
        if (gate_k == 8) return TN_GMMA(4, 8);
        if (gate_k == 16) return TN_GMMA(4, 16);
      } else {
        if (gate_k == 4) return TN_GMMA(2, 4);
        if (gate_k == 8) return TN_GMMA(2, 8);
        if (gate_k == 16) return TN_GMMA(2, 16);
      }
#undef TN_GMMA
    }
    return launch_gate(d_desc, planes, gate_k, g, leaf_off, s);
  }
  if (kind == 4) {   // bit-permutation transposer, tiles of tile_T <= 4096 elements
    if (cudaError_t e = set_smem_attr(reinterpret_cast<const void*>(planes == 4 ? prep_bp_kernel<4> : prep_bp_kernel<2>),
                                      (int)BP_SMEM))
      return e;
    const int64_t tiles = total / std::max(tile_T, 1);
    const int g = (int)std::min<int64_t>(std::max<int64_t>(tiles, 1), 148 * 4);
    if (planes == 4)
      prep_bp_kernel<4><<<g, th, BP_SMEM, s>>>(d_desc, leaf_off);
    else
      prep_bp_kernel<2><<<g, th, BP_SMEM, s>>>(d_desc, leaf_off);
    return cudaGetLastError();
  }
  if (kind == 2) {   // general transposer, tiles of T <= 4096 elements
    if (cudaError_t e = set_smem_attr(reinterpret_cast<const void*>(planes == 4 ? prep_gt_kernel<4> : prep_gt_kernel<2>),
                                      120 * 1024))
      return e;
    const size_t smem = (size_t)tile_T * (8 + 8 + 8 + 4);
    int64_t tiles = total / std::max(tile_T, 1);
    const int g = (int)std::min<int64_t>(std::max<int64_t>(tiles, 1), 148 * 6);
    if (planes == 4)
      prep_gt_kernel<4><<<g, th, smem, s>>>(d_desc, leaf_off);
    else
      prep_gt_kernel<2><<<g, th, smem, s>>>(d_desc, leaf_off);
    return cudaGetLastError();
  }
  if (kind == 1 || kind == 3) {   // k-walking source / gathered rows: 8 elements per thread
    const int g = grid_for(total / 8, th);
    if (planes == 4)
      prep_direct_kernel<4><<<g, th, 0, s>>>(d_desc, leaf_off);
    else
      prep_direct_kernel<2><<<g, th, 0, s>>>(d_desc, leaf_off);
    return cudaGetLastError();
  }
  if (planes == 4)
    prep_kernel<4><<<grid_for(total, th), th, 0, s>>>(d_desc, leaf_off, total);
  else
    prep_kernel<2><<<grid_for(total, th), th, 0, s>>>(d_desc, leaf_off, total);
  return cudaGetLastError();
}

bool tn_vec2_enabled() { return g_knobs.skinny_vec2 != 0; }   // TN_SKINNY_VEC2=0: tests

template <typename F>
cudaError_t allow_big_smem(F* kern) {
  // the staged small operand can exceed the 48 KB default dynamic smem window
  return set_smem_attr(reinterpret_cast<const void*>(kern), 96 * 1024);
}

// instantiated (NMAX, VEC, R) combinations keep the accumulators in registers
template <int NMAX, int VEC, int R>
constexpr bool skinny_ok() { return NMAX * VEC * R <= 32 || R == 1; }

template <int NMAX, int VEC, int R>
cudaError_t enable_skinny_r(cudaError_t e) {
  if constexpr (skinny_ok<NMAX, VEC, R>()) {
    if (e == cudaSuccess) e = allow_big_smem(einsum_skinny_kernel<NMAX, VEC, true, 1, R>);
    if (VEC == 1 && e == cudaSuccess) e = allow_big_smem(einsum_skinny_kernel<NMAX, 1, true, 2, R>);
  }
  return e;
}

template <int NMAX>
cudaError_t enable_skinny(cudaError_t e) {
  if (e == cudaSuccess) e = allow_big_smem(einsum_skinny_kernel<NMAX, 1, false, 1, 1>);
  e = enable_skinny_r<NMAX, 1, 1>(e); e = enable_skinny_r<NMAX, 1, 2>(e); e = enable_skinny_r<NMAX, 1, 4>(e);
  if constexpr (NMAX <= 16) {
    e = enable_skinny_r<NMAX, 2, 1>(e); e = enable_skinny_r<NMAX, 2, 2>(e);
  }
  return e;
}

template <int KMAX>
cudaError_t enable_wide(cudaError_t e) {
  if (e == cudaSuccess) e = allow_big_smem(einsum_wide_kernel<KMAX, 1, 1>);
  if (e == cudaSuccess) e = allow_big_smem(einsum_wide_kernel<KMAX, 2, 1>);
  if (e == cudaSuccess) e = allow_big_smem(einsum_wide_kernel<KMAX, 1, 2>);
  return e;
}

cudaError_t enable_einsum_smem() {   // set_smem_attr: once per (kernel, device)
  cudaError_t e = cudaSuccess;
  e = enable_skinny<4>(e); e = enable_skinny<8>(e); e = enable_skinny<16>(e);
  e = enable_skinny<32>(e); e = enable_skinny<64>(e);
  e = enable_wide<2>(e); e = enable_wide<4>(e); e = enable_wide<8>(e); e = enable_wide<16>(e);
  return e;
}

template <int NMAX, int VEC, int R>
bool launch_skinny_r(const EinsumDesc* d_desc, const EinsumDesc& h, const int64_t* leaf_off, size_t smem,
                     bool kpair, cudaStream_t s) {
  if constexpr (skinny_ok<NMAX, VEC, R>()) {
    const int g = grid_for((h.J * (h.M / VEC) + R - 1) / R, 256);
    if (VEC == 1 && kpair) einsum_skinny_kernel<NMAX, 1, true, 2, R><<<g, 256, smem, s>>>(d_desc, leaf_off);
    else einsum_skinny_kernel<NMAX, VEC, true, 1, R><<<g, 256, smem, s>>>(d_desc, leaf_off);
    return true;
  }
  return false;
}

// rows per thread: enough that one round of loads is >= 16 complex (128 B) in flight
template <int NMAX, int VEC>
void launch_skinny(const EinsumDesc* d_desc, const EinsumDesc& h, const int64_t* leaf_off, size_t smem,
                   bool kpair, int rows, cudaStream_t s) {
  if constexpr (VEC == 1 || NMAX <= 16) {   // paired lanes only up to N = 16 (registers)
    if (!h.pow2) {
      einsum_skinny_kernel<NMAX, VEC, false, 1, 1><<<grid_for(h.M / VEC, 256), 256, smem, s>>>(d_desc, leaf_off);
      return;
    }
    const int rforce = g_knobs.skinny_rows;
    const int64_t kl = h.K < 8 ? h.K : 8;
    int R = (int)std::max<int64_t>(1, std::min<int64_t>(4, 16 / (kl * VEC)));
    if (rows) R = rows;
    if (rforce) R = rforce;
    if (h.J > 1) R = 1;                // batched: one slab of the small operand per row
    if (R >= 4 && launch_skinny_r<NMAX, VEC, 4>(d_desc, h, leaf_off, smem, kpair, s)) return;
    if (R >= 2 && launch_skinny_r<NMAX, VEC, 2>(d_desc, h, leaf_off, smem, kpair, s)) return;
    launch_skinny_r<NMAX, VEC, 1>(d_desc, h, leaf_off, smem, kpair, s);
  }
}

template <int KMAX>
void launch_wide(const EinsumDesc* d_desc, const EinsumDesc& h, const int64_t* leaf_off, size_t smem,
                 bool vec2, bool kpair, cudaStream_t s) {
  if (vec2) einsum_wide_kernel<KMAX, 2, 1><<<grid_for(h.M / 2, 256), 256, smem, s>>>(d_desc, leaf_off);
  else if (kpair) einsum_wide_kernel<KMAX, 1, 2><<<grid_for(h.M, 256), 256, smem, s>>>(d_desc, leaf_off);
  else einsum_wide_kernel<KMAX, 1, 1><<<grid_for(h.M, 256), 256, smem, s>>>(d_desc, leaf_off);
}

size_t chain_smem_bytes(const ChainDesc& d) {
  size_t ys = 0;
  for (int i = 0; i < d.L; ++i) ys += ((size_t)d.st[i].N * d.st[i].K + 1) & ~(size_t)1;
  return sizeof(float2) * (32 * ((size_t)d.buf_a + d.buf_b + 2 * ((size_t)1 << d.a0)) + ys) +
         sizeof(int32_t) * (size_t)d.n_tab;
}

cudaError_t launch_chain(const ChainDesc* d_desc, const ChainDesc& h, const int64_t* leaf_off, cudaStream_t s) {
  const size_t smem = chain_smem_bytes(h);
  if (cudaError_t e = set_smem_attr(reinterpret_cast<const void*>(einsum_chain_kernel), (int)smem)) return e;
  int per_sm = 0;
  if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, einsum_chain_kernel, CH_THREADS, smem) != cudaSuccess ||
      per_sm < 1)
    per_sm = 1;
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const int64_t g = std::min<int64_t>(h.n_tiles, (int64_t)sms * per_sm);
  einsum_chain_kernel<<<(unsigned)std::max<int64_t>(g, 1), CH_THREADS, smem, s>>>(d_desc, leaf_off);
  return cudaGetLastError();
}

int einsum_variants(const EinsumDesc& h) {
  if (h.mode == 1) return h.J > 1 ? 1 : 4;   // 0 heuristic rows, 1 previous design, 2..3: R = 1, 2
                                             // (batched merges: the new design only)
  if (h.mode == 3) return 2;   // 0 new design, 1 previous design
  if (h.mode == 4)             // 0 lanes over k, 1 lanes over (k group, n), 2 warps per batch,
                               // 3 slab-staged warps per batch (when eligible)
    return h.wd_ok ? 4 : (h.M <= 4 ? 3 : 2);
  return 1;
}

cudaError_t launch_einsum(const EinsumDesc* d_desc, const EinsumDesc& h, const int64_t* leaf_off,
                          cudaStream_t s, int variant) {
  const int th = 256;
  if (h.mode == 1 || h.mode == 3) {
    cudaError_t e = enable_einsum_smem();
    if (e != cudaSuccess) return e;
  }
  // pairs of lanes (16-B accesses) when the lane run is unit-stride and even and the
  // big operand's base is 16-B aligned (a leaf's dynamic slice offset is a sum of
  // strides of power-of-two dims above the unit-stride one, hence even)
  const bool vec2 = h.pow2 && h.m_sa[h.nm - 1] == 1 && h.V % 2 == 0 && h.a_off % 2 == 0 &&
                    tn_vec2_enabled();
  // pairs of k (16-B loads along a row of A) when A's innermost k dim is unit-stride
  // with an even extent and every other stride of A is even
  bool kpair = h.pow2 && h.nk > 0 && h.k_sa[h.nk - 1] == 1 && h.k_ext[h.nk - 1] % 2 == 0 &&
               h.K % 2 == 0 && h.a_off % 2 == 0 && tn_vec2_enabled();
  for (int i = 0; i < h.nm && kpair; ++i) kpair = h.m_sa[i] % 2 == 0 || h.m_ext[i] == 1;
  for (int i = 0; i + 1 < h.nk && kpair; ++i) kpair = h.k_sa[i] % 2 == 0;
  if ((g_knobs.simt_old || variant == 1) && (h.mode == 1 || h.mode == 3) && h.J == 1) {
    {
      allow_big_smem(einsum_skinny_old_kernel<4, true>); allow_big_smem(einsum_skinny_old_kernel<8, true>);
      allow_big_smem(einsum_skinny_old_kernel<16, true>); allow_big_smem(einsum_skinny_old_kernel<32, true>);
      allow_big_smem(einsum_skinny_old_kernel<64, true>); allow_big_smem(einsum_skinny_old_kernel<4, false>);
      allow_big_smem(einsum_skinny_old_kernel<8, false>); allow_big_smem(einsum_skinny_old_kernel<16, false>);
      allow_big_smem(einsum_skinny_old_kernel<32, false>); allow_big_smem(einsum_skinny_old_kernel<64, false>);
      allow_big_smem(einsum_skinny2_old_kernel<4, true>); allow_big_smem(einsum_skinny2_old_kernel<8, true>);
      allow_big_smem(einsum_skinny2_old_kernel<16, true>); allow_big_smem(einsum_wide_old_kernel<2>);
      allow_big_smem(einsum_wide_old_kernel<4>); allow_big_smem(einsum_wide_old_kernel<8>);
      allow_big_smem(einsum_wide_old_kernel<16>);
    }
    if (h.mode == 1) {
      const size_t smem = sizeof(float2) * h.K * h.N + sizeof(int64_t) * h.K;
      const int g = grid_for(h.M, 256);
      const bool v2 = h.pow2 && h.m_sa[h.nm - 1] == 1 && h.V % 2 == 0 && h.a_leaf < 0 && h.a_off % 2 == 0 && h.N <= 16;
#define TN_SKO(NM) (v2 ? (void)(einsum_skinny2_old_kernel<NM, true><<<grid_for(h.M / 2, 256), 256, smem, s>>>(d_desc, leaf_off)) \
                       : (void)(h.pow2 ? einsum_skinny_old_kernel<NM, true><<<g, 256, smem, s>>>(d_desc, leaf_off) \
                                       : einsum_skinny_old_kernel<NM, false><<<g, 256, smem, s>>>(d_desc, leaf_off)))
      if (h.N <= 4) TN_SKO(4); else if (h.N <= 8) TN_SKO(8); else if (h.N <= 16) TN_SKO(16);
      else if (h.N <= 32) { h.pow2 ? einsum_skinny_old_kernel<32, true><<<g, 256, smem, s>>>(d_desc, leaf_off) : einsum_skinny_old_kernel<32, false><<<g, 256, smem, s>>>(d_desc, leaf_off); }
      else { h.pow2 ? einsum_skinny_old_kernel<64, true><<<g, 256, smem, s>>>(d_desc, leaf_off) : einsum_skinny_old_kernel<64, false><<<g, 256, smem, s>>>(d_desc, leaf_off); }
#undef TN_SKO
    } else {
      const size_t smem = sizeof(float2) * h.K * h.N;
      const int g = grid_for(h.M, 256);
      if (h.K <= 2) einsum_wide_old_kernel<2><<<g, 256, smem, s>>>(d_desc, leaf_off);
      else if (h.K <= 4) einsum_wide_old_kernel<4><<<g, 256, smem, s>>>(d_desc, leaf_off);
      else if (h.K <= 8) einsum_wide_old_kernel<8><<<g, 256, smem, s>>>(d_desc, leaf_off);
      else einsum_wide_old_kernel<16><<<g, 256, smem, s>>>(d_desc, leaf_off);
    }
    return cudaGetLastError();
  }
  if (h.mode == 1) {
    const int rows = variant >= 2 ? variant - 1 : 0;
    const size_t smem = sizeof(float2) * (h.J > 1 ? h.n_yslabs : 1) * h.K * ((h.N + 1) & ~1) +
                        sizeof(int64_t) * h.K;
#define TN_SKINNY(NM)                                                            \
  (vec2 && NM <= 16 ? launch_skinny<NM, 2>(d_desc, h, leaf_off, smem, false, rows, s)  \
                    : launch_skinny<NM, 1>(d_desc, h, leaf_off, smem, kpair, rows, s))
    if (h.N <= 4) TN_SKINNY(4);
    else if (h.N <= 8) TN_SKINNY(8);
    else if (h.N <= 16) TN_SKINNY(16);
    else if (h.N <= 32) TN_SKINNY(32);
    else TN_SKINNY(64);
#undef TN_SKINNY
    return cudaGetLastError();
  }
  if (h.mode == 3) {
    const size_t smem = sizeof(float2) * ((h.K + 1) & ~1) * h.N;
    if (h.K <= 2) launch_wide<2>(d_desc, h, leaf_off, smem, vec2, kpair, s);
    else if (h.K <= 4) launch_wide<4>(d_desc, h, leaf_off, smem, vec2, kpair, s);
    else if (h.K <= 8) launch_wide<8>(d_desc, h, leaf_off, smem, vec2, kpair, s);
    else launch_wide<16>(d_desc, h, leaf_off, smem, vec2, kpair, s);
    return cudaGetLastError();
  }
  if (h.mode == 4) {
    const int64_t rows = h.J * h.M;
    int64_t blocks = (rows + 7) / 8;
    if (blocks > 148 * 16) blocks = 148 * 16;
    if (variant == 3 && h.wd_ok) {
      const size_t smem = sizeof(float2) * ((size_t)1 << h.wd_lb) + sizeof(int32_t) * (size_t)h.K;
      if (cudaError_t e = set_smem_attr(reinterpret_cast<const void*>(einsum_wdots_kernel), (int)smem)) return e;
      int64_t nb = h.wd_nslabs << h.wd_t;
      int per_sm = 0;
      if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, einsum_wdots_kernel, 32 * WDS_WARPS, smem) != cudaSuccess ||
          per_sm < 1)
        per_sm = 1;
      int dev = 0, sms = 148;
      cudaGetDevice(&dev);
      cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
      if (nb > (int64_t)sms * per_sm) nb = (int64_t)sms * per_sm;
      einsum_wdots_kernel<<<(unsigned)std::max<int64_t>(nb, 1), 32 * WDS_WARPS, smem, s>>>(d_desc, leaf_off);
      return cudaGetLastError();
    }
    if (variant == 2 || variant == 3) {
      int64_t jb = (h.J * ((h.N + 7) / 8) + 3) / 4;
      if (jb > 148 * 24) jb = 148 * 24;
      einsum_wdotj_kernel<4, 8><<<(unsigned)std::max<int64_t>(jb, 1), 128, 0, s>>>(d_desc, leaf_off);
    } else if (variant == 1)
      einsum_wdot2_kernel<<<(unsigned)std::max<int64_t>(blocks, 1), 256, 0, s>>>(d_desc, leaf_off);
    else
      einsum_wdot_kernel<<<(unsigned)std::max<int64_t>(blocks, 1), 256, 0, s>>>(d_desc, leaf_off);
    return cudaGetLastError();
  }
  if (h.mode == 2) {
    const int64_t P = h.J * h.M * h.N;
    const int64_t nchunk = (h.K + h.kchunk - 1) / h.kchunk;
    cudaError_t e = cudaMemsetAsync(h.partial, 0, sizeof(double) * 2 * P, s);
    if (e != cudaSuccess) return e;
    int64_t blocks = P * nchunk;
    if (blocks > 148 * 16) blocks = 148 * 16;
    einsum_dot_kernel<<<(unsigned)blocks, th, 0, s>>>(d_desc, leaf_off, nchunk);
    einsum_dot_finalize<<<grid_for(P, th), th, 0, s>>>(d_desc);
    return cudaGetLastError();
  }
  const int64_t total = h.J * h.M * h.N;
  einsum_kernel<<<grid_for(total, th), th, 0, s>>>(d_desc, leaf_off, total);
  return cudaGetLastError();
}

cudaError_t launch_gather_out(const double2* acc, const int32_t* pos, double2* out, int64_t n,
                              const int* flag, cudaStream_t s) {
  gather_out_kernel<<<grid_for(n, 256), 256, 0, s>>>(acc, pos, out, n, flag);
  return cudaGetLastError();
}

}  // namespace tn

namespace tn {
namespace {
__global__ void absmax_kernel(const float2* __restrict__ x, int64_t n, unsigned* out) {
  float m = 0.f;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    const float2 v = x[i];
    m = fmaxf(m, fmaxf(fabsf(v.x), fabsf(v.y)));
  }
  for (int o = 16; o > 0; o >>= 1) m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, o));
  if ((threadIdx.x & 31) == 0 && m > 0.f) atomicMax(out, __float_as_uint(m));
}
}  // namespace

cudaError_t launch_absmax(const float2* x, int64_t n, unsigned* out, cudaStream_t s) {
  int64_t b = (n + 255) / 256;
  if (b > 148 * 8) b = 148 * 8;
  if (b < 1) b = 1;
  absmax_kernel<<<(unsigned)b, 256, 0, s>>>(x, n, out);
  return cudaGetLastError();
}
}  // namespace tn

// ---------------------------------------------------------------- knobs, per-device attributes
#include <map>
#include <mutex>
namespace tn {
Knobs g_knobs;

namespace {
int env_or(const char* name, int dflt) {
  const char* v = getenv(name);
  return v ? atoi(v) : dflt;
}
std::mutex g_attr_mu;
std::map<std::pair<const void*, int>, int> g_attr;       // (kernel, device) -> smem bytes set
std::map<std::pair<const void*, int>, int> g_clusters;   // (kernel, device) -> max clusters
}  // namespace

void refresh_knobs() {
  Knobs k;
  k.gate_bps = env_or("TN_GATE_BPS", 4);
  k.skinny_rows = env_or("TN_SKINNY_ROWS", 0);
  k.simt_old = env_or("TN_SIMT_OLD", 0);
  k.skinny_vec2 = env_or("TN_SKINNY_VEC2", 1);
  k.narrow_mma = env_or("TN_NARROW_MMA", 1);
  k.l2hint = env_or("TN_GEMM_L2HINT", 0);   // measured neutral
  k.gate_mma = env_or("TN_GATE_MMA", 0);   // measured slower than the FFMA kernel
  k.prep_bp = env_or("TN_PREP_BP", 1);
  k.pair_min_m = env_or("TN_GEMM_PAIR_MIN_M", 512);
  g_knobs = k;
}

cudaError_t set_smem_attr(const void* kernel, int bytes) {
  int dev = 0;
  if (cudaError_t e = cudaGetDevice(&dev)) return e;
  std::lock_guard<std::mutex> lk(g_attr_mu);
  auto it = g_attr.find({kernel, dev});
  if (it != g_attr.end() && it->second >= bytes) return cudaSuccess;
  cudaError_t e = cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes);
  if (e == cudaSuccess) g_attr[{kernel, dev}] = bytes;
  return e;
}

int max_active_clusters(const void* kernel, const cudaLaunchConfig_t& cfg, int fallback) {
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) return fallback;
  std::lock_guard<std::mutex> lk(g_attr_mu);
  auto it = g_clusters.find({kernel, dev});
  if (it != g_clusters.end()) return it->second;
  int n = 0;
  if (cudaOccupancyMaxActiveClusters(&n, kernel, &cfg) != cudaSuccess || n <= 0) {
    cudaGetLastError();
    n = fallback;
  }
  g_clusters[{kernel, dev}] = n;
  return n;
}
}  // namespace tn
