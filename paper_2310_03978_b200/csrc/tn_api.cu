// Host side of the library: network validation, sparse-state tables, path replay
// and step planning, slice bookkeeping (a2), buffer liveness,
// the per-slice launch sequence (a3-a8), output mapping (a9) and the C ABI
// declared in include/tn.h.  Every arithmetic step of a contraction runs in the
// CUDA kernels of kernels.cu / gemm_tcgen05.cu; this file only plans and launches.
#include "tn_internal.h"
#include "tn.h"

#include <algorithm>
#include <array>
#include <climits>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <numeric>
#include <string>
#include <unordered_map>
#include <unordered_set>
#include <vector>

namespace {

thread_local std::string g_err;

tn_status fail(tn_status s, const std::string& m) {
  g_err = m;
  return s;
}

#define TN_CUDA(x)                                                                       \
  do {                                                                                   \
    cudaError_t e_ = (x);                                                                \
    if (e_ != cudaSuccess)                                                               \
      return fail(TN_ERR_CUDA, std::string(#x) + ": " + cudaGetErrorString(e_));          \
  } while (0)

constexpr int64_t GROUP = INT64_MIN;   // label of the merged open-group (sample) dim

struct VDim {
  int64_t label, ext, stride;
};

// A strided view of a live tensor.  The group dim (label GROUP) indexes the
// tensor's merged open group: entry g <-> table[g] (sorted projections of the
// samples onto `q`, qubit q[0] most significant).
struct View {
  int buf = 0;          // 0 = leaf buffer, 1 = arena
  int64_t off = 0;      // element offset
  int leaf = -1;        // leaf index (dynamic slice offset) or -1
  std::vector<VDim> dims;
  std::vector<int> q;
  std::vector<uint64_t> table;
  int absmax_slot = 0;
  bool has_group() const { return !q.empty(); }
  int64_t size() const {
    int64_t s = 1;
    for (auto& d : dims) s *= d.ext;
    return s;
  }
};

struct StepPlan {
  int i = 0, j = 0;
  bool merge = false, tc = false, final_step = false, swap = false;
  int64_t J = 1, m = 1, n = 1, k = 1;
  double tcc = 0, tmc = 0;
  std::vector<int32_t> ia, ib;
  int64_t ia_off = -1, ib_off = -1;     // offsets into the device table buffer
  int64_t wd_start_off = -1, wd_list_off = -1, wd_nslabs = 0;   // mode 4: batches by B slab
  int64_t out_off = -1, out_elems = 0;  // arena element offset
  View out;
  // device descriptor indices
  int einsum_idx = -1, prep_idx = -1;   // prep_idx: P at prep_idx, Q at prep_idx+1
  tn::GemmArgs gemm;
  int64_t prep_total[2] = {0, 0};
  int64_t R[2] = {0, 0}, Kpad = 0, G[2] = {1, 1};
  int in_slot[2] = {0, 0};
  int r_fast[2] = {0, 0};       // prep kernel kind per side (choose_prep_kind)
  int gtT[2] = {0, 0};          // general-transposer tile size per side
  int mode = 0;                 // SIMT mode: 0 general, 1 skinny, 2 split-K dot
  bool x_is_b = false;          // skinny: the big (streamed) operand is B
  std::vector<int64_t> vlabels; // skinny: labels of the lane (vector) run, outer -> inner
  // output label order chosen by the planner (consumer look-ahead): order1 = P side
  // (tensor cores) / A side (SIMT general) / X outer dims (skinny); order2 = Q / B / Y
  std::vector<int64_t> order1, order2;
  tn::EinsumDesc hdesc;         // host copy of the SIMT descriptor (launch parameters)
  // slab-grouped merge (tensor cores): the P side's rows are gathered (j, q) rows sorted
  // by the Q side's slab, each slab group padded to 128 rows; see DESIGN.md "Sparse merges"
  bool grouped = false;
  // dense merge: an Eq. 7 merge whose pairs (slabA(j), slabB(j)) cover most of the slab
  // product runs as ONE dense GEMM over [slabA rows] x [slabB rows] and the epilogue keeps
  // the pairs that exist (pair_map[a][b] = j, -1 = dropped); DESIGN.md "Sparse merges"
  bool dense_merge = false;
  // gate folding: this skinny SIMT step is not launched;
  // its tensor-core consumer's prep applies it while transposing (x_slot / y_slot: absmax
  // slots of its big and small operands)
  bool folded = false;
  // fused skinny chain (tn::ChainDesc): every member carries the chain index (tn_ctx::chains,
  // -1 = none); the last member launches the whole chain, the others (chained) are skipped
  int chain = -1;
  bool chained = false;
  double chain_tcc = 0, chain_tmc = 0;   // head: the chain's Eq. 4 flops; bytes it moves
  int x_slot = -1, y_slot = -1;
  std::vector<int32_t> pair_map;
  int64_t pair_off = -1;
  int64_t g_rows = 0;           // gathered rows (multiple of 128)
  std::vector<int32_t> g_rowmap, g_blk;   // output row of each gathered row; Q slab per block
  int64_t g_rowmap_off = -1, g_blk_off = -1;
  // tensor-core output map: the GEMM's row digits (P dims,
  // order1) and column digits (Q dims, order2) with their strides in the output view
  bool out_gen = false;
  std::vector<VDim> po, qo;
  int simt_variant = -1;        // SIMT kernel variant chosen by the first-slice autotuner
  // fused operand prep: side s of this tensor-core step
  // reads fp16 planes its producer's epilogue wrote (no prep launch); planes_consumer =
  // the step whose planes this step's epilogue writes (-1: writes complex64)
  bool skip_prep[2] = {false, false};
  int gate_k[2] = {0, 0};       // gate-folded prep: K of the folded gate per side
  int gate_n[2] = {0, 0};       // ... and its N (outputs per carry position)
  int planes_consumer = -1;
  tn::GemmArgs gemm_plain;      // the step's GEMM without fusion (first, absmax-seeding slice)
};

struct KStats {
  int64_t launches = 0;
  double ms = 0, flops = 0, bytes = 0;
};

struct Pending {
  cudaEvent_t a, b;
  int family;
  double flops, bytes;
  int step;                     // path step the launch belongs to, -1 = none
};

}  // namespace

struct tn_ctx {
  int device = 0;
  bool host_only = false;   // device = -1: plan/bookkeeping only, no CUDA calls
  cudaStream_t stream = nullptr;
  // device memory source (SURVEY.md §8 b: the caller's allocator, e.g. torch's caching
  // allocator); has_alloc = false: cudaMalloc / cudaFree.  owned: live blocks -> bytes
  tn_allocator alloc{};
  bool has_alloc = false;
  std::unordered_map<void*, size_t> owned;
  int num_sms = 148;
  // k-blocks per promoted TMEM chunk: 3-pass / 1-pass
  int kchunk3 = 1, kchunk1 = 0;
  int kchunk3_short = 1, shortk_max = 16;
  int group_m = 16;             // GEMM tile rasterization group (tile rows)
  bool autotune = true;         // TN_AUTOTUNE=0: SIMT steps use the heuristic kernel variant
  // CUDA graph of one slice's launch sequence (TN_GRAPHS=0 disables)
  bool use_graphs = true, tuned = false;
  cudaStream_t cap_stream = nullptr;
  cudaGraphExec_t gexec = nullptr;
  int g_prec = -1, g_topk = -1;
  int64_t graph_launches = 0;
  int64_t g_launch[4] = {0, 0, 0, 0};   // kernel launches per family inside the graph
  int simt_force = -1;          // TN_SIMT_VARIANT=v: every SIMT step uses variant v (tests)
  bool debug_plan = false;      // TN_DEBUG_PLAN=1: print operand layouts while planning
  int chain_mode = 1;           // TN_CHAIN=0: skinny chains run step by step (A/B, tests)
  int chain_maxbits = 8;        // TN_CHAIN_MAXBITS: touched bits per carry position
  double chain_min_save = 0;    // TN_CHAIN_MIN_SAVE_LOG2: HBM bytes a chain must save (2^x elements x 16 B)
  // network
  bool loaded = false, pathed = false, planned = false;
  int n_tensors = 0;
  std::vector<std::vector<int64_t>> labels, dims;
  std::vector<int64_t> data_off;             // complex offsets into host data
  int64_t n_data = 0;
  int n_open = 0;
  std::vector<int64_t> open_labels;
  std::unordered_map<int64_t, int> qubit_of;
  std::unordered_map<int64_t, int64_t> dim_of;
  std::unordered_map<int64_t, int> count_of;
  int64_t n_samples = 0;
  bool full_state = false;
  std::vector<uint64_t> packed;              // packed samples (qubit 0 = MSB)
  // leaves (after open-group gather)
  std::vector<View> leaf_views;              // unsliced leaf views
  std::vector<int64_t> leaf_src;             // device leaf element -> host complex index
  std::vector<int64_t> leaf_begin;           // element offset of each leaf in leaf buffer
  int64_t leaf_elems = 0;
  std::vector<float> leaf_absmax;
  float2* d_leaf = nullptr;
  float2* h_leaf_pinned = nullptr;
  // path / slices
  std::vector<std::pair<int, int>> path;
  std::vector<int64_t> sliced;
  int64_t n_slices = 1;
  // plan
  std::vector<StepPlan> steps;
  View root;
  // gate folding decided by a previous planning pass: the folded step's output is not
  // allocated and its inputs stay live until its consumer's prep has read them
  std::vector<char> fold_hint;
  // fused skinny chains: per step, the chain's launch step if the step is a chained
  // (not launched) member, else -1; set by one planning pass, honoured by the next (its
  // output is not materialised, its inputs live until the launch step)
  std::vector<int> chain_hint;
  bool replan = false;
  // index reordering (§4.1): 2 = every step's output in its consumer's
  // order (the generalised look-ahead, default), 1 = the paper's top-k rule (Fig. 3),
  // 0 = none (every output in Eq. 3's natural [J][P][Q] order); TN_REORDER / _TOPK
  int reorder_mode = 2, reorder_topk = 10;
  std::vector<char> reorder_sel, reorder_mod;   // mode 1: selected / modified steps
  std::vector<int32_t> out_pos;
  int64_t n_out = 0, acc_elems = 1;
  double flops_per_slice = 0, tc_flops = 0, bytes_per_slice = 0, peak = 0;
  int64_t arena_elems = 0, scratch_bytes = 0;
  // device buffers
  float2* d_arena = nullptr;
  uint8_t* d_scratch = nullptr;
  int32_t* d_tables = nullptr;
  double2* d_acc = nullptr;
  unsigned* d_absmax = nullptr;
  int* d_scales = nullptr;
  int64_t* d_leaf_off = nullptr;
  int64_t* d_counter = nullptr;
  int32_t* d_out_pos = nullptr;
  tn::SliceDesc* d_slice_desc = nullptr;
  int32_t* d_terms_i = nullptr;
  int64_t* d_terms_s = nullptr;
  tn::EinsumDesc* d_einsum = nullptr;
  std::vector<tn::ChainDesc> chains;   // host copies (launch parameters)
  tn::ChainDesc* d_chain = nullptr;
  int32_t* d_chain_tab = nullptr;
  tn::PrepDesc* d_prep = nullptr;
  float2* d_one = nullptr;
  double* d_partial = nullptr;     // split-K dot partial sums
  unsigned* d_hist = nullptr;      // delayed scaling: running output absmax per step
  int* d_pexp = nullptr;           // delayed scaling: exponent per step (slice_select)
  int* d_flag = nullptr;           // fused plane overflow flag
  double2* d_gather = nullptr;     // tn_sum_slices_host staging (n_out amplitudes)
  unsigned long long* d_wave = nullptr;   // GEMM wave-sync counter
  int64_t* d_gt = nullptr;         // general-transposer tile tables
  int64_t device_bytes = 0;
  // profiling
  bool profiling = false;
  std::vector<Pending> pending;
  KStats stats[4];
  std::vector<double> step_ms[4];  // per kernel family and path step (profiling)
};

namespace {

// ---------------------------------------------------------------- helpers

uint64_t project(uint64_t v, const std::vector<int>& q, int n_open) {
  uint64_t r = 0;
  for (int x : q) r = (r << 1) | ((v >> (n_open - 1 - x)) & 1ull);
  return r;
}

std::vector<uint64_t> table_for(const tn_ctx* c, const std::vector<int>& q) {
  std::vector<uint64_t> t;
  t.reserve(c->packed.size());
  for (uint64_t s : c->packed) t.push_back(project(s, q, c->n_open));
  std::sort(t.begin(), t.end());
  t.erase(std::unique(t.begin(), t.end()), t.end());
  return t;
}

int64_t index_in(const std::vector<uint64_t>& t, uint64_t v) {
  auto it = std::lower_bound(t.begin(), t.end(), v);
  if (it == t.end() || *it != v) return -1;
  return it - t.begin();
}

// Device memory of a context: every block comes from the caller's allocator when one
// was given to tn_create (on the context stream), else from cudaMalloc.
tn_status mem_alloc(tn_ctx* c, void** p, size_t bytes) {
  *p = nullptr;
  if (c->has_alloc) {
    *p = c->alloc.alloc(bytes, c->device, reinterpret_cast<void*>(c->stream), c->alloc.user);
    if (!*p) return fail(TN_ERR_RESOURCE, "allocator returned NULL for " + std::to_string(bytes) + " bytes");
  } else {
    cudaError_t e = cudaMalloc(p, bytes);
    if (e == cudaErrorMemoryAllocation) {
      cudaGetLastError();
      *p = nullptr;
      return fail(TN_ERR_RESOURCE, "device allocation of " + std::to_string(bytes) + " bytes failed");
    }
    if (e != cudaSuccess) return fail(TN_ERR_CUDA, std::string("cudaMalloc: ") + cudaGetErrorString(e));
  }
  c->owned[*p] = bytes;
  return TN_OK;
}

void mem_free(tn_ctx* c, void* p) {
  if (!p) return;
  auto it = c->owned.find(p);
  const size_t bytes = it == c->owned.end() ? 0 : it->second;
  if (it != c->owned.end()) c->owned.erase(it);
  if (c->has_alloc) c->alloc.free(p, bytes, c->device, reinterpret_cast<void*>(c->stream), c->alloc.user);
  else cudaFree(p);
}

void free_dev(tn_ctx* c) {
  if (c->host_only) { c->planned = false; return; }
  if (c->gexec) { cudaGraphExecDestroy(c->gexec); c->gexec = nullptr; }
  c->tuned = false;
  c->g_prec = c->g_topk = -1;
  void* ptrs[] = {c->d_arena, c->d_scratch, c->d_tables, c->d_acc, c->d_absmax, c->d_scales,
                  c->d_leaf_off, c->d_counter, c->d_out_pos, c->d_slice_desc, c->d_terms_i,
                  c->d_terms_s, c->d_einsum, c->d_prep, c->d_one, c->d_partial, c->d_gt,
                  c->d_hist, c->d_pexp, c->d_flag, c->d_wave, c->d_gather, c->d_chain, c->d_chain_tab};
  for (void* p : ptrs) mem_free(c, p);
  c->d_arena = nullptr; c->d_scratch = nullptr; c->d_tables = nullptr; c->d_acc = nullptr;
  c->d_absmax = nullptr; c->d_scales = nullptr; c->d_leaf_off = nullptr; c->d_counter = nullptr;
  c->d_out_pos = nullptr; c->d_slice_desc = nullptr; c->d_terms_i = nullptr; c->d_terms_s = nullptr;
  c->d_einsum = nullptr; c->d_prep = nullptr; c->d_one = nullptr;
  c->d_partial = nullptr;
  c->d_gt = nullptr;
  c->d_hist = nullptr; c->d_pexp = nullptr; c->d_flag = nullptr; c->d_wave = nullptr;
  c->d_gather = nullptr;
  c->d_chain = nullptr; c->d_chain_tab = nullptr;
  c->planned = false;
}

template <typename T>
tn_status dev_alloc(tn_ctx* c, T** p, size_t count) {
  size_t bytes = std::max<size_t>(count * sizeof(T), 16);
  void* q = nullptr;
  tn_status st = mem_alloc(c, &q, bytes);
  if (st) return st;
  *p = reinterpret_cast<T*>(q);
  c->device_bytes += bytes;
  return TN_OK;
}

// merge adjacent dims whose strides chain (row-major runs) — single stride list
void coalesce1(std::vector<VDim>& d) {
  std::vector<VDim> o;
  for (auto& x : d) {
    if (x.ext == 1) continue;
    if (!o.empty() && o.back().stride == x.ext * x.stride) {
      o.back().ext *= x.ext;
      o.back().stride = x.stride;
    } else {
      o.push_back(x);
    }
  }
  d.swap(o);
}

struct KDim {
  int64_t ext, sa, sb;
};
void coalesce2(std::vector<KDim>& d) {
  std::vector<KDim> o;
  for (auto& x : d) {
    if (x.ext == 1) continue;
    if (!o.empty() && o.back().sa == x.ext * x.sa && o.back().sb == x.ext * x.sb) {
      o.back().ext *= x.ext;
      o.back().sa = x.sa;
      o.back().sb = x.sb;
    } else {
      o.push_back(x);
    }
  }
  d.swap(o);
}

// dims reordered to follow `order` (labels; every dim's label appears once in it)
std::vector<VDim> arrange(const std::vector<VDim>& d, const std::vector<int64_t>& order) {
  std::vector<VDim> o;
  o.reserve(d.size());
  for (int64_t l : order)
    for (auto& x : d)
      if (x.label == l) { o.push_back(x); break; }
  return o;
}

// Bit-permutation transposer plan (prep kind 4, kernels.cu prep_bp_kernel).  With
// every row / k extent a power of two and K = Kpad, destination element index bit
// b (k bits innermost, then r bits) has a source weight ws_b.  The tile takes the
// destination's innermost bits (>= 3: 8-element plane vectors) and the source's
// smallest-weight bits; e (load order) sorts tile bits by source weight, f (store
// order) by destination bit.  Fills the kind-4 fields and the tile tables.
bool plan_bp(tn::PrepDesc& p, std::vector<int64_t>& tab) {
  auto p2 = [](int64_t x) { return x > 0 && (x & (x - 1)) == 0; };
  if (p.Kpad != p.K || p.K < 8 || !p2(p.K) || !p2(p.R) || p.rowoff) return false;
  std::vector<int64_t> ws;
  for (int d = p.nk - 1; d >= 0; --d) {
    if (!p2(p.k_ext[d])) return false;
    for (int64_t e = 1; e < p.k_ext[d]; e <<= 1) ws.push_back(e * p.k_s[d]);
  }
  for (int d = p.nr - 1; d >= 0; --d) {
    if (!p2(p.r_ext[d])) return false;
    for (int64_t e = 1; e < p.r_ext[d]; e <<= 1) ws.push_back(e * p.r_s[d]);
  }
  const int nb = (int)ws.size();
  if (nb < 8 || nb - 8 > TN_MAXD) return false;
  const int t = std::min(12, nb);
  std::vector<int> bysrc(nb);
  std::iota(bysrc.begin(), bysrc.end(), 0);
  std::stable_sort(bysrc.begin(), bysrc.end(), [&](int a, int b) { return ws[a] < ws[b]; });
  std::vector<char> in(nb, 0);
  int cnt = 0;
  auto add = [&](int b) { if (cnt < t && !in[b]) { in[b] = 1; ++cnt; } };
  for (int b = 0; b < 3; ++b) add(b);                      // 8-element plane vectors
  for (int i = 0; i < 6 && i < nb; ++i) add(bysrc[i]);     // source run (up to 512 B)
  for (int b = 3; b < 6; ++b) add(b);                      // destination run (128 B / plane)
  for (int i = 6; i < nb; ++i) add(bysrc[i]);              // more source locality
  std::vector<int> ebit, fbit;                             // tile bits in e / f order
  for (int i = 0; i < nb; ++i) if (in[bysrc[i]]) ebit.push_back(bysrc[i]);
  for (int b = 0; b < nb; ++b) if (in[b]) fbit.push_back(b);
  std::vector<int> epos(nb, -1);
  for (int i = 0; i < t; ++i) epos[ebit[i]] = i;
  const int T = 1 << t;
  // swizzle: lanes of the store phase vary f bits 3..7; give each of their e
  // positions >= 4 a distinct slot bit in {1,2,3} not already varied (bit 0 stays:
  // pairs (e, e+1) are stored as one 16-B vector)
  std::vector<int> mp(t, 0);
  {
    std::vector<char> used(4, 0);
    for (int i = 3; i < 8 && i < t; ++i) if (epos[fbit[i]] < 4) used[epos[fbit[i]]] = 1;
    for (int i = 3; i < 8 && i < t; ++i) {
      const int pe = epos[fbit[i]];
      if (pe < 4) continue;
      for (int u = 1; u < 4; ++u)
        if (!used[u]) { used[u] = 1; mp[pe] = 1 << u; break; }
    }
  }
  std::vector<uint8_t> m(T / 16, 0);
  for (int h = 0; h < T / 16; ++h)
    for (int pe = 4; pe < t; ++pe) if ((h << 4) >> pe & 1) m[h] ^= (uint8_t)mp[pe];
  tab.assign(128 + T / 8 + T / 4 + (T / 16 + 7) / 8, 0);
  for (int x = 0; x < 64; ++x)
    for (int i = 0; i < 6; ++i) {
      if ((x >> i & 1) && i < t) tab[x] += ws[ebit[i]];
      if ((x >> i & 1) && 6 + i < t) tab[64 + x] += ws[ebit[6 + i]];
    }
  for (int q = 0; q < T / 8; ++q)
    for (int i = 3; i < t; ++i) if (q >> (i - 3) & 1) tab[128 + q] += int64_t(1) << fbit[i];
  uint16_t* slot = reinterpret_cast<uint16_t*>(tab.data() + 128 + T / 8);
  for (int f = 0; f < T; ++f) {
    int e = 0;
    for (int i = 0; i < t; ++i) if (f >> i & 1) e |= 1 << epos[fbit[i]];
    slot[f] = (uint16_t)(e ^ m[e >> 4]);
  }
  memcpy(tab.data() + 128 + T / 8 + T / 4, m.data(), m.size());
  p.nc = 0;
  for (int b = 0; b < nb; ++b)
    if (!in[b]) {
      p.c_src[p.nc] = ws[b];
      p.c_dst[p.nc] = int64_t(1) << b;
      ++p.nc;
    }
  p.nC = int64_t(1) << p.nc;
  bool vec = ws[ebit[0]] == 1 && (p.G == 1 || p.g_stride % 2 == 0);
  for (int b = 0; b < nb; ++b) if (b != ebit[0] && ws[b] % 2 != 0) vec = false;
  p.bp_vec = vec ? 1 : 0;
  p.bp_t = t;
  p.T = T;
  // self-check (host, a few tiles): replay the kernel's load / store addressing and
  // compare every element with the plain digit decomposition of its destination
  {
    std::vector<int> einv(T, -1);
    for (int e = 0; e < T; ++e) {
      const int sl = e ^ m[e >> 4];
      if (sl < 0 || sl >= T || einv[sl] >= 0) return false;
      einv[sl] = e;
    }
    auto ref_src = [&](int64_t di) {
      const int64_t rk = p.R * p.K;
      const int64_t g = di / rk;
      int64_t r = (di % rk) / p.K, k = di % p.K, off = g * p.g_stride;
      for (int d = p.nk - 1; d >= 0; --d) { off += (k % p.k_ext[d]) * p.k_s[d]; k /= p.k_ext[d]; }
      for (int d = p.nr - 1; d >= 0; --d) { off += (r % p.r_ext[d]) * p.r_s[d]; r /= p.r_ext[d]; }
      return off;
    };
    const int64_t tiles = p.G * p.nC;
    for (int64_t c : {int64_t(0), int64_t(1), tiles / 3, tiles - 1}) {
      if (c < 0 || c >= tiles) continue;
      const int64_t g = c >> p.nc, cc = c - (g << p.nc);
      int64_t sc = g * p.g_stride, dc = g * p.R * p.Kpad;
      for (int i = 0; i < p.nc; ++i) if ((cc >> i) & 1) { sc += p.c_src[i]; dc += p.c_dst[i]; }
      for (int f = 0; f < T; ++f) {
        const int e = einv[slot[f]];
        const int64_t so = sc + tab[e & 63] + tab[64 + (e >> 6)];
        const int64_t di = dc + tab[128 + (f >> 3)] + (f & 7);
        if (so != ref_src(di)) return false;
      }
    }
  }
  return true;
}

// Gate-folded prep plan (prep kind 5, kernels.cu prep_gate_kernel).  The operand is
// the output out[o][n][v] (contiguous [Xo][N][V]) of the skinny SIMT step `e`; each
// plane-layout bit is a carry bit (an o or v bit: an X weight) or an n bit.  The tile
// holds every n bit, the plane vectors' 3 lowest destination bits and the carry bits of
// smallest X weight; the source tile is its carry bits plus all k bits.
bool plan_gate(tn::PrepDesc& p, const tn::EinsumDesc& e, std::vector<int64_t>& tab) {
  auto p2 = [](int64_t x) { return x > 0 && (x & (x - 1)) == 0; };
  auto lg = [](int64_t x) { int q = 0; while ((int64_t(1) << q) < x) ++q; return q; };
  if (p.Kpad != p.K || p.K < 8 || !p2(p.K) || !p2(p.R) || p.G != 1 || p.rowoff) return false;
  if (e.mode != 1 || e.J != 1 || e.acc || !p2(e.N) || !p2(e.K) || !p2(e.V) || !p2(e.M)) return false;
  if (e.N * e.K > 512 || e.N > 256 || e.K > 16 || e.nn > 8 || e.nk > 8) return false;
  const int lv = lg(e.V), ln = lg(e.N), lk = lg(e.K), lo = lg(e.M / e.V);
  // X weight of each o-index bit (Xo dims, outer -> inner in m_ext / m_sa [0, nm-1))
  std::vector<int64_t> ow;
  for (int d = e.nm - 2; d >= 0; --d) {
    if (!p2(e.m_ext[d])) return false;
    for (int64_t t = 1; t < e.m_ext[d]; t <<= 1) ow.push_back(e.m_sa[d] * t);
  }
  if ((int)ow.size() != lo) return false;
  const int64_t vs = e.m_sa[e.nm - 1];
  std::vector<int64_t> kw;                         // X weight of each k-index bit
  for (int d = e.nk - 1; d >= 0; --d) {
    if (!p2(e.k_ext[d])) return false;
    for (int64_t t = 1; t < e.k_ext[d]; t <<= 1) kw.push_back(e.k_sa[d] * t);
  }
  if ((int)kw.size() != lk) return false;
  // destination bits -> S-output weights (as in plan_bp)
  std::vector<int64_t> ws;
  for (int d = p.nk - 1; d >= 0; --d) {
    if (!p2(p.k_ext[d])) return false;
    for (int64_t t = 1; t < p.k_ext[d]; t <<= 1) ws.push_back(t * p.k_s[d]);
  }
  for (int d = p.nr - 1; d >= 0; --d) {
    if (!p2(p.r_ext[d])) return false;
    for (int64_t t = 1; t < p.r_ext[d]; t <<= 1) ws.push_back(t * p.r_s[d]);
  }
  const int nb = (int)ws.size();
  if (nb != lv + ln + lo || nb < 8) return false;
  std::vector<int> nbit(nb, -1);                   // n-index bit, or -1 for a carry bit
  std::vector<int64_t> xw(nb, 0);                  // X weight of a carry bit
  for (int b = 0; b < nb; ++b) {
    if (!p2(ws[b])) return false;
    const int beta = lg(ws[b]);
    if (beta < lv) xw[b] = vs << beta;
    else if (beta < lv + ln) nbit[b] = beta - lv;
    else xw[b] = ow[beta - lv - ln];
  }
  std::vector<char> in(nb, 0);
  int td = 0;
  auto ts_of = [&](int t) { return t - ln + lk; };
  auto add = [&](int b) {
    if (in[b] || td >= 12 || ts_of(td + 1) > 12 + (nbit[b] >= 0 ? 1 : 0)) return;
    in[b] = 1;
    ++td;
  };
  for (int b = 0; b < nb; ++b) if (nbit[b] >= 0) { in[b] = 1; ++td; }
  if (ts_of(td) > 12 || td > 12) return false;
  for (int b = 0; b < 3; ++b) add(b);
  // an expanding gate (N >= K) writes at least as many bytes as it reads: destination
  // bits 3-4 next, so a tile's plane stores are 64-B runs (whole sectors) instead of
  // scattered 16-B vectors (C4-sparse step 210 -> 217: N = 16, K = 4)
  if (e.N >= e.K)
    for (int b = 3; b < 5 && b < nb; ++b) add(b);
  std::vector<int> bysrc;                          // carry bits by X weight
  for (int b = 0; b < nb; ++b) if (nbit[b] < 0) bysrc.push_back(b);
  std::stable_sort(bysrc.begin(), bysrc.end(), [&](int a, int b) { return xw[a] < xw[b]; });
  for (int i = 0; i < 5 && i < (int)bysrc.size(); ++i) add(bysrc[i]);
  for (int b = 3; b < 6 && b < nb; ++b) add(b);
  for (int i = 5; i < (int)bysrc.size(); ++i) add(bysrc[i]);
  for (int b = 0; b < 3; ++b) if (!in[b]) return false;
  if (td > 12 || ts_of(td) > 12) return false;
  const int cb = td - ln, tsb = cb + lk, TD = 1 << td;
  std::vector<int> ebit;                           // carry tile bits in X-weight order
  for (int b : bysrc) if (in[b]) ebit.push_back(b);
  std::vector<int> epos(nb, -1);
  for (int i = 0; i < cb; ++i) epos[ebit[i]] = i;
  std::vector<int> fbit;
  for (int b = 0; b < nb; ++b) if (in[b]) fbit.push_back(b);
  tab.assign(128 + TD / 8 + (4096 + 256) / 4, 0);   // fc[4096] u16 then fn[256] u16
  auto ew = [&](int i) { return i < cb ? xw[ebit[i]] : kw[i - cb]; };   // X weight of e bit i
  for (int x = 0; x < 64; ++x)
    for (int i = 0; i < 6; ++i) {
      if ((x >> i & 1) && i < tsb) tab[x] += ew(i);
      if ((x >> i & 1) && 6 + i < tsb) tab[64 + x] += ew(6 + i);
    }
  for (int q = 0; q < TD / 8; ++q)
    for (int i = 3; i < td; ++i) if (q >> (i - 3) & 1) tab[128 + q] += int64_t(1) << fbit[i];
  // f (dest-order tile index) is separable into its carry bits and its n bits
  uint16_t* fc = reinterpret_cast<uint16_t*>(tab.data() + 128 + TD / 8);
  uint16_t* fnn = fc + 4096;
  std::vector<int32_t> cn(TD);
  for (int f = 0; f < TD; ++f) {
    int cp = 0, n = 0;
    for (int i = 0; i < td; ++i)
      if (f >> i & 1) {
        if (nbit[fbit[i]] >= 0) n |= 1 << nbit[fbit[i]];
        else cp |= 1 << epos[fbit[i]];
      }
    cn[f] = cp | (n << 16);
    if (n == 0) fc[cp] = (uint16_t)f;
    if (cp == 0) fnn[n] = (uint16_t)f;
  }
  for (int f = 0; f < TD; ++f)   // separability check: f = fc[carry] + fn[n]
    if (fc[cn[f] & 0xFFFF] + fnn[cn[f] >> 16] != f) return false;
  p.nc = 0;
  for (int b = 0; b < nb; ++b)
    if (!in[b]) {
      if (p.nc >= TN_MAXD) return false;
      p.c_src[p.nc] = xw[b];
      p.c_dst[p.nc] = int64_t(1) << b;
      ++p.nc;
    }
  p.nC = int64_t(1) << p.nc;
  p.bp_t = td;
  p.g_ts = tsb;
  {                                                // 16-B pair loads: e bit 0 has X weight 1
    bool vec = tsb >= 1 && ew(0) == 1;
    for (int i = 1; i < tsb && vec; ++i) vec = ew(i) % 2 == 0;
    for (int i = 0; i < p.nc && vec; ++i) vec = p.c_src[i] % 2 == 0;
    p.bp_vec = vec ? 1 : 0;
  }
  p.g_cbits = cb;
  p.g_N = (int32_t)e.N;
  p.g_K = (int32_t)e.K;
  p.T = TD;
  p.g_nn = e.nn;
  p.g_nk = e.nk;
  for (int d = 0; d < e.nn; ++d) { p.gy_n_ext[d] = e.n_ext[d]; p.gy_n_s[d] = e.n_sb[d]; }
  for (int d = 0; d < e.nk; ++d) { p.gy_k_ext[d] = e.k_ext[d]; p.gy_k_s[d] = e.k_sb[d]; }
  // self-check (a few tiles): carry X offset and n index of every destination element
  // against the plain decomposition of its S-output offset
  auto xoff = [&](int64_t so) {                    // S-output offset -> (X offset of (o, v), n)
    const int64_t v = so & (e.V - 1), o = so >> (lv + ln);
    int64_t off = v * vs;
    for (int i = 0; i < lo; ++i) if (o >> i & 1) off += ow[i];
    return std::make_pair(off, (so >> lv) & (e.N - 1));
  };
  for (int64_t c : {int64_t(0), int64_t(1), p.nC / 3, p.nC - 1}) {
    if (c < 0 || c >= p.nC) continue;
    int64_t sc = 0, dc = 0;
    for (int i = 0; i < p.nc; ++i) if ((c >> i) & 1) { sc += p.c_src[i]; dc += p.c_dst[i]; }
    for (int f = 0; f < TD; ++f) {
      const int cp = cn[f] & 0xFFFF, n = cn[f] >> 16;
      const int64_t di = dc + tab[128 + (f >> 3)] + (f & 7);
      int64_t so = 0;
      for (int b = 0; b < nb; ++b) if (di >> b & 1) so += ws[b];
      const auto ref = xoff(so);
      if (sc + tab[cp & 63] + tab[64 + (cp >> 6)] != ref.first || n != ref.second) return false;
      for (int k = 0; k < e.K; ++k) {         // the k part: kernel e index vs plain X offset
        const int ek = cp + (k << cb);
        int64_t kx = 0, t = k;
        for (int d = e.nk - 1; d >= 0; --d) { kx += (t % e.k_ext[d]) * e.k_sa[d]; t /= e.k_ext[d]; }
        if (ek >= (1 << tsb) || sc + tab[ek & 63] + tab[64 + (ek >> 6)] != ref.first + kx) return false;
      }
    }
  }
  return true;
}

// Operand-prep kernel choice: 1 = direct (source walks k with a
// contiguous innermost k run of >= 8), 4 = bit-permutation transposer (power-of-
// two extents), 2 = general transposer (blocks: the destination's contiguous
// k-run x the source's innermost run), 0 = r/k tile transposer (fallback).
// Fills the transposer fields; `tab` receives kind 2 / 4 tile tables.
int choose_prep_kind(tn::PrepDesc& p, int force, std::vector<int64_t>& tab) {
  if (force == 0 || force == 1) return force;
  if (force != 2 && force != 4 && p.nk > 0 && p.k_s[p.nk - 1] == 1 && p.k_ext[p.nk - 1] % 8 == 0) return 1;
  if (force != 2 && (tn::g_knobs.prep_bp || force == 4) && plan_bp(p, tab)) return 4;
  if (p.K % 8 != 0 || p.Kpad != p.K || (force != 2 && p.G * p.R * p.K < 2048))
    return p.read_r_fast ? 0 : 1;
  struct D { int64_t e, s, t; };
  std::vector<D> pool;
  if (p.G > 1) pool.push_back({p.G, p.g_stride, p.R * p.Kpad});
  int64_t t = p.Kpad;
  for (int d = p.nr - 1; d >= 0; --d) { pool.push_back({p.r_ext[d], p.r_s[d], t}); t *= p.r_ext[d]; }
  t = 1;
  for (int d = p.nk - 1; d >= 0; --d) { pool.push_back({p.k_ext[d], p.k_s[d], t}); t *= p.k_ext[d]; }
  // Tile = set of dims holding the source's innermost run (>= 32 elements, walked
  // by the load phase) and the destination's contiguous k-run (>= 64, walked by
  // the half2 store phase).  Dims are split (power-of-two extents) to hit sizes.
  std::vector<D> tl;
  auto grab = [&](int q, int64_t need) {          // move (the inner `need` part of) pool[q]
    D x = pool[q];
    if (x.e > need && x.e % need == 0) {
      tl.push_back({need, x.s, x.t});
      pool[q] = {x.e / need, x.s * need, x.t * need};
    } else {
      tl.push_back(x);
      pool.erase(pool.begin() + q);
    }
  };
  int64_t run = 1;                                 // source run
  while (run < 32 && !pool.empty()) {
    int q = 0;
    for (int i = 1; i < (int)pool.size(); ++i) if (pool[i].s < pool[q].s) q = i;
    const int64_t before = tl.size();
    grab(q, (32 + run - 1) / run);
    run *= tl[before].e;
  }
  int64_t drun = 1;                                // destination run (stride-1 chain)
  while (drun < 64) {
    int q = -1;
    bool in_tile = false;
    for (int i = 0; i < (int)tl.size(); ++i) if (tl[i].t == drun) { q = i; in_tile = true; }
    if (!in_tile)
      for (int i = 0; i < (int)pool.size(); ++i) if (pool[i].t == drun) q = i;
    if (q < 0) break;
    if (in_tile) {
      drun *= tl[q].e;
    } else {
      const int64_t before = tl.size();
      grab(q, (64 + drun - 1) / drun);
      drun *= tl[before].e;
    }
  }
  int64_t T = 1;
  for (auto& x : tl) T *= x.e;
  while (T < 2048 && !pool.empty()) {             // amortise the per-tile overhead
    int q = 0;
    for (int i = 1; i < (int)pool.size(); ++i) if (pool[i].s < pool[q].s) q = i;
    const int64_t before = tl.size();
    grab(q, (2048 + T - 1) / T);
    T *= tl[before].e;
  }
  for (auto& x : pool)
    if (x.e & (x.e - 1)) return p.read_r_fast ? 0 : 1;   // outer dims use shift tables
  if (drun < 2 || drun % 2 != 0 || T > 4096 || T % 2 != 0 || (int)tl.size() > 12 ||
      (int)pool.size() > TN_MAXD)
    return p.read_r_fast ? 0 : 1;
  // source order (outer -> inner = descending source stride) and destination order
  std::vector<D> ts = tl, td = tl;
  std::sort(ts.begin(), ts.end(), [](const D& a, const D& b) { return a.s > b.s; });
  std::vector<int> idx(tl.size());
  std::iota(idx.begin(), idx.end(), 0);
  std::sort(idx.begin(), idx.end(), [&](int a, int b) { return tl[a].t > tl[b].t; });
  p.nt = (int)tl.size();
  for (int i = 0; i < p.nt; ++i) { p.ts_ext[i] = ts[i].e; p.ts_src[i] = ts[i].s; p.ts_dst[i] = ts[i].t; }
  for (int i = 0; i < p.nt; ++i) {
    const D& x = tl[idx[i]];
    p.td_ext[i] = x.e;
    int pos = -1;
    for (int j = 0; j < p.nt; ++j)
      if (ts[j].s == x.s && ts[j].t == x.t && ts[j].e == x.e) pos = j;
    p.td_pos[i] = pos;
  }
  p.nc = (int)pool.size();
  p.nC = 1;
  for (int i = 0; i < p.nc; ++i) {
    p.c_ext[i] = pool[i].e; p.c_src[i] = pool[i].s; p.c_dst[i] = pool[i].t; p.nC *= pool[i].e;
    int sh = 0;
    while ((int64_t(1) << sh) < pool[i].e) ++sh;
    p.c_sh[i] = (uint8_t)sh;
  }
  p.T = (int32_t)T;
  return 2;
}

// General-transposer tile tables (plan time): srcoff[e] for tile element e in
// source order, then dstoff[f] and the source-order position spos[f] of element f
// in destination order (int32, packed two per int64 word).
std::vector<int64_t> gt_tables(const tn::PrepDesc& p) {
  const int T = p.T, nt = p.nt;
  std::vector<int64_t> tab(2 * (size_t)T + ((size_t)T + 1) / 2, 0);
  int32_t* spos = reinterpret_cast<int32_t*>(tab.data() + 2 * T);
  std::vector<int64_t> lstride(nt, 1);
  for (int q = nt - 2; q >= 0; --q) lstride[q] = lstride[q + 1] * p.ts_ext[q + 1];
  for (int e = 0; e < T; ++e) {
    int64_t t = e, so = 0;
    for (int i = nt - 1; i >= 0; --i) { so += (t % p.ts_ext[i]) * p.ts_src[i]; t /= p.ts_ext[i]; }
    tab[e] = so;
    int64_t f = e, pos = 0, dof = 0;
    for (int i = nt - 1; i >= 0; --i) {
      const int q = p.td_pos[i];
      const int64_t digit = f % p.td_ext[i];
      f /= p.td_ext[i];
      pos += digit * lstride[q];
      dof += digit * p.ts_dst[q];
    }
    tab[T + e] = dof;
    spos[e] = (int32_t)pos;
  }
  return tab;
}

// log2 shift tables for the SIMT kernels (pow2 = every extent a power of two)
void fill_shifts(tn::EinsumDesc& e) {
  auto lg = [](int64_t x) -> int { int s = 0; while ((int64_t(1) << s) < x) ++s; return s; };
  auto p2 = [](int64_t x) { return x > 0 && (x & (x - 1)) == 0; };
  bool ok = true;
  for (int i = 0; i < e.nm; ++i) { ok &= p2(e.m_ext[i]); e.m_sh[i] = (uint8_t)lg(e.m_ext[i]); }
  for (int i = 0; i < e.nn; ++i) { ok &= p2(e.n_ext[i]); e.n_sh[i] = (uint8_t)lg(e.n_ext[i]); }
  for (int i = 0; i < e.nk; ++i) { ok &= p2(e.k_ext[i]); e.k_sh[i] = (uint8_t)lg(e.k_ext[i]); }
  e.pow2 = ok ? 1 : 0;
}

// Slab-staged warp dot (mode 4 variant 3): eligible when B's n and k bits tile its slab
// exactly (the offsets of one slab are a bit permutation of [0, N*K)) and the top bits of
// the slab offset are n bits, so a part of 2^lb elements — all k of N >> t columns — is
// one contiguous run that fits shared memory.  Fills the wd_* fields (wd_ok = 1) or
// leaves wd_ok = 0.
void plan_wd_staged(tn::EinsumDesc& e, int64_t nslabs) {
  e.wd_ok = 0;
  if (!e.pow2 || e.J <= 1 || e.M > 4 || e.N > 256 || e.K > 8192 || e.a_gs >= (int64_t(1) << 31)) return;
  if (e.J < 4 * nslabs) return;   // staging pays only when several batches share a slab
  const int64_t NK = e.N * e.K;
  int L = 0;
  while ((int64_t(1) << L) < NK) ++L;
  if ((int64_t(1) << L) != NK || L > 30 || e.b_gs < NK) return;
  // weight bit -> (is_n, canonical weight)
  std::vector<int> isn(L, -1);
  std::vector<int64_t> canon(L, 0);
  auto add = [&](int64_t stride, int sh, int64_t cw, int n) {
    for (int b = 0; b < sh; ++b) {
      const int64_t w = stride << b;
      if ((w & (w - 1)) != 0 || w >= NK) return false;
      int q = 0;
      while ((int64_t(1) << q) < w) ++q;
      if (isn[q] >= 0) return false;
      isn[q] = n;
      canon[q] = cw << b;
    }
    return true;
  };
  int64_t cw = 1;
  for (int i = e.nn - 1; i >= 0; --i) {
    if (!add(e.n_sb[i], e.n_sh[i], cw, 1)) return;
    cw *= e.n_ext[i];
  }
  cw = 1;
  for (int i = e.nk - 1; i >= 0; --i) {
    if (!add(e.k_sb[i], e.k_sh[i], cw, 0)) return;
    cw *= e.k_ext[i];
  }
  for (int q = 0; q < L; ++q) if (isn[q] < 0) return;
  // smallest t with a part of <= 16384 elements (128 KiB) whose top t bits are n bits
  int t = 0;
  while (L - t > 14) {
    if (t >= 3 || isn[L - 1 - t] != 1) return;
    ++t;
  }
  const int lb = L - t;
  // local n bits: the non-top n bits ranked by canonical weight
  std::vector<std::pair<int64_t, int>> nb;
  for (int q = 0; q < lb; ++q) if (isn[q] == 1) nb.push_back({canon[q], q});
  std::sort(nb.begin(), nb.end());
  if (nb.size() > 5) return;   // <= 32 local columns
  for (int q = 0; q < 16; ++q) e.wd_contrib[q] = 0;
  for (int q = 0; q < lb; ++q) {
    if (isn[q] == 0) e.wd_contrib[q] = (int32_t)canon[q];
    else {
      int r = 0;
      while (nb[r].second != q) ++r;
      e.wd_contrib[q] = (int32_t)((int64_t(1) << r) * e.K);
    }
  }
  const int np = 1 << (int)nb.size();
  for (int x = 0; x < 32; ++x) {
    int64_t v = 0;
    for (int r = 0; r < (int)nb.size(); ++r) if ((x >> r) & 1) v += nb[r].first;
    e.wd_nloc[x] = x < np ? (int32_t)v : 0;
  }
  for (int p = 0; p < 8; ++p) {
    int64_t v = 0;
    for (int i = 0; i < t; ++i) if ((p >> i) & 1) v += canon[lb + i];
    e.wd_ptop[p] = p < (1 << t) ? (int32_t)v : 0;
  }
  e.wd_t = t;
  e.wd_lb = lb;
  e.wd_np = np;
  e.wd_nslabs = nslabs;
  e.wd_ok = 1;
}

// Fused skinny chain (tn::ChainDesc): steps es[0..L-1] are mode-1 skinny
// einsums, es[i+1] reading es[i]'s output [o][n][v] as its big operand X.  Every index bit
// gets a global id (the first input's offset bits 0..a-1; an output's v / o bits inherit
// the ids of the X bits they come from, its n bits are fresh); U = ids some step contracts
// (k) or creates (n).  Carry bits (first-input ids outside U) pass every step unchanged.
// Accepted when: every X view is an exact bit permutation of its tensor, offset bits 0-4
// of the first input and of the last output are the same carry ids (the 32 lanes, unit
// stride at both ends), <= 32 further carry bits, K <= 16, and every tensor keeps
// <= maxbits touched bits per carry position.  Fills cd (pointers except tab) and tab.
bool plan_chain(const std::vector<const tn::EinsumDesc*>& es, int maxbits, tn::ChainDesc& cd,
                std::vector<int32_t>& tab) {
  auto lg = [](int64_t x) { int q = 0; while ((int64_t(1) << q) < x) ++q; return q; };
  auto p2 = [](int64_t x) { return x > 0 && (x & (x - 1)) == 0; };
  const int L = (int)es.size();
  if (L < 2 || L > tn::TN_CHAIN_MAX) return false;
  int next_gid = 0;
  std::vector<int> prev;                       // gid of each offset bit of the current input
  std::vector<std::vector<int>> tens;          // gids of T_0 .. T_L by offset bit
  std::vector<std::vector<int>> kg(L), pog(L), ng(L);
  std::vector<char> inU(4096, 0);
  for (int i = 0; i < L; ++i) {
    const tn::EinsumDesc& e = *es[i];
    if (e.mode != 1 || e.J != 1 || e.acc || !e.pow2 || e.K > 16 || e.N > 256 || e.N * e.K > 4096) return false;
    if (!p2(e.N) || !p2(e.K) || !p2(e.V) || !p2(e.M)) return false;
    // X weights by role: o (innermost digit first), v, k (innermost digit first)
    std::vector<int64_t> ow, vw, kw;
    for (int d = e.nm - 2; d >= 0; --d)
      for (int t = 0; t < e.m_sh[d]; ++t) ow.push_back(e.m_sa[d] << t);
    for (int t = 0; t < e.m_sh[e.nm - 1]; ++t) vw.push_back(e.m_sa[e.nm - 1] << t);
    for (int d = e.nk - 1; d >= 0; --d)
      for (int t = 0; t < e.k_sh[d]; ++t) kw.push_back(e.k_sa[d] << t);
    const int nb = (int)(ow.size() + vw.size() + kw.size());
    if ((int64_t(1) << nb) != e.M * e.K) return false;
    std::vector<int> bitof(nb, -1);            // X offset bit -> role slot
    auto place = [&](int64_t w) -> int {
      if (!p2(w)) return -1;
      const int b = lg(w);
      if (b >= nb || bitof[b] >= 0) return -1;
      bitof[b] = 1;
      return b;
    };
    std::vector<int> ob, vb, kb;
    for (int64_t w : ow) { const int b = place(w); if (b < 0) return false; ob.push_back(b); }
    for (int64_t w : vw) { const int b = place(w); if (b < 0) return false; vb.push_back(b); }
    for (int64_t w : kw) { const int b = place(w); if (b < 0) return false; kb.push_back(b); }
    if (i == 0) {
      prev.resize(nb);
      for (int b = 0; b < nb; ++b) prev[b] = next_gid++;
      tens.push_back(prev);
    } else if ((int)prev.size() != nb) {
      return false;                            // X is not exactly the previous output
    }
    for (int b : kb) { kg[i].push_back(prev[b]); inU[prev[b]] = 1; }
    for (int b : vb) pog[i].push_back(prev[b]);
    for (int b : ob) pog[i].push_back(prev[b]);
    std::vector<int> out;                      // [o][n][v]: v bits, n bits, o bits
    for (int b : vb) out.push_back(prev[b]);
    for (int t = 0; t < lg(e.N); ++t) {
      const int g = next_gid++;
      if (g >= 4096) return false;
      inU[g] = 1;
      ng[i].push_back(g);
      out.push_back(g);
    }
    for (int b : ob) out.push_back(prev[b]);
    tens.push_back(out);
    prev = out;
  }
  // working-set index of each tensor: its touched gids in offset-bit order
  std::vector<std::vector<int>> widx(L + 1);
  std::vector<std::unordered_map<int, int>> wpos(L + 1);
  int wmax_a = 0, wmax_b = 0;
  for (int i = 0; i <= L; ++i) {
    for (int g : tens[i]) if (inU[g]) { wpos[i][g] = (int)widx[i].size(); widx[i].push_back(g); }
    if ((int)widx[i].size() > maxbits) return false;
    if (i % 2 == 0) wmax_a = std::max(wmax_a, (int)widx[i].size());
    else wmax_b = std::max(wmax_b, (int)widx[i].size());
  }
  // lanes: the 5 lowest-weight carry bits of T0 (ideally T0's and TL's offset bits 0-4:
  // unit-stride lanes at both ends; otherwise the lanes stride and L1 merges the sectors)
  const std::vector<int>& T0 = tens[0];
  const std::vector<int>& TL = tens[L];
  std::unordered_map<int, int> tl_bit;
  for (int b = 0; b < (int)TL.size(); ++b) tl_bit[TL[b]] = b;
  int nct = 0, nl = 0;
  for (int b = 0; b < (int)T0.size(); ++b) {
    if (inU[T0[b]]) continue;
    auto it = tl_bit.find(T0[b]);
    if (it == tl_bit.end()) return false;
    if (nl < 5) {
      cd.lw_src[nl] = int64_t(1) << b;
      cd.lw_dst[nl] = int64_t(1) << it->second;
      ++nl;
      continue;
    }
    if (nct >= 32) return false;
    cd.ct_src[nct] = int64_t(1) << b;
    cd.ct_dst[nct] = int64_t(1) << it->second;
    ++nct;
  }
  if (nl < 5) return false;
  // both ends must stay reasonably local: a 32-lane access spans <= 8 KiB (the tile's other
  // touched elements fill the rest of those sectors from L1)
  if (cd.lw_src[4] > 512 || cd.lw_dst[4] > 512) return false;
  cd.nct = nct;
  cd.n_tiles = int64_t(1) << nct;
  cd.L = L;
  cd.a0 = (int)widx[0].size();
  cd.aL = (int)widx[L].size();
  cd.buf_a = 1 << wmax_a;
  cd.buf_b = 1 << wmax_b;
  tab.clear();
  std::unordered_map<int, int> t0_bit;
  for (int b = 0; b < (int)T0.size(); ++b) t0_bit[T0[b]] = b;
  for (int x = 0; x < (1 << cd.a0); ++x) {     // t0off
    int64_t o = 0;
    for (int j = 0; j < cd.a0; ++j) if ((x >> j) & 1) o += int64_t(1) << t0_bit[widx[0][j]];
    if (o > INT32_MAX) return false;
    tab.push_back((int32_t)o);
  }
  for (int x = 0; x < (1 << cd.aL); ++x) {     // tLoff
    int64_t o = 0;
    for (int j = 0; j < cd.aL; ++j) if ((x >> j) & 1) o += int64_t(1) << tl_bit[widx[L][j]];
    if (o > INT32_MAX) return false;
    tab.push_back((int32_t)o);
  }
  for (int i = 0; i < L; ++i) {
    const tn::EinsumDesc& e = *es[i];
    tn::ChainStep& st = cd.st[i];
    std::vector<int> pt;                       // touched o / v ids: the o-positions
    for (int g : pog[i]) if (inU[g]) pt.push_back(g);
    st.N = (int32_t)e.N;
    st.K = (int32_t)e.K;
    st.P = 1 << (int)pt.size();
    st.in_buf = i % 2;
    st.tab = (int32_t)tab.size();
    auto wsum = [&](int x, const std::vector<int>& gids, const std::unordered_map<int, int>& pos) {
      int32_t o = 0;
      for (size_t j = 0; j < gids.size(); ++j) if ((x >> j) & 1) o += 1 << pos.at(gids[j]);
      return o;
    };
    for (int x = 0; x < st.P; ++x) tab.push_back(wsum(x, pt, wpos[i]));          // in_p
    for (int x = 0; x < st.P; ++x) tab.push_back(wsum(x, pt, wpos[i + 1]));      // out_p
    for (int x = 0; x < st.K; ++x) tab.push_back(wsum(x, kg[i], wpos[i]));       // in_k
    for (int x = 0; x < st.N; ++x) tab.push_back(wsum(x, ng[i], wpos[i + 1]));   // out_n
    for (int n = 0; n < st.N; ++n)                                               // yoff[n][k]
      for (int k = 0; k < st.K; ++k) {
        int64_t o = 0, t = n;
        for (int d = e.nn - 1; d >= 0; --d) { o += (t & ((int64_t(1) << e.n_sh[d]) - 1)) * e.n_sb[d]; t >>= e.n_sh[d]; }
        t = k;
        for (int d = e.nk - 1; d >= 0; --d) { o += (t & ((int64_t(1) << e.k_sh[d]) - 1)) * e.k_sb[d]; t >>= e.k_sh[d]; }
        if (o > INT32_MAX) return false;
        tab.push_back((int32_t)o);
      }
  }
  cd.n_tab = (int32_t)tab.size();
  return tn::chain_smem_bytes(cd) <= 110 * 1024;
}

void contiguous_strides(std::vector<VDim>& d) {
  int64_t s = 1;
  for (int p = (int)d.size() - 1; p >= 0; --p) {
    d[p].stride = s;
    s *= d[p].ext;
  }
}

// first-fit arena with liveness
struct Arena {
  std::vector<std::pair<int64_t, int64_t>> used;   // (offset, size), sorted
  int64_t high = 0;
  static int64_t align(int64_t x) { return (x + 31) & ~int64_t(31); }   // 256 B for complex64
  int64_t alloc(int64_t n) {
    n = align(std::max<int64_t>(n, 1));
    int64_t at = 0;
    size_t pos = 0;
    for (; pos < used.size(); ++pos) {
      if (used[pos].first - at >= n) break;
      at = align(used[pos].first + used[pos].second);
    }
    used.insert(used.begin() + pos, {at, n});
    high = std::max(high, at + n);
    return at;
  }
  void release(int64_t off) {
    for (size_t p = 0; p < used.size(); ++p)
      if (used[p].first == off) {
        used.erase(used.begin() + p);
        return;
      }
  }
};

int env_int(const char* name, int dflt) {
  const char* v = getenv(name);
  return v ? atoi(v) : dflt;
}

// ---------------------------------------------------------------- planning

// The paper's top-k index-reordering rule (§4.1, Fig. 3), on a label
// replay of the path: (1) rank all contractions by T_cc (Eq. 4; ties: earlier step
// first), keep the top k; (2) a contraction qualifies when no reordering has modified
// it (its [J][P][Q] output is then GEMM-form, so reordering its inputs alone makes it a
// GEMM); (3) the contractions that produced its two inputs ("associated", L337) must
// not have been modified either (a leaf input has none); (4) reorder: the current and
// the associated contractions are marked modified.  Sets c->reorder_sel / reorder_mod.
void paper_reorder(tn_ctx* c, const std::unordered_map<int, View>& live0, int topk) {
  const int n_steps = (int)c->path.size();
  struct T { std::vector<std::pair<int64_t, int64_t>> d; std::vector<int> q; int64_t G = 1; int prod = -1; };
  std::unordered_map<int, T> st;
  for (auto& kv : live0) {
    T t;
    for (auto& d : kv.second.dims) if (d.label != GROUP) t.d.push_back({d.label, d.ext});
    t.q = kv.second.q;
    t.G = kv.second.has_group() ? (int64_t)kv.second.table.size() : 1;
    st[kv.first] = t;
  }
  std::vector<unsigned __int128> w(n_steps);   // J*m*n*k (T_cc / 8), exact
  std::vector<std::array<int, 2>> prod(n_steps);
  for (int s = 0; s < n_steps; ++s) {
    T& A = st[c->path[s].first];
    T& B = st[c->path[s].second];
    prod[s] = {A.prod, B.prod};
    unsigned __int128 m = 1, n = 1, k = 1, J = 1;
    T out;
    for (auto& a : A.d) {
      bool shared = false;
      for (auto& b : B.d) shared = shared || b.first == a.first;
      if (shared) k *= (unsigned __int128)a.second; else { m *= (unsigned __int128)a.second; out.d.push_back(a); }
    }
    for (auto& b : B.d) {
      bool shared = false;
      for (auto& a : A.d) shared = shared || a.first == b.first;
      if (!shared) { n *= (unsigned __int128)b.second; out.d.push_back(b); }
    }
    if (!A.q.empty() && !B.q.empty()) {
      out.q = A.q;
      out.q.insert(out.q.end(), B.q.begin(), B.q.end());
      std::sort(out.q.begin(), out.q.end());
      out.G = (int64_t)table_for(c, out.q).size();
      J = (unsigned __int128)out.G;
    } else if (!A.q.empty()) {
      m *= (unsigned __int128)A.G; out.q = A.q; out.G = A.G;
    } else if (!B.q.empty()) {
      n *= (unsigned __int128)B.G; out.q = B.q; out.G = B.G;
    }
    w[s] = J * m * n * k;
    out.prod = s;
    st.erase(c->path[s].second);
    st[c->path[s].first] = out;
  }
  std::vector<int> rank(n_steps);
  std::iota(rank.begin(), rank.end(), 0);
  std::stable_sort(rank.begin(), rank.end(), [&](int a, int b) { return w[a] > w[b]; });
  for (int r = 0; r < std::min(topk, n_steps); ++r) {
    const int s = rank[r];
    if (c->reorder_mod[s]) continue;                              // (2) modified already
    bool ok = true;
    for (int p : prod[s]) if (p >= 0 && c->reorder_mod[p]) ok = false;
    if (!ok) continue;                                            // (3) an associated one is
    c->reorder_sel[s] = 1;                                        // (4) reorder
    c->reorder_mod[s] = 1;
    for (int p : prod[s]) if (p >= 0) c->reorder_mod[p] = 1;
  }
}

tn_status build_plan(tn_ctx* c) {
  free_dev(c);
  c->device_bytes = c->leaf_elems * sizeof(float2);
  const int tc_big = env_int("TN_TC_MIN_BIG", 128);
  const int tc_small = env_int("TN_TC_MIN_SMALL", 16);
  const int tc_k = env_int("TN_TC_MIN_K", 16);
  const int disable_tc = env_int("TN_DISABLE_TC", 0);
  const int skinny_big = env_int("TN_SKINNY_MIN_BIG", 1024);
  const int dot_min_k = env_int("TN_DOT_MIN_K", 4096);
  const int dot_max_out = env_int("TN_DOT_MAX_OUT", 4096);
  const int tc_deep_k = env_int("TN_TC_DEEP_K", 1024);
  const int64_t tc_out_min = env_int("TN_TC_OUT_MIN", 1 << 20);   // 0: never (see below)
  const int tc_out_side = env_int("TN_TC_OUT_SIDE", 32);
  const int wdot_min_k = env_int("TN_WDOT_MIN_K", 256);    // SIMT mode 4 (warp dot) from this K
  const int skinny_max_small = env_int("TN_SKINNY_MAX_SMALL", 64);
  const int prep_force = env_int("TN_PREP_FORCE", -1);   // tests: force a prep kernel kind
  const int group_mode = env_int("TN_GROUP", 1);          // 0 off, 1 cost model, 2 always
  const double group_max_bytes = 1e9 * env_int("TN_GROUP_MAX_GB", 32);
  const int group_min_use = env_int("TN_GROUP_MIN_USE", 8);   // route when useful >= 1/this
  const int pair_min_m = tn::g_knobs.pair_min_m;            // CTA-pair GEMM for M >= this
  const int out_layout = env_int("TN_OUT_LAYOUT", 1);      // 1: [P keep][Q keep][con] for TC steps
  const int fuse_planes = env_int("TN_FUSE_PLANES", 1);    // producer epilogue writes consumer planes
  const int plane_v16 = env_int("TN_PLANE_V16", 1);       // 256-bit plane stores where 16 columns are contiguous
  const int wd_staged = env_int("TN_WD_STAGED", 1);       // mode-4 merges: slab-staged warp dot where eligible
  const int gate_regroup = env_int("TN_GATE_REGROUP", 1);  // gate-folded prep: regrouped compute phase
  const int dense_mode = env_int("TN_DENSE_MERGE", 1);     // 0 off, 1 cost rule, 2 always (tests)
  // skinny steps folded into TC preps; gates with K > 8 stay separate
  // (their gate-prep is slower than skinny kernel + transposer on C4)
  const int fold_gates = env_int("TN_FOLD_GATES", 1);
  const int fold_maxk = env_int("TN_FOLD_MAXK", 8), fold_maxn = env_int("TN_FOLD_MAXN", 65535);
  const int wave_sync = env_int("TN_WAVE_SYNC", 1);        // GEMM wave synchronisation (L2 reuse)
  const int wave_min_k = env_int("TN_WAVE_MIN_K", 1024);   // ... for GEMMs with K >= this
  const int cols_single = env_int("TN_COLS_SINGLE", 1);    // strided single-dim column fast path
                                                           // (2: column-contiguous case only)
  const int n_leaves = c->n_tensors;
  const int n_steps = (int)c->path.size();

  // leaf views with sliced bonds removed; dynamic offset terms
  std::unordered_map<int64_t, int> slice_pos;
  for (size_t p = 0; p < c->sliced.size(); ++p) slice_pos[c->sliced[p]] = (int)p;
  std::vector<int32_t> term_leaf, term_p;
  std::vector<int64_t> term_stride;
  std::unordered_map<int, View> live;
  for (int t = 0; t < n_leaves; ++t) {
    View v = c->leaf_views[t];
    std::vector<VDim> kept;
    for (auto& d : v.dims) {
      auto it = slice_pos.find(d.label);
      if (it != slice_pos.end()) {
        term_leaf.push_back(t);
        term_p.push_back(it->second);
        term_stride.push_back(d.stride);
      } else {
        kept.push_back(d);
      }
    }
    v.dims = kept;
    v.absmax_slot = t;
    live[t] = v;
  }

  // Consumer look-ahead (index reordering, §4.1, generalised to
  // every step): for each step's output, the bonds its consumer will contract.
  // Producers place those bonds last (sorted), so the consumer's operand prep
  // reads long contiguous runs.
  std::vector<std::unordered_set<int64_t>> consumer_k(n_steps);
  std::vector<int> consumer_step(n_steps, -1);
  // K order of a step's operands (outer -> inner labels), chosen by the tensor-core
  // producer of one operand so that its epilogue can write the operand's fp16 planes
  // in 16-B vectors; default: sorted by label
  std::vector<std::vector<int64_t>> korder(n_steps);
  // per step: log2-ish size of its output and the producer / size of its consumer's other
  // operand, so that the producer of a consumer's BIGGER operand fixes the K order (its
  // planes are the ones worth writing from the epilogue; the small side is transposed)
  std::vector<double> out_size(n_steps, 0.0), other_size(n_steps, 0.0);
  std::vector<int> other_prod(n_steps, -1);
  {
    std::vector<std::unordered_set<int64_t>> lab(n_leaves);
    std::vector<int> producer(n_leaves, -1);
    for (int t = 0; t < n_leaves; ++t)
      for (auto& d : live[t].dims)
        if (d.label != GROUP) lab[t].insert(d.label);
    auto size_of = [&](const std::unordered_set<int64_t>& L) {
      double z = 1.0;
      for (int64_t x : L) { auto it = c->dim_of.find(x); if (it != c->dim_of.end()) z *= (double)it->second; }
      return z;
    };
    for (int s = 0; s < n_steps; ++s) {
      const int i = c->path[s].first, j = c->path[s].second;
      std::unordered_set<int64_t> shared;
      for (int64_t x : lab[i]) if (lab[j].count(x)) shared.insert(x);
      const double zi = size_of(lab[i]), zj = size_of(lab[j]);
      if (producer[i] >= 0) { other_prod[producer[i]] = producer[j]; other_size[producer[i]] = zj; }
      if (producer[j] >= 0) { other_prod[producer[j]] = producer[i]; other_size[producer[j]] = zi; }
      if (producer[i] >= 0) { consumer_k[producer[i]] = shared; consumer_step[producer[i]] = s; }
      if (producer[j] >= 0) { consumer_k[producer[j]] = shared; consumer_step[producer[j]] = s; }
      std::unordered_set<int64_t> out;
      for (int64_t x : lab[i]) if (!shared.count(x)) out.insert(x);
      for (int64_t x : lab[j]) if (!shared.count(x)) out.insert(x);
      lab[i] = out;
      lab[j].clear();
      producer[i] = s;
      out_size[s] = size_of(out);
    }
  }
  const int korder_big = env_int("TN_KORDER_BIG", 1);   // 0: the first producer decides (round 1-2)
  // Which producers write their output in the consumer's order (index reordering).
  c->reorder_mode = env_int("TN_REORDER", 2);
  c->reorder_topk = env_int("TN_REORDER_TOPK", 10);
  c->reorder_sel.assign(n_steps, 0);
  c->reorder_mod.assign(n_steps, 0);
  if (c->reorder_mode == 1) paper_reorder(c, live, c->reorder_topk);
  for (int s = 0; s < n_steps; ++s) {
    const bool keep = c->reorder_mode == 2 ||
                      (c->reorder_mode == 1 && consumer_step[s] >= 0 && c->reorder_sel[consumer_step[s]]);
    if (!keep) consumer_k[s].clear();
  }
  // stable partition: bonds the consumer keeps first, bonds it contracts last (sorted)
  auto consumer_order = [](std::vector<VDim>& d, const std::unordered_set<int64_t>& kc) {
    std::vector<VDim> keep, con;
    for (auto& x : d) (kc.count(x.label) ? con : keep).push_back(x);
    std::sort(con.begin(), con.end(), [](const VDim& a, const VDim& b) { return a.label < b.label; });
    keep.insert(keep.end(), con.begin(), con.end());
    d.swap(keep);
  };

  Arena arena;
  std::vector<std::vector<int64_t>> deferred(n_steps);   // arena releases moved to a later step
  std::unordered_set<int> unalloc;                         // live ids = unmaterialised folded outputs
  auto folded_out = [&](int id) { return unalloc.count(id) > 0; };
  std::vector<int32_t> tables;
  int64_t scratch = 0;
  c->steps.clear();
  c->flops_per_slice = c->tc_flops = c->bytes_per_slice = c->peak = 0;
  for (auto& kv : live) c->peak = std::max(c->peak, (double)kv.second.size());
  int n_einsum = 0, n_prep = 0;
  int64_t partial_elems = 0;

  for (int s = 0; s < n_steps; ++s) {
    StepPlan sp;
    sp.i = c->path[s].first;
    sp.j = c->path[s].second;
    sp.final_step = (s == n_steps - 1);
    View A = live[sp.i], B = live[sp.j];
    sp.in_slot[0] = A.absmax_slot;
    sp.in_slot[1] = B.absmax_slot;
    // Eq. 3 set rule: δ = shared bond labels, γ = the rest
    std::unordered_set<int64_t> lb;
    for (auto& d : B.dims) if (d.label != GROUP) lb.insert(d.label);
    std::vector<VDim> Kd_A, Kd_B, FA, FB;
    std::unordered_set<int64_t> kset;
    for (auto& d : A.dims)
      if (d.label != GROUP && lb.count(d.label)) { Kd_A.push_back(d); kset.insert(d.label); }
    for (auto& d : A.dims) if (!(d.label != GROUP && kset.count(d.label))) FA.push_back(d);
    for (auto& d : Kd_A)
      for (auto& e : B.dims) if (e.label == d.label) Kd_B.push_back(e);
    for (auto& d : B.dims) if (!(d.label != GROUP && kset.count(d.label))) FB.push_back(d);
    sp.merge = A.has_group() && B.has_group();
    VDim gA{GROUP, 1, 0}, gB{GROUP, 1, 0};
    View out;
    if (sp.merge) {
      // Eq. 7: merged configurations = unique sample projections onto qA ∪ qB
      for (auto it = FA.begin(); it != FA.end(); ++it) if (it->label == GROUP) { gA = *it; FA.erase(it); break; }
      for (auto it = FB.begin(); it != FB.end(); ++it) if (it->label == GROUP) { gB = *it; FB.erase(it); break; }
      std::vector<int> q = A.q;
      q.insert(q.end(), B.q.begin(), B.q.end());
      std::sort(q.begin(), q.end());
      std::vector<uint64_t> tq = table_for(c, q);
      // map each merged config to its projections (from the samples: the map is a function)
      std::unordered_map<uint64_t, std::pair<uint64_t, uint64_t>> proj;
      proj.reserve(tq.size() * 2);
      for (uint64_t smp : c->packed)
        proj.emplace(project(smp, q, c->n_open),
                     std::make_pair(project(smp, A.q, c->n_open), project(smp, B.q, c->n_open)));
      sp.ia.resize(tq.size());
      sp.ib.resize(tq.size());
      for (size_t f = 0; f < tq.size(); ++f) {
        auto pr = proj[tq[f]];
        int64_t a = index_in(A.table, pr.first), b = index_in(B.table, pr.second);
        if (a < 0 || b < 0) return fail(TN_ERR_INTERNAL, "merge table lookup failed");
        sp.ia[f] = (int32_t)a;
        sp.ib[f] = (int32_t)b;
      }
      sp.J = (int64_t)tq.size();
      out.q = q;
      out.table = tq;
    } else if (A.has_group()) {
      out.q = A.q;
      out.table = A.table;
    } else if (B.has_group()) {
      out.q = B.q;
      out.table = B.table;
    }
    for (auto& d : FA) sp.m *= d.ext;
    for (auto& d : FB) sp.n *= d.ext;
    for (auto& d : Kd_A) sp.k *= d.ext;
    sp.tcc = 8.0 * (double)sp.J * (double)sp.m * (double)sp.n * (double)sp.k;   // Eq. 4
    const int64_t out_elems = sp.J * sp.m * sp.n;
    sp.tmc = 8.0 * ((double)A.size() + (double)B.size() + (double)out_elems);    // Eq. 5
    c->flops_per_slice += sp.tcc;
    c->bytes_per_slice += sp.tmc;
    c->peak = std::max(c->peak, (double)out_elems);

    const int64_t big = std::max(sp.m, sp.n), small = std::min(sp.m, sp.n);
    // tensor cores for GEMM-shaped steps; a deep K (>= tc_deep_k) keeps a step on the
    // tensor cores even with a narrow side: it is bound by streaming the big operand
    // once, which the TMA pipeline does at HBM speed (padding N only costs MMA slots).
    sp.tc = !disable_tc && big >= tc_big && sp.k >= tc_k &&
            (small >= tc_small || sp.k >= tc_deep_k) && !sp.final_step &&
            sp.m < INT32_MAX && sp.n < INT32_MAX && sp.k < INT32_MAX && sp.J < INT32_MAX;
    sp.swap = sp.tc && sp.n > sp.m;   // tensor-core M side = larger free extent
    if (sp.merge && sp.J > 1 && group_mode > 0 && !disable_tc && !sp.final_step &&
        sp.k >= tc_k && sp.k < INT32_MAX) {
      // Slab-grouped merge: with X the side whose slab is shared and Y the other, the
      // batches j with slabX(j) = a form one GEMM  C[(j,y)][x] = Σ_k Y'[(j,y)][k] X[a][x][k]
      // whose rows are Y's gathered rows.  Worth it when the per-batch tiles are mostly
      // padding (a narrow free side) and the batches share few X slabs; it also moves
      // merges too narrow per batch for the tensor cores onto them.
      auto tiles_for = [&](const std::vector<int32_t>& sx, int64_t GX, int64_t P, int64_t Q,
                           int64_t& rows) {
        std::vector<int64_t> cnt((size_t)GX, 0);
        for (int32_t a : sx) cnt[a]++;
        rows = 0;
        for (int64_t n_ : cnt) rows += (n_ * Q + 127) / 128 * 128;
        return rows / 128 * ((P + 127) / 128);
      };
      int64_t rA = 0, rB = 0;
      const int64_t tA = tiles_for(sp.ia, gA.ext, sp.m, sp.n, rA);   // X = A, Y = B
      const int64_t tB = tiles_for(sp.ib, gB.ext, sp.n, sp.m, rB);   // X = B, Y = A
      const int64_t cur = sp.J * ((sp.m + 127) / 128) * ((sp.n + 127) / 128);
      const bool xa = tA <= tB;
      const int64_t t = xa ? tA : tB, rows = xa ? rA : rB;
      const int64_t kpad = (sp.k + 7) / 8 * 8;
      // useful fraction of the grouped GEMM's MMA work
      const double useful = (double)sp.J * sp.m * sp.n / ((double)t * 128.0 * 128.0);
      const bool want = sp.tc ? (group_mode == 2 || 5 * t < 4 * cur)
                              : (group_mode == 2 || useful * group_min_use >= 1.0);
      if (want && rows < INT32_MAX &&
          sp.J * (xa ? sp.n : sp.m) < INT32_MAX &&
          (double)rows * kpad * 8.0 <= group_max_bytes) {
        sp.grouped = true;
        sp.tc = true;
        sp.swap = xa;                 // tensor-core M side (prep side 0) = Y
        sp.g_rows = rows;
        const std::vector<int32_t>& sx = xa ? sp.ia : sp.ib;
        const int64_t GX = xa ? gA.ext : gB.ext;
        const int64_t Q = xa ? sp.n : sp.m;      // Y's free extent
        std::vector<std::vector<int32_t>> members((size_t)GX);
        for (int64_t j = 0; j < sp.J; ++j) members[sx[j]].push_back((int32_t)j);
        sp.g_rowmap.assign((size_t)rows, -1);
        sp.g_blk.assign((size_t)(rows / 128), 0);
        int64_t r = 0;
        for (int64_t a = 0; a < GX; ++a) {
          if (members[a].empty()) continue;
          const int64_t r0 = r;
          for (int32_t j : members[a])
            for (int64_t q = 0; q < Q; ++q) sp.g_rowmap[r++] = (int32_t)(j * Q + q);
          r = r0 + ((r - r0) + 127) / 128 * 128;
          for (int64_t b_ = r0 / 128; b_ < r / 128; ++b_) sp.g_blk[b_] = (int32_t)a;
        }
      }
    }
    if (sp.merge && sp.J > 1 && !sp.grouped && dense_mode > 0 && !disable_tc && !sp.final_step &&
        sp.k >= tc_k && sp.k < INT32_MAX) {
      auto p2 = [](int64_t x) { return x > 0 && (x & (x - 1)) == 0; };
      const double slabs = (double)gA.ext * (double)gB.ext;
      const bool narrow = !sp.tc || std::min(sp.m, sp.n) < 128;   // batched tiles mostly padding
      if ((dense_mode == 2 || (narrow && (double)sp.J >= 0.5 * slabs)) && p2(sp.m) && p2(sp.n) &&
          gA.ext * sp.m < INT32_MAX && gB.ext * sp.n < INT32_MAX && slabs < 1e8 &&
          (dense_mode == 2 || std::max(gA.ext * sp.m, gB.ext * sp.n) >= 128)) {
        sp.dense_merge = true;
        sp.tc = true;
        sp.swap = gB.ext * sp.n > gA.ext * sp.m;   // M side = the larger dense extent
        const int64_t G0 = sp.swap ? gB.ext : gA.ext, G1 = sp.swap ? gA.ext : gB.ext;
        sp.pair_map.assign((size_t)(G0 * G1), -1);
        for (int64_t j = 0; j < sp.J; ++j) {
          const int64_t s0 = sp.swap ? sp.ib[j] : sp.ia[j], s1 = sp.swap ? sp.ia[j] : sp.ib[j];
          sp.pair_map[s0 * G1 + s1] = (int32_t)j;
        }
      }
    }

    // output layout: [J][P dims][Q dims], P = A side unless swapped
    // SIMT mode (see kernels.cu): 2 = split-K dot, 1 = skinny (one small operand)
    if (!sp.tc) {
      const int64_t outs = sp.J * sp.m * sp.n;
      auto skinny = [&](int64_t big, int64_t small) {
        return big >= skinny_big && small <= skinny_max_small && small * sp.k <= 8192 && sp.k <= 256;
      };
      const bool one_batch = !sp.merge || sp.J == 1;   // J = 1 merges fold their slabs
      // batched skinny (J > 1 merges): every slab of the small side staged in smem
      auto batched_skinny = [&](int64_t big, int64_t small, int64_t gsmall) {
        return sp.merge && sp.J > 1 && skinny(big, small) && gsmall * ((small + 1) & ~1) * sp.k <= 8192;
      };
      if (outs <= dot_max_out && sp.k >= dot_min_k) {
        sp.mode = 2;
        partial_elems = std::max(partial_elems, 2 * outs);
      } else if (sp.merge && sp.J > 1 && sp.n <= 32 && sp.k >= wdot_min_k) {
        sp.mode = 4;                  // batched merge, tiny outputs per batch, long K
      } else if ((one_batch && skinny(sp.m, sp.n)) || batched_skinny(sp.m, sp.n, gB.ext)) {
        sp.mode = 1;
        sp.x_is_b = false;
      } else if ((one_batch && skinny(sp.n, sp.m)) || batched_skinny(sp.n, sp.m, gA.ext)) {
        sp.mode = 1;
        sp.x_is_b = true;
      } else if (one_batch) {
        // wide skinny: outer-product-like (k <= 16), small side up to 4096
        auto wide = [&](int64_t big, int64_t small) {
          return big >= skinny_big && big >= small && small * sp.k <= 8192 && sp.k <= 16;
        };
        if (wide(sp.m, sp.n)) {
          sp.mode = 3;
          sp.x_is_b = false;
        } else if (wide(sp.n, sp.m)) {
          sp.mode = 3;
          sp.x_is_b = true;
        }
      }
    }
    // A step left to the general SIMT kernel (mode 0: one thread per output with a full
    // index decomposition) whose output is large and whose free sides are both GEMM-sized
    // -- e.g. a batched merge with a tiny K (C4-sparse: J = 32 batches of 4096 x 2048,
    // K = 4) -- runs on the tensor cores instead: the GEMM streams its output from TMEM
    // (K is zero-padded to one k-block; the MMA work is negligible next to the stores).
    if (!sp.tc && sp.mode == 0 && !disable_tc && !sp.final_step && tc_out_min > 0 &&
        sp.J * sp.m * sp.n >= tc_out_min && std::min(sp.m, sp.n) >= tc_out_side && std::max(sp.m, sp.n) >= tc_big &&
        sp.m < INT32_MAX && sp.n < INT32_MAX && sp.J < INT32_MAX) {
      sp.tc = true;
      sp.swap = sp.n > sp.m;
    }
    std::vector<VDim> od;
    const auto& kc = consumer_k[s];
    if (sp.mode == 1 || sp.mode == 3) {
      // output [J][X outer dims][Y dims][v], v = the big operand's smallest-stride dim
      if (sp.merge && sp.J > 1) od.push_back({GROUP, sp.J, 0});
      const auto& X = sp.x_is_b ? FB : FA;
      std::vector<VDim> Y = sp.x_is_b ? FA : FB;
      // lane dims v: the contiguous run of X's memory that starts at its smallest
      // stride (lanes then read consecutive addresses); kept innermost in the output
      std::vector<int> vrun;
      int vi = -1;
      for (int p = 0; p < (int)X.size(); ++p)
        if (X[p].ext > 1 && (vi < 0 || X[p].stride < X[vi].stride)) vi = p;
      vrun.push_back(vi);
      for (int64_t next = X[vi].stride * X[vi].ext;;) {
        int q = -1;
        for (int p = 0; p < (int)X.size(); ++p)
          if (X[p].ext > 1 && X[p].stride == next &&
              std::find(vrun.begin(), vrun.end(), p) == vrun.end()) q = p;
        if (q < 0) break;
        vrun.push_back(q);
        next *= X[q].ext;
      }
      sp.vlabels.clear();
      for (int r = (int)vrun.size() - 1; r >= 0; --r) sp.vlabels.push_back(X[vrun[r]].label);
      std::vector<VDim> Xo;
      for (int p = 0; p < (int)X.size(); ++p)
        if (std::find(vrun.begin(), vrun.end(), p) == vrun.end()) Xo.push_back(X[p]);
      consumer_order(Xo, kc);
      consumer_order(Y, kc);
      for (auto& d : Xo) { od.push_back({d.label, d.ext, 0}); sp.order1.push_back(d.label); }
      for (auto& d : Y) { od.push_back({d.label, d.ext, 0}); sp.order2.push_back(d.label); }
      for (int r = (int)vrun.size() - 1; r >= 0; --r)
        od.push_back({X[vrun[r]].label, X[vrun[r]].ext, 0});
    } else {
      if (sp.merge) od.push_back({GROUP, sp.J, 0});
      std::vector<VDim> P = sp.swap ? FB : FA;
      std::vector<VDim> Q = sp.swap ? FA : FB;
      consumer_order(P, kc);
      consumer_order(Q, kc);
      for (auto& d : P) sp.order1.push_back(d.label);
      for (auto& d : Q) sp.order2.push_back(d.label);
      // tensor-core producers write [P keep][Q keep][contracted by the consumer, sorted
      // by label]: the consumer's operand is then K-contiguous in the canonical (sorted)
      // K order, so its prep is a streaming copy instead of a transpose
      auto p2 = [](int64_t x) { return x > 0 && (x & (x - 1)) == 0; };
      bool gen = sp.tc && !sp.grouped && !sp.dense_merge && out_layout && !kc.empty();
      for (auto& d : P) gen = gen && p2(d.ext);
      for (auto& d : Q) gen = gen && p2(d.ext);
      if (gen) {
        std::vector<VDim> con, conp, conq;
        for (auto& d : P) (kc.count(d.label) ? conp : od).push_back({d.label, d.ext, 0});
        for (auto& d : Q) (kc.count(d.label) ? conq : od).push_back({d.label, d.ext, 0});
        auto by_label = [](const VDim& a, const VDim& b) { return a.label < b.label; };
        std::sort(conp.begin(), conp.end(), by_label);
        std::sort(conq.begin(), conq.end(), by_label);
        // innermost: the consumer-contracted bonds of one side (>= 8 elements if possible:
        // 16-B plane vectors along columns (Q) or rows (P) of this GEMM's tile)
        int64_t ep = 1, eq = 1;
        for (auto& d : conp) ep *= d.ext;
        for (auto& d : conq) eq *= d.ext;
        const bool q_inner = eq >= 8 || ep < 8;
        for (auto& d : (q_inner ? conp : conq)) con.push_back(d);
        for (auto& d : (q_inner ? conq : conp)) con.push_back(d);
        // a later producer of the consumer's >= 4x bigger operand decides instead
        const bool defer = korder_big && other_prod[s] > s && other_size[s] >= 4.0 * out_size[s];
        if (consumer_step[s] >= 0 && !defer) {
          std::vector<int64_t>& ko = korder[consumer_step[s]];
          if (ko.empty()) {            // the consumer's first tensor-core producer decides
            for (auto& d : con) ko.push_back(d.label);
          } else {                     // the other operand follows it (same K order)
            auto rank = [&](int64_t l) {
              for (size_t q = 0; q < ko.size(); ++q) if (ko[q] == l) return (int64_t)q;
              return (int64_t)ko.size();
            };
            std::stable_sort(con.begin(), con.end(),
                             [&](const VDim& x, const VDim& y) { return rank(x.label) < rank(y.label); });
          }
        }
        od.insert(od.end(), con.begin(), con.end());
        std::vector<VDim> tmp = od;
        contiguous_strides(tmp);
        auto ostride = [&](int64_t l) {
          for (auto& d : tmp) if (d.label == l) return d.stride;
          return (int64_t)0;
        };
        sp.po.clear();
        sp.qo.clear();
        for (auto& d : P) sp.po.push_back({d.label, d.ext, ostride(d.label)});
        for (auto& d : Q) sp.qo.push_back({d.label, d.ext, ostride(d.label)});
        coalesce1(sp.po);
        coalesce1(sp.qo);
        const bool plain = sp.po.size() <= 1 && sp.qo.size() == 1 && sp.qo[0].stride == 1 &&
                           (sp.po.empty() || sp.po[0].stride == sp.qo[0].ext);
        if (sp.po.size() > 16 || sp.qo.size() > 16 || plain) {
          gen = false;     // plain [P][Q] layout (or too many dims): the fixed epilogue
          od.resize(sp.merge ? 1 : 0);
        }
      }
      sp.out_gen = gen;
      if (!gen)
        for (auto& d : P) od.push_back({d.label, d.ext, 0});
      if (!gen)
        for (auto& d : Q) od.push_back({d.label, d.ext, 0});
    }
    contiguous_strides(od);
    out.dims = od;
    out.buf = 1;
    out.absmax_slot = n_leaves + s;

    if (sp.merge) {
      sp.ia_off = (int64_t)tables.size();
      tables.insert(tables.end(), sp.ia.begin(), sp.ia.end());
      sp.ib_off = (int64_t)tables.size();
      tables.insert(tables.end(), sp.ib.begin(), sp.ib.end());
    }
    if (sp.merge && !sp.tc && sp.mode == 4 && sp.J > 1) {
      // batches grouped by their B slab (CSR), for the slab-staged warp-dot kernel
      int32_t ns = 0;
      for (int32_t v : sp.ib) ns = std::max(ns, v + 1);
      std::vector<int32_t> start(ns + 1, 0), list(sp.ib.size());
      for (int32_t v : sp.ib) start[v + 1]++;
      for (int32_t q = 0; q < ns; ++q) start[q + 1] += start[q];
      std::vector<int32_t> fill(start.begin(), start.end() - 1);
      for (size_t jj = 0; jj < sp.ib.size(); ++jj) list[fill[sp.ib[jj]]++] = (int32_t)jj;
      sp.wd_nslabs = ns;
      sp.wd_start_off = (int64_t)tables.size();
      tables.insert(tables.end(), start.begin(), start.end());
      sp.wd_list_off = (int64_t)tables.size();
      tables.insert(tables.end(), list.begin(), list.end());
    }
    if (sp.dense_merge) {
      sp.pair_off = (int64_t)tables.size();
      tables.insert(tables.end(), sp.pair_map.begin(), sp.pair_map.end());
    }
    if (sp.grouped) {
      sp.g_rowmap_off = (int64_t)tables.size();
      tables.insert(tables.end(), sp.g_rowmap.begin(), sp.g_rowmap.end());
      sp.g_blk_off = (int64_t)tables.size();
      tables.insert(tables.end(), sp.g_blk.begin(), sp.g_blk.end());
    }
    const bool fold_hinted = s < (int)c->fold_hint.size() && c->fold_hint[s] && consumer_step[s] > s;
    const int chain_at = s < (int)c->chain_hint.size() ? c->chain_hint[s] : -1;
    const bool hinted = fold_hinted || chain_at > s;
    const int keep_to = fold_hinted ? consumer_step[s] : chain_at;   // inputs released there
    if (!sp.final_step) {
      sp.out_elems = out_elems;
      sp.out_off = hinted ? 0 : arena.alloc(out_elems);   // folded / chained: never materialised
      out.off = sp.out_off;
    }
    if (sp.tc) {
      sp.einsum_idx = -1;
      sp.prep_idx = n_prep;
      n_prep += 2;
      sp.Kpad = (sp.k + 7) / 8 * 8;
      sp.R[0] = sp.swap ? sp.n : sp.m;
      sp.R[1] = sp.swap ? sp.m : sp.n;
      sp.G[0] = sp.merge ? (sp.swap ? gB.ext : gA.ext) : 1;
      sp.G[1] = sp.merge ? (sp.swap ? gA.ext : gB.ext) : 1;
      if (sp.grouped) {   // side 0 = the gathered Y' rows, one slab
        sp.R[0] = sp.g_rows;
        sp.G[0] = 1;
      }
      int64_t bytes0 = (4 * sp.G[0] * sp.R[0] * sp.Kpad * 2 + 1023) / 1024 * 1024;
      int64_t bytes1 = (4 * sp.G[1] * sp.R[1] * sp.Kpad * 2 + 1023) / 1024 * 1024;
      scratch = std::max(scratch, bytes0 + bytes1);
      c->tc_flops += sp.tcc;
    } else {
      sp.einsum_idx = n_einsum++;
    }
    // release consumed arena inputs (their only consumer is this step); a folded step's
    // inputs are read by its consumer's prep, so they are released there
    if (hinted) {
      if (A.buf == 1 && !(s > 0 && folded_out(sp.i))) deferred[keep_to].push_back(A.off);
      if (B.buf == 1 && !(s > 0 && folded_out(sp.j))) deferred[keep_to].push_back(B.off);
    } else {
      if (A.buf == 1 && !(s > 0 && folded_out(sp.i))) arena.release(A.off);
      if (B.buf == 1 && !(s > 0 && folded_out(sp.j))) arena.release(B.off);
    }
    for (int64_t off : deferred[s]) arena.release(off);
    unalloc.erase(sp.j);
    if (hinted) unalloc.insert(sp.i); else unalloc.erase(sp.i);
    live.erase(sp.j);
    live[sp.i] = out;
    sp.out = out;
    c->steps.push_back(sp);
  }

  // root
  if (n_steps == 0) return fail(TN_ERR_USAGE, "networks with a single tensor are not supported");
  c->root = c->steps.back().out;
  for (auto& d : c->root.dims)
    if (d.label != GROUP) return fail(TN_ERR_DATA, "bond label left uncontracted at the root");
  if (c->n_open > 0) {
    std::vector<int> all(c->n_open);
    std::iota(all.begin(), all.end(), 0);
    if (c->root.q != all) return fail(TN_ERR_DATA, "root group does not cover all open bonds");
    c->acc_elems = (int64_t)c->root.table.size();
    c->out_pos.resize(c->n_samples);
    for (int64_t s = 0; s < c->n_samples; ++s)
      c->out_pos[s] = (int32_t)index_in(c->root.table, c->packed[s]);
    c->n_out = c->n_samples;
  } else {
    c->acc_elems = 1;
    c->out_pos.assign(1, 0);
    c->n_out = 1;
  }
  c->arena_elems = arena.high;
  c->scratch_bytes = scratch;
  if (c->sliced.size() > 64) return fail(TN_ERR_DATA, "at most 64 sliced bonds");
  cudaStream_t sm = c->stream;
  if (!c->host_only) {   // host-only planners build the descriptors below without CUDA
  // ------------------------------------------------------------ device buffers
  tn_status st;
  if ((st = dev_alloc(c, &c->d_arena, (size_t)std::max<int64_t>(c->arena_elems, 1)))) return st;
  if ((st = dev_alloc(c, &c->d_scratch, (size_t)std::max<int64_t>(scratch, 1024)))) return st;
  if ((st = dev_alloc(c, &c->d_tables, std::max<size_t>(tables.size(), 1)))) return st;
  if ((st = dev_alloc(c, &c->d_acc, (size_t)c->acc_elems))) return st;
  if ((st = dev_alloc(c, &c->d_absmax, (size_t)(n_leaves + n_steps)))) return st;
  if ((st = dev_alloc(c, &c->d_scales, (size_t)(2 * n_steps)))) return st;
  if ((st = dev_alloc(c, &c->d_leaf_off, (size_t)n_leaves))) return st;
  if ((st = dev_alloc(c, &c->d_counter, 1))) return st;
  if ((st = dev_alloc(c, &c->d_out_pos, c->out_pos.size()))) return st;
  if ((st = dev_alloc(c, &c->d_slice_desc, 1))) return st;
  if ((st = dev_alloc(c, &c->d_terms_i, std::max<size_t>(2 * term_leaf.size(), 1)))) return st;
  if ((st = dev_alloc(c, &c->d_terms_s, std::max<size_t>(term_stride.size(), 1)))) return st;
  if ((st = dev_alloc(c, &c->d_einsum, (size_t)std::max(n_einsum, 1)))) return st;
  if ((st = dev_alloc(c, &c->d_prep, (size_t)std::max(n_prep, 1)))) return st;
  if ((st = dev_alloc(c, &c->d_one, 1))) return st;
  if ((st = dev_alloc(c, &c->d_partial, (size_t)std::max<int64_t>(partial_elems, 2)))) return st;
  if ((st = dev_alloc(c, &c->d_hist, (size_t)n_steps))) return st;
  if ((st = dev_alloc(c, &c->d_pexp, (size_t)n_steps))) return st;
  if ((st = dev_alloc(c, &c->d_flag, 1))) return st;
  if ((st = dev_alloc(c, &c->d_wave, 1))) return st;
  if ((st = dev_alloc(c, &c->d_gather, (size_t)std::max<int64_t>(c->n_out, 1)))) return st;
  TN_CUDA(cudaMemsetAsync(c->d_hist, 0, n_steps * sizeof(unsigned), sm));
  TN_CUDA(cudaMemsetAsync(c->d_flag, 0, sizeof(int), sm));
  if (!tables.empty())
    TN_CUDA(cudaMemcpyAsync(c->d_tables, tables.data(), tables.size() * 4, cudaMemcpyHostToDevice, sm));
  TN_CUDA(cudaMemcpyAsync(c->d_out_pos, c->out_pos.data(), c->out_pos.size() * 4,
                          cudaMemcpyHostToDevice, sm));
  TN_CUDA(cudaMemsetAsync(c->d_acc, 0, c->acc_elems * sizeof(double2), sm));
  TN_CUDA(cudaMemsetAsync(c->d_leaf_off, 0, n_leaves * sizeof(int64_t), sm));
  {
    std::vector<unsigned> am(n_leaves + n_steps, 0u);
    for (int t = 0; t < n_leaves; ++t) memcpy(&am[t], &c->leaf_absmax[t], 4);
    TN_CUDA(cudaMemcpyAsync(c->d_absmax, am.data(), am.size() * 4, cudaMemcpyHostToDevice, sm));
    float2 one = make_float2(1.f, 0.f);
    TN_CUDA(cudaMemcpyAsync(c->d_one, &one, sizeof(one), cudaMemcpyHostToDevice, sm));
  }
  // slice descriptor
  {
    tn::SliceDesc sd{};
    sd.n_sliced = (int32_t)c->sliced.size();
    for (size_t p = 0; p < c->sliced.size(); ++p) sd.dims[p] = c->dim_of[c->sliced[p]];
    sd.n_terms = (int32_t)term_leaf.size();
    std::vector<int32_t> ti(term_leaf);
    ti.insert(ti.end(), term_p.begin(), term_p.end());
    if (!ti.empty())
      TN_CUDA(cudaMemcpyAsync(c->d_terms_i, ti.data(), ti.size() * 4, cudaMemcpyHostToDevice, sm));
    if (!term_stride.empty())
      TN_CUDA(cudaMemcpyAsync(c->d_terms_s, term_stride.data(), term_stride.size() * 8,
                              cudaMemcpyHostToDevice, sm));
    sd.term_leaf = c->d_terms_i;
    sd.term_p = c->d_terms_i + term_leaf.size();
    sd.term_stride = c->d_terms_s;
    sd.n_leaves = n_leaves;
    sd.leaf_off = c->d_leaf_off;
    sd.counter = c->d_counter;
    sd.absmax = c->d_absmax;
    sd.absmax_first = n_leaves;
    sd.absmax_count = n_steps;
    sd.hist = c->d_hist;
    sd.pexp = c->d_pexp;
    TN_CUDA(cudaMemcpyAsync(c->d_slice_desc, &sd, sizeof(sd), cudaMemcpyHostToDevice, sm));
  }
  }  // !host_only
  // per-step device descriptors
  std::vector<tn::EinsumDesc> eds(std::max(n_einsum, 1));
  std::vector<tn::PrepDesc> pds(std::max(n_prep, 1));
  std::vector<int64_t> gt_all;             // concatenated GT tables
  std::vector<std::pair<int, int64_t>> gt_ref;   // (prep index, offset in gt_all)
  std::vector<std::pair<int, int64_t>> rw_ref;   // grouped-merge row tables, same pool
  std::vector<std::pair<int, int64_t>> bp_ref;   // bit-permutation tile tables, same pool
  std::vector<std::pair<int, int64_t>> gate_ref;  // gate-folded prep tables, same pool
  auto base_of = [&](const View& v) -> const float2* { return v.buf == 0 ? c->d_leaf : c->d_arena; };
  // rebuild the live views to fill descriptors (same replay as above)
  live.clear();
  for (int t = 0; t < n_leaves; ++t) {
    View v = c->leaf_views[t];
    std::vector<VDim> kept;
    for (auto& d : v.dims) if (!slice_pos.count(d.label)) kept.push_back(d);
    v.dims = kept;
    v.absmax_slot = t;
    live[t] = v;
  }
  char errbuf[256];
  std::unordered_map<int, int> producer_of;     // live tensor id -> producing step
  std::vector<std::array<int, 2>> side_producer(n_steps, {-1, -1});   // per TC side
  std::vector<int> x_producer(n_steps, -1);     // skinny steps: producer of the big operand X
  std::vector<int> y_producer(n_steps, -1);     // ... and of the small operand Y
  for (int s = 0; s < n_steps; ++s) {
    StepPlan& sp = c->steps[s];
    View A = live[sp.i], B = live[sp.j];
    if (!sp.tc && sp.mode == 1) {
      auto it = producer_of.find(sp.x_is_b ? sp.j : sp.i);
      x_producer[s] = it == producer_of.end() ? -1 : it->second;
      auto iy = producer_of.find(sp.x_is_b ? sp.i : sp.j);
      y_producer[s] = iy == producer_of.end() ? -1 : iy->second;
    }
    if (sp.tc)
      for (int side = 0; side < 2; ++side) {
        const int id = ((side == 0) != sp.swap) ? sp.i : sp.j;
        auto it = producer_of.find(id);
        side_producer[s][side] = it == producer_of.end() ? -1 : it->second;
      }
    std::unordered_set<int64_t> lb;
    for (auto& d : B.dims) if (d.label != GROUP) lb.insert(d.label);
    std::vector<VDim> FA, FB;
    std::vector<KDim> K;
    std::unordered_set<int64_t> kset;
    VDim gA{GROUP, 1, 0}, gB{GROUP, 1, 0};
    {
      // canonical K order: the order a tensor-core producer wrote the contracted bonds
      // in (korder), else sorted by label
      std::vector<std::pair<int64_t, KDim>> kl;
      for (auto& d : A.dims)
        if (d.label != GROUP && lb.count(d.label)) {
          kset.insert(d.label);
          int64_t sb = 0;
          for (auto& e : B.dims) if (e.label == d.label) sb = e.stride;
          kl.push_back({d.label, {d.ext, d.stride, sb}});
        }
      {
        const std::vector<int64_t>& ko = korder[s];
        auto rank = [&](int64_t l) {
          for (size_t q = 0; q < ko.size(); ++q) if (ko[q] == l) return (int64_t)q;
          return (int64_t)ko.size();
        };
        std::sort(kl.begin(), kl.end(),
                  [&](const std::pair<int64_t, KDim>& a, const std::pair<int64_t, KDim>& b) {
                    const int64_t ra = rank(a.first), rb = rank(b.first);
                    return ra != rb ? ra < rb : a.first < b.first;
                  });
      }
      for (auto& x : kl) K.push_back(x.second);
    }
    for (auto& d : A.dims) {
      if (d.label != GROUP && kset.count(d.label)) continue;
      if (sp.merge && d.label == GROUP) { gA = d; continue; }
      FA.push_back(d);
    }
    for (auto& d : B.dims) {
      if (d.label != GROUP && kset.count(d.label)) continue;
      if (sp.merge && d.label == GROUP) { gB = d; continue; }
      FB.push_back(d);
    }
    const std::vector<VDim> FA0 = FA, FB0 = FB;
    const std::vector<KDim> K0 = K;
    if (sp.mode != 1 && sp.mode != 3) {   // the planner's output order (consumer look-ahead)
      FA = arrange(FA, sp.swap ? sp.order2 : sp.order1);
      FB = arrange(FB, sp.swap ? sp.order1 : sp.order2);
    }
    coalesce1(FA);
    coalesce1(FB);
    coalesce2(K);
    if ((int)FA.size() > TN_MAXD || (int)FB.size() > TN_MAXD || (int)K.size() > TN_MAXD)
      return fail(TN_ERR_INTERNAL, "step " + std::to_string(s) + ": too many non-coalescable dims");
    unsigned* absmax_out = sp.final_step ? nullptr : c->d_absmax + (n_leaves + s);
    float2* Cptr = sp.final_step ? nullptr : c->d_arena + sp.out_off;
    if (!sp.tc && (sp.mode == 1 || sp.mode == 3)) {
      // skinny: X = big operand (streamed), Y = small operand (smem); out [Xo][Y][v]
      const View& XV = sp.x_is_b ? B : A;
      const View& YV = sp.x_is_b ? A : B;
      const auto& X0 = sp.x_is_b ? FB0 : FA0;
      std::vector<VDim> Xo, Ys = sp.x_is_b ? FA0 : FB0;
      // merged lane dim: the run is contiguous in X and innermost (same order) in C
      VDim v{0, 1, INT64_MAX};
      for (auto& d : X0) {
        if (std::find(sp.vlabels.begin(), sp.vlabels.end(), d.label) != sp.vlabels.end()) {
          v.ext *= d.ext;
          v.stride = std::min(v.stride, d.stride);
        } else {
          Xo.push_back(d);
        }
      }
      Xo = arrange(Xo, sp.order1);
      Ys = arrange(Ys, sp.order2);
      coalesce1(Xo);
      coalesce1(Ys);
      std::vector<KDim> Kx = K0;
      if (sp.x_is_b) for (auto& x : Kx) std::swap(x.sa, x.sb);
      coalesce2(Kx);
      if ((int)Xo.size() + 1 > TN_MAXD || (int)Ys.size() > TN_MAXD || (int)Kx.size() > TN_MAXD)
        return fail(TN_ERR_INTERNAL, "step " + std::to_string(s) + ": too many dims (skinny)");
      tn::EinsumDesc& e = eds[sp.einsum_idx];
      memset(&e, 0, sizeof(e));
      e.mode = sp.mode;
      e.A = base_of(XV); e.B = base_of(YV); e.C = Cptr;
      e.a_off = XV.off; e.b_off = YV.off;
      if (sp.merge && sp.J == 1) {   // fold the single slab of each side into the offsets
        const int64_t sa = (int64_t)sp.ia[0] * gA.stride, sb = (int64_t)sp.ib[0] * gB.stride;
        e.a_off += sp.x_is_b ? sb : sa;
        e.b_off += sp.x_is_b ? sa : sb;
      }
      e.a_leaf = XV.buf == 0 ? XV.leaf : -1;
      e.b_leaf = YV.buf == 0 ? YV.leaf : -1;
      e.J = 1;
      if (sp.merge && sp.J > 1) {     // batched skinny: X / Y slabs per batch j
        const int32_t* ta = c->host_only ? nullptr : c->d_tables + sp.ia_off;
        const int32_t* tb = c->host_only ? nullptr : c->d_tables + sp.ib_off;
        e.J = sp.J;
        e.ia = sp.x_is_b ? tb : ta;
        e.ib = sp.x_is_b ? ta : tb;
        e.a_gs = sp.x_is_b ? gB.stride : gA.stride;
        e.b_gs = sp.x_is_b ? gA.stride : gB.stride;
        e.n_yslabs = sp.x_is_b ? gA.ext : gB.ext;
      }
      e.M = sp.x_is_b ? sp.n : sp.m;
      e.N = sp.x_is_b ? sp.m : sp.n;
      e.K = sp.k;
      e.V = v.ext;
      e.nm = (int)Xo.size() + 1;
      for (int p = 0; p < (int)Xo.size(); ++p) { e.m_ext[p] = Xo[p].ext; e.m_sa[p] = Xo[p].stride; }
      e.m_ext[e.nm - 1] = v.ext;
      e.m_sa[e.nm - 1] = v.stride;
      e.nn = (int)Ys.size();
      for (int p = 0; p < e.nn; ++p) { e.n_ext[p] = Ys[p].ext; e.n_sb[p] = Ys[p].stride; }
      e.nk = (int)Kx.size();
      for (int p = 0; p < e.nk; ++p) { e.k_ext[p] = Kx[p].ext; e.k_sa[p] = Kx[p].sa; e.k_sb[p] = Kx[p].sb; }
      e.absmax_out = absmax_out;
      e.acc = sp.final_step ? c->d_acc : nullptr;
      fill_shifts(e);
      sp.hdesc = e;
      sp.x_slot = XV.absmax_slot;
      sp.y_slot = YV.absmax_slot;
      if (c->debug_plan) {
        fprintf(stderr, "[tn] step %d simt mode %d M=%lld N=%lld K=%lld V=%lld vstride=%lld a_off%%2=%lld leaf=%d pow2=%d x:", s,
                e.mode, (long long)e.M, (long long)e.N, (long long)e.K, (long long)e.V,
                (long long)e.m_sa[e.nm - 1], (long long)(e.a_off % 2), e.a_leaf, e.pow2);
        for (int d = 0; d < e.nm; ++d) fprintf(stderr, " %lldx%lld", (long long)e.m_ext[d], (long long)e.m_sa[d]);
        fprintf(stderr, " | k:");
        for (int d = 0; d < e.nk; ++d) fprintf(stderr, " %lldx%lld", (long long)e.k_ext[d], (long long)e.k_sa[d]);
        fprintf(stderr, "\n");
      }
    } else if (!sp.tc) {
      tn::EinsumDesc& e = eds[sp.einsum_idx];
      memset(&e, 0, sizeof(e));
      e.A = base_of(A); e.B = base_of(B); e.C = Cptr;
      e.a_off = A.off; e.b_off = B.off;
      e.a_leaf = A.buf == 0 ? A.leaf : -1;
      e.b_leaf = B.buf == 0 ? B.leaf : -1;
      e.J = sp.J;
      e.ia = sp.merge ? c->d_tables + sp.ia_off : nullptr;
      e.ib = sp.merge ? c->d_tables + sp.ib_off : nullptr;
      e.a_gs = gA.stride; e.b_gs = gB.stride;
      e.M = sp.m; e.N = sp.n; e.K = sp.k;
      e.nm = (int)FA.size(); e.nn = (int)FB.size(); e.nk = (int)K.size();
      for (int p = 0; p < e.nm; ++p) { e.m_ext[p] = FA[p].ext; e.m_sa[p] = FA[p].stride; }
      for (int p = 0; p < e.nn; ++p) { e.n_ext[p] = FB[p].ext; e.n_sb[p] = FB[p].stride; }
      for (int p = 0; p < e.nk; ++p) { e.k_ext[p] = K[p].ext; e.k_sa[p] = K[p].sa; e.k_sb[p] = K[p].sb; }
      e.absmax_out = absmax_out;
      e.acc = sp.final_step ? c->d_acc : nullptr;
      if (sp.mode == 2) {
        e.mode = 2;
        e.partial = c->d_partial;
        e.kchunk = 1 << 16;
      }
      if (sp.mode == 4) e.mode = 4;
      fill_shifts(e);
      if (e.mode == 4 && sp.wd_start_off >= 0 && wd_staged) plan_wd_staged(e, sp.wd_nslabs);
      if (e.wd_ok) {
        e.wd_start = c->host_only ? nullptr : c->d_tables + sp.wd_start_off;
        e.wd_list = c->host_only ? nullptr : c->d_tables + sp.wd_list_off;
      }
      sp.hdesc = e;
      if (c->debug_plan) {
        fprintf(stderr, "[tn] step %d simt mode %d J=%lld M=%lld N=%lld K=%lld a_gs=%lld b_gs=%lld wd=%d(t=%d lb=%d np=%d) m:",
                s, e.mode, (long long)e.J, (long long)e.M, (long long)e.N, (long long)e.K, (long long)e.a_gs,
                (long long)e.b_gs, e.wd_ok, e.wd_t, e.wd_lb, e.wd_np);
        for (int d = 0; d < e.nm; ++d) fprintf(stderr, " %lldx%lld", (long long)e.m_ext[d], (long long)e.m_sa[d]);
        fprintf(stderr, " | n:");
        for (int d = 0; d < e.nn; ++d) fprintf(stderr, " %lldx%lld", (long long)e.n_ext[d], (long long)e.n_sb[d]);
        fprintf(stderr, " | k:");
        for (int d = 0; d < e.nk; ++d)
          fprintf(stderr, " %lldx(%lld,%lld)", (long long)e.k_ext[d], (long long)e.k_sa[d], (long long)e.k_sb[d]);
        fprintf(stderr, "\n");
      }
    } else {
      // P operand = A side unless swapped; both share the canonical K order
      memset(&sp.gemm, 0, sizeof(sp.gemm));
      for (int side = 0; side < 2; ++side) {
        const bool fromA = (side == 0) != sp.swap;
        const View& V = fromA ? A : B;
        const auto& F = fromA ? FA : FB;
        tn::PrepDesc& p = pds[sp.prep_idx + side];
        memset(&p, 0, sizeof(p));
        p.src = base_of(V);
        p.off = V.off;
        p.leaf = V.buf == 0 ? V.leaf : -1;
        p.G = sp.G[side];
        p.R = sp.R[side];
        p.K = sp.k;
        p.Kpad = sp.Kpad;
        p.g_stride = sp.merge ? (fromA ? gA.stride : gB.stride) : 0;
        p.nr = (int)F.size();
        for (int d = 0; d < p.nr; ++d) { p.r_ext[d] = F[d].ext; p.r_s[d] = F[d].stride; }
        std::vector<VDim> kd;
        for (auto& x : K) kd.push_back({0, x.ext, fromA ? x.sa : x.sb});
        coalesce1(kd);   // per-operand merge keeps the shared row-major k order
        p.nk = (int)kd.size();
        for (int d = 0; d < p.nk; ++d) { p.k_ext[d] = kd[d].ext; p.k_s[d] = kd[d].stride; }
        {
          const int64_t rs = p.nr ? p.r_s[p.nr - 1] : INT64_MAX;
          const int64_t ks = p.nk ? p.k_s[p.nk - 1] : INT64_MAX;
          p.read_r_fast = rs < ks ? 1 : 0;
        }
        if (sp.grouped && side == 0) {
          // gathered rows: row r = (j, q) of the Y side -> slabY(j)·stride + offset of q
          const std::vector<int32_t>& sy = fromA ? sp.ia : sp.ib;
          const int64_t gys = fromA ? gA.stride : gB.stride;
          const int64_t Q = fromA ? sp.m : sp.n;
          std::vector<int64_t> rowoff((size_t)sp.g_rows, -1);
          for (int64_t r = 0; r < sp.g_rows; ++r) {
            const int32_t mrow = sp.g_rowmap[r];
            if (mrow < 0) continue;
            int64_t q = mrow % Q, off = (int64_t)sy[mrow / Q] * gys;
            for (int d = p.nr - 1; d >= 0; --d) { off += (q % p.r_ext[d]) * p.r_s[d]; q /= p.r_ext[d]; }
            rowoff[r] = off;
          }
          p.g_stride = 0;
          p.kind = 3;
          sp.r_fast[side] = 3;
          sp.gtT[side] = 0;
          rw_ref.push_back({sp.prep_idx + side, (int64_t)gt_all.size()});
          gt_all.insert(gt_all.end(), rowoff.begin(), rowoff.end());
        } else {
          const int64_t Kpad_ = sp.Kpad;
          p.Kpad = Kpad_;
          std::vector<int64_t> tab;
          p.kind = choose_prep_kind(p, prep_force, tab);
          sp.r_fast[side] = p.kind;
          sp.gtT[side] = (p.kind == 2 || p.kind == 4) ? p.T : 0;
          if (p.kind == 2) tab = gt_tables(p);
          if (p.kind == 2 || p.kind == 4) {
            (p.kind == 2 ? gt_ref : bp_ref).push_back({sp.prep_idx + side, (int64_t)gt_all.size()});
            gt_all.insert(gt_all.end(), tab.begin(), tab.end());
          }
        }
        int64_t off0 = 0;
        int64_t bytes0 = (4 * sp.G[0] * sp.R[0] * sp.Kpad * 2 + 1023) / 1024 * 1024;
        if (side == 1) off0 = bytes0;
        p.dst = reinterpret_cast<__half*>(c->d_scratch + off0);
        p.plane_elems = sp.G[side] * sp.R[side] * sp.Kpad;
        p.absmax_in = c->d_absmax + V.absmax_slot;
        p.scale_out = c->d_scales + 2 * s + side;
        sp.prep_total[side] = p.plane_elems;
        CUtensorMap* map = side == 0 ? &sp.gemm.mapA : &sp.gemm.mapB;
        if (!c->host_only &&
            (!tn::encode_plane_map(map, p.dst, sp.Kpad, sp.dense_merge ? sp.G[side] * sp.R[side] : sp.R[side],
                                   sp.dense_merge ? 1 : sp.G[side], 4, 128, errbuf, sizeof(errbuf)) ||
             (side == 1 && !tn::encode_plane_map(&sp.gemm.mapB2, p.dst, sp.Kpad,
                                                 sp.dense_merge ? sp.G[side] * sp.R[side] : sp.R[side],
                                                 sp.dense_merge ? 1 : sp.G[side], 4, 64, errbuf,
                                                 sizeof(errbuf)))))
          return fail(TN_ERR_INTERNAL, errbuf);
        if (c->debug_plan) {
          fprintf(stderr, "[tn] step %d prep%c G=%lld R=%lld K=%lld kind=%d T=%d rows:", s,
                  side ? 'Q' : 'P', (long long)p.G, (long long)p.R, (long long)p.K, p.kind, p.T);
          for (int d = 0; d < p.nr; ++d) fprintf(stderr, " %lldx%lld", (long long)p.r_ext[d], (long long)p.r_s[d]);
          fprintf(stderr, " | k:");
          for (int d = 0; d < p.nk; ++d) fprintf(stderr, " %lldx%lld", (long long)p.k_ext[d], (long long)p.k_s[d]);
          fprintf(stderr, "\n");
        }
      }
      tn::GemmArgs& g = sp.gemm;
      g.J = (int32_t)sp.J;
      g.M = (int32_t)sp.R[0];
      g.N = (int32_t)sp.R[1];
      g.K = (int32_t)sp.k;
      const int32_t* ta = sp.merge ? c->d_tables + sp.ia_off : nullptr;
      const int32_t* tb = sp.merge ? c->d_tables + sp.ib_off : nullptr;
      g.ia = sp.swap ? tb : ta;
      g.ib = sp.swap ? ta : tb;
      g.C = Cptr;
      g.scaleA = c->d_scales + 2 * s;
      g.scaleB = c->d_scales + 2 * s + 1;
      g.absmax_out = absmax_out;
      g.acc = sp.final_step ? c->d_acc : nullptr;
      g.tiles_m = (int32_t)((sp.R[0] + 127) / 128);
      g.tiles_n = (int32_t)((sp.R[1] + 127) / 128);
      g.n_tiles = (int64_t)g.tiles_m * g.tiles_n * sp.J;
      g.blk_slab_b = nullptr;
      g.rowmap = nullptr;
      g.use_pair = 0;
      if (sp.dense_merge) {   // one dense GEMM over the slab product, pair-mapped epilogue
        g.J = 1;
        g.ia = nullptr;
        g.ib = nullptr;
        g.M = (int32_t)(sp.G[0] * sp.R[0]);
        g.N = (int32_t)(sp.G[1] * sp.R[1]);
        g.tiles_m = (g.M + 127) / 128;
        g.tiles_n = (g.N + 127) / 128;
        g.n_tiles = (int64_t)g.tiles_m * g.tiles_n;
        g.pair_map = c->d_tables + sp.pair_off;
        int lm = 0, ln = 0;
        while ((int64_t(1) << lm) < sp.R[0]) ++lm;
        while ((int64_t(1) << ln) < sp.R[1]) ++ln;
        g.pm_sh_m = lm;
        g.pm_sh_n = ln;
        g.pm_g1 = (int32_t)sp.G[1];
      }
      if (sp.grouped) {   // one GEMM over the gathered rows; X slab per 128-row block
        g.J = 1;
        g.ia = nullptr;
        g.ib = nullptr;
        g.blk_slab_b = c->d_tables + sp.g_blk_off;
        g.rowmap = c->d_tables + sp.g_rowmap_off;
        g.n_tiles = (int64_t)g.tiles_m * g.tiles_n;
      }
      g.use_pair = tn::gemm_pair_ok(g, pair_min_m) ? 1 : 0;
      g.wave_ctr = c->d_wave;
      g.wave_sync = (wave_sync && sp.k >= wave_min_k) ? 1 : 0;
      g.out_gen = sp.out_gen ? 1 : 0;
      if (sp.out_gen) {
        auto lg = [](int64_t x) { int q = 0; while ((int64_t(1) << q) < x) ++q; return q; };
        g.n_po = (int32_t)sp.po.size();
        g.n_qo = (int32_t)sp.qo.size();
        for (int q = 0; q < g.n_po; ++q) { g.po_sh[q] = (uint8_t)lg(sp.po[q].ext); g.po_str[q] = sp.po[q].stride; }
        for (int q = 0; q < g.n_qo; ++q) { g.qo_sh[q] = (uint8_t)lg(sp.qo[q].ext); g.qo_str[q] = sp.qo[q].stride; }
        g.cols_contig = (g.n_qo > 0 && g.qo_str[g.n_qo - 1] == 1 && g.qo_sh[g.n_qo - 1] >= 6) ? 1 : 0;
        g.cols_stride = (cols_single && g.n_qo == 1 && g.qo_str[0] > 1) ? g.qo_str[0] : 0;
        if (c->debug_plan) {
          fprintf(stderr, "[tn] step %d out_gen M=%d N=%d rows:", s, g.M, g.N);
          for (int q = 0; q < g.n_po; ++q) fprintf(stderr, " 2^%dx%lld", g.po_sh[q], (long long)g.po_str[q]);
          fprintf(stderr, " | cols:");
          for (int q = 0; q < g.n_qo; ++q) fprintf(stderr, " 2^%dx%lld", g.qo_sh[q], (long long)g.qo_str[q]);
          fprintf(stderr, "\n");
        }
      }
    }
    live.erase(sp.j);
    live[sp.i] = sp.out;
    producer_of.erase(sp.j);
    producer_of[sp.i] = s;
  }
  // ---- fused plane output (a3 + a6 folded into the producer's GEMM epilogue): a
  // tensor-core step whose output is a tensor-core operand writes that operand's fp16
  // planes in the consumer's [G][R][Kpad] layout straight into its arena slot (same
  // 8 bytes per element as complex64), and the consumer skips that side's prep.
  for (auto& st_ : c->steps) st_.gemm_plain = st_.gemm;
  if (fuse_planes)
    for (int s = 0; s < n_steps; ++s) {
      StepPlan& cs = c->steps[s];
      if (!cs.tc || cs.grouped || cs.dense_merge) continue;
      for (int side = 0; side < 2; ++side) {
        const int ps = side_producer[s][side];
        if (ps < 0) continue;
        StepPlan& pp = c->steps[ps];
        if (!pp.tc || pp.grouped || pp.dense_merge || pp.final_step || pp.planes_consumer >= 0) continue;
        if (c->debug_plan) fprintf(stderr, "[tn] fuse candidate %d->%d side %d\n", ps, s, side);
        const tn::PrepDesc& pd = pds[cs.prep_idx + side];
        const int64_t Kp = cs.Kpad;
        auto skip = [&](const char* why) {
          if (c->debug_plan) fprintf(stderr, "[tn] fuse %d->%d side %d: no (%s)\n", ps, s, side, why);
        };
        if (Kp != cs.k || Kp % 8 != 0) { skip("K"); continue; }
        if (pd.G * pd.R * Kp != pp.out_elems) { skip("size"); continue; }
        if (pd.G > 1 && pd.g_stride != pd.R * Kp) { skip("group"); continue; }
        // source (producer complex64 offset) bit weight -> consumer plane-element weight
        std::unordered_map<int64_t, int64_t> wmap;
        bool ok = true;
        auto p2 = [](int64_t x) { return x > 0 && (x & (x - 1)) == 0; };
        int64_t inner = 1;
        for (int d = pd.nk - 1; d >= 0 && ok; --d) {
          ok = p2(pd.k_ext[d]) && p2(pd.k_s[d]);
          for (int64_t e = 1; ok && e < pd.k_ext[d]; e <<= 1) ok = wmap.emplace(pd.k_s[d] * e, inner * e).second;
          inner *= pd.k_ext[d];
        }
        inner = Kp;
        for (int d = pd.nr - 1; d >= 0 && ok; --d) {
          ok = p2(pd.r_ext[d]) && p2(pd.r_s[d]);
          for (int64_t e = 1; ok && e < pd.r_ext[d]; e <<= 1) ok = wmap.emplace(pd.r_s[d] * e, inner * e).second;
          inner *= pd.r_ext[d];
        }
        if (!ok) { skip("prep dims"); continue; }
        // the producer's row / column digit maps (outer -> inner), one bit per entry,
        // re-expressed in plane units, then re-coalesced
        auto side_dims = [&](bool rows, std::vector<std::pair<int, int64_t>>& out) {
          const tn::GemmArgs& g = pp.gemm;
          std::vector<VDim> dims;
          if (pp.out_gen) {
            const int n = rows ? g.n_po : g.n_qo;
            for (int q = 0; q < n; ++q)
              dims.push_back({0, int64_t(1) << (rows ? g.po_sh[q] : g.qo_sh[q]), rows ? g.po_str[q] : g.qo_str[q]});
          } else {   // plain [J][M][N]
            if (rows) dims.push_back({0, (int64_t)g.M, (int64_t)g.N});
            else dims.push_back({0, (int64_t)g.N, 1});
          }
          std::vector<int64_t> bits;   // plane weight per digit bit, inner -> outer
          for (int q = (int)dims.size() - 1; q >= 0; --q) {
            if (!p2(dims[q].ext)) return false;
            for (int64_t e = 1; e < dims[q].ext; e <<= 1) {
              auto it = wmap.find(dims[q].stride * e);
              if (it == wmap.end()) return false;
              bits.push_back(it->second);
            }
          }
          out.clear();                 // coalesce inner -> outer, emit outer -> inner
          for (int64_t w : bits) {
            if (!out.empty() && (out.back().second << out.back().first) == w) out.back().first++;
            else out.push_back({1, w});
          }
          std::reverse(out.begin(), out.end());
          return (int)out.size() <= 16;
        };
        std::vector<std::pair<int, int64_t>> po, qo;
        if (!side_dims(true, po) || !side_dims(false, qo)) { skip("producer dims"); continue; }
        // 16-B plane vectors: the 8 lowest column indices must be plane-contiguous
        const bool cols = !qo.empty() && qo.back().second == 1 && qo.back().first >= 3;
        const bool rows = fuse_planes != 2 && !po.empty() && po.back().second == 1 && po.back().first >= 3 &&
                          pp.gemm.M % 8 == 0;
        if (pp.gemm.N % 8 != 0 || (!cols && !rows)) {
          skip("no plane-contiguous run of 8 rows or columns");
          continue;
        }
        tn::GemmArgs& g = pp.gemm;
        g.planes_rows = cols ? 0 : 1;
        if (c->debug_plan)
          fprintf(stderr, "[tn] fuse %d->%d side %d: yes (%s, producer K=%lld)\n", ps, s, side, cols ? "cols" : "rows",
                  (long long)pp.k);
        g.out_gen = 1;
        g.out_planes = 1;
        g.n_po = (int)po.size();
        g.n_qo = (int)qo.size();
        for (int q = 0; q < g.n_po; ++q) { g.po_sh[q] = (uint8_t)po[q].first; g.po_str[q] = po[q].second; }
        for (int q = 0; q < g.n_qo; ++q) { g.qo_sh[q] = (uint8_t)qo[q].first; g.qo_str[q] = qo[q].second; }
        g.cols_contig = 0;   // plane mode has its own 8-column vectors
        g.cols_stride = 0;
        // 256-bit plane stores: 16 plane-contiguous columns whose offsets are 16-element
        // (32-B) aligned (every other stride and the plane size multiples of 16)
        {
          bool v16 = cols && qo.back().first >= 4 && pp.gemm.N % 16 == 0 && pp.out_elems % 16 == 0;
          for (auto& d : po) v16 = v16 && d.second % 16 == 0;
          for (size_t q = 0; q + 1 < qo.size(); ++q) v16 = v16 && qo[q].second % 16 == 0;
          g.planes_v16 = (v16 && plane_v16) ? 1 : 0;
        }
        if (c->debug_plan) {
          fprintf(stderr, "[tn] step %d planes%s rows:", ps, g.planes_v16 ? " v16" : "");
          for (auto& d : po) fprintf(stderr, " 2^%dx%lld", d.first, (long long)d.second);
          fprintf(stderr, " | cols:");
          for (auto& d : qo) fprintf(stderr, " 2^%dx%lld", d.first, (long long)d.second);
          fprintf(stderr, "\n");
        }
        int lk = 0;
        while ((int64_t(1) << lk) < pp.k) ++lk;
        g.plane_exp = -16 - lk;
        g.plane_elems = pp.out_elems;
        g.plane_scale_out = c->d_scales + 2 * s + side;
        g.plane_pexp = c->d_pexp + ps;
        g.overflow = c->d_flag;
        pp.out_gen = true;
        pp.planes_consumer = s;
        cs.skip_prep[side] = true;
        if (!c->host_only) {
          const __half* base = reinterpret_cast<const __half*>(c->d_arena + pp.out_off);
          CUtensorMap* map = side == 0 ? &cs.gemm.mapA : &cs.gemm.mapB;
          if (!tn::encode_plane_map(map, base, Kp, cs.R[side], cs.G[side], 4, 128, errbuf, sizeof(errbuf)) ||
              (side == 1 && !tn::encode_plane_map(&cs.gemm.mapB2, base, Kp, cs.R[side], cs.G[side], 4, 64,
                                                  errbuf, sizeof(errbuf))))
            return fail(TN_ERR_INTERNAL, errbuf);
        }
      }
    }
  // ---- gate folding: a skinny SIMT step (a small gate absorbed into a big tensor) whose
  // output is a tensor-core operand is applied inside that operand's prep instead
  const bool hint_pass = !c->fold_hint.empty();
  if (fold_gates)
    for (int s = 0; s < n_steps; ++s) {
      StepPlan& cs = c->steps[s];
      if (!cs.tc || cs.grouped || cs.dense_merge) continue;
      for (int side = 0; side < 2; ++side) {
        const int ps = side_producer[s][side];
        if (ps < 0 || cs.skip_prep[side]) continue;
        StepPlan& pp = c->steps[ps];
        if (pp.tc || pp.mode != 1 || pp.final_step || pp.folded) continue;
        if (pp.hdesc.K > fold_maxk || pp.hdesc.N > fold_maxn) continue;
        if (hint_pass && !c->fold_hint[ps]) continue;
        tn::PrepDesc& pd = pds[cs.prep_idx + side];
        tn::PrepDesc trial = pd;
        std::vector<int64_t> tab;
        if (!plan_gate(trial, pp.hdesc, tab)) {
          if (c->debug_plan) fprintf(stderr, "[tn] fold %d->%d side %d: no\n", ps, s, side);
          continue;
        }
        if (c->debug_plan)
          fprintf(stderr, "[tn] fold %d->%d side %d: yes (N=%lld K=%lld, tile 2^%d / src 2^%d)\n", ps, s, side,
                  (long long)pp.hdesc.N, (long long)pp.hdesc.K, trial.bp_t, trial.g_ts);
        trial.kind = 5;
        trial.src = pp.hdesc.A;
        trial.off = pp.hdesc.a_off;
        trial.leaf = pp.hdesc.a_leaf;
        trial.gy = pp.hdesc.B;
        trial.gy_off = pp.hdesc.b_off;
        trial.gy_leaf = pp.hdesc.b_leaf;
        trial.g_regroup = gate_regroup;
        if (!c->host_only) {
          trial.absmax_in = c->d_absmax + pp.x_slot;
          trial.absmax_y = c->d_absmax + pp.y_slot;
        }
        pd = trial;
        cs.r_fast[side] = 5;
        cs.gtT[side] = trial.T;
        cs.gate_k[side] = (int)pp.hdesc.K;
        cs.gate_n[side] = (int)pp.hdesc.N;
        gate_ref.push_back({cs.prep_idx + side, (int64_t)gt_all.size()});
        gt_all.insert(gt_all.end(), tab.begin(), tab.end());
        pp.folded = true;
      }
    }
  {
    std::vector<char> decided(n_steps, 0);
    bool any = false;
    for (int s = 0; s < n_steps; ++s) if (c->steps[s].folded) { decided[s] = 1; any = true; }
    if (hint_pass) {
      if (decided != c->fold_hint) return fail(TN_ERR_INTERNAL, "gate folding changed between planning passes");
    } else if (any) {
      c->fold_hint = decided;        // tn_set_slices re-plans with the folds' liveness
      return TN_OK;
    }
  }
  // ---- fused skinny chains: maximal runs of skinny steps feeding each
  // other's big operand, cut greedily where plan_chain rejects the extension
  c->chains.clear();
  std::vector<int32_t> chain_tab_all;
  std::vector<int32_t> chain_tab_at;
  for (auto& sp : c->steps) { sp.chain = -1; sp.chained = false; }
  if (c->chain_mode) {
    auto ok = [&](int s) {
      const StepPlan& sp = c->steps[s];
      return !sp.tc && !sp.folded && sp.mode == 1 && !sp.final_step && sp.J == 1 && sp.einsum_idx >= 0;
    };
    auto unmaterialised = [&](int w) {
      return c->steps[w].folded || (w < (int)c->chain_hint.size() && c->chain_hint[w] > w);
    };
    auto overlaps = [&](int w, int p) {     // step w's output slot overlaps step p's output slot
      const StepPlan& W = c->steps[w];
      const StepPlan& P = c->steps[p];
      if (W.final_step || unmaterialised(w) || P.final_step) return false;
      return W.out_off < P.out_off + P.out_elems && P.out_off < W.out_off + W.out_elems;
    };
    auto chain_inputs_survive = [&](const std::vector<int>& run, size_t a, size_t b) {
      const int last = run[b - 1];
      std::vector<char> member(n_steps, 0);
      for (size_t q = a; q < b; ++q) member[run[q]] = 1;
      std::vector<std::pair<int, int>> ins;  // (producer of the input, step consuming it)
      ins.push_back({x_producer[run[a]], run[a]});
      for (size_t q = a; q < b; ++q) ins.push_back({y_producer[run[q]], run[q]});
      for (auto& in : ins) {
        if (in.first < 0) continue;          // a leaf: never overwritten
        for (int w = in.second + 1; w < last; ++w)
          if (!member[w] && overlaps(w, in.first)) return false;
      }
      return true;
    };
    std::vector<int> nxt(n_steps, -1), has_prev(n_steps, 0);
    for (int s = 0; s < n_steps; ++s) {
      const int cn = consumer_step[s];
      if (ok(s) && cn >= 0 && ok(cn) && x_producer[cn] == s) { nxt[s] = cn; has_prev[cn] = 1; }
    }
    for (int s0 = 0; s0 < n_steps; ++s0) {
      if (nxt[s0] < 0 || has_prev[s0]) continue;
      std::vector<int> run;
      for (int s = s0; s >= 0; s = nxt[s]) run.push_back(s);
      // partition the run into chains maximising the HBM bytes saved (each intermediate of a
      // chain is neither written nor read back): DP over accepted sub-chains [a, b)
      const size_t R = run.size();
      std::vector<double> gain(R + 1, 0.0);
      std::vector<size_t> cut(R + 1, 0);
      for (size_t a = R; a-- > 0;) {
        gain[a] = gain[a + 1];
        cut[a] = a + 1;          // a alone
        double saved = 0.0;
        for (size_t b = a + 2; b <= R && b - a <= (size_t)tn::TN_CHAIN_MAX; ++b) {
          const tn::EinsumDesc& em = eds[c->steps[run[b - 2]].einsum_idx];
          saved += 16.0 * (double)(em.M * em.N);   // intermediate run[b-2] -> run[b-1]
          std::vector<const tn::EinsumDesc*> es;
          for (size_t q = a; q < b; ++q) es.push_back(&eds[c->steps[run[q]].einsum_idx]);
          tn::ChainDesc cd;
          memset(&cd, 0, sizeof(cd));
          std::vector<int32_t> tab;
          // profitable only when the chain keeps a big intermediate out of HBM: measured on
          // C4-sparse, a chain saving 2^30+2^29 elements wins (11.1 -> 9.5 ms), one saving
          // 2^28+2^29 breaks even and small ones lose (the per-tile barriers and load latency
          // of the fused kernel outweigh the traffic)
          // ... and each tile must carry enough work (>= 64 touched elements in some tensor)
          if (saved >= c->chain_min_save && plan_chain(es, c->chain_maxbits, cd, tab) &&
              std::max(cd.buf_a, cd.buf_b) >= 64 && saved + gain[b] > gain[a]) {
            gain[a] = saved + gain[b];
            cut[a] = b;
          }
        }
      }
      for (size_t a = 0; a < R;) {
        const size_t best = cut[a];
        if (best == a + 1) { a = best; continue; }
        // the chain runs at its last member's position: its inputs (the head's X, every
        // member's Y) must have survived until then (the hinted pass keeps them live)
        if (!c->chain_hint.empty() && !chain_inputs_survive(run, a, best))
          return fail(TN_ERR_INTERNAL, "chain inputs not kept live");
        tn::ChainDesc bd;
        memset(&bd, 0, sizeof(bd));
        std::vector<int32_t> btab;
        {
          std::vector<const tn::EinsumDesc*> es;
          for (size_t q = a; q < best; ++q) es.push_back(&eds[c->steps[run[q]].einsum_idx]);
          if (!plan_chain(es, c->chain_maxbits, bd, btab)) return fail(TN_ERR_INTERNAL, "chain re-plan");
        }
        const tn::EinsumDesc& e0 = eds[c->steps[run[a]].einsum_idx];
        const tn::EinsumDesc& eL = eds[c->steps[run[best - 1]].einsum_idx];
        bd.src = e0.A; bd.src_off = e0.a_off; bd.src_leaf = e0.a_leaf;
        bd.dst = eL.C; bd.absmax_out = eL.absmax_out;
        for (size_t q = a; q < best; ++q) {
          const tn::EinsumDesc& e = eds[c->steps[run[q]].einsum_idx];
          bd.st[q - a].Y = e.B; bd.st[q - a].y_off = e.b_off; bd.st[q - a].y_leaf = e.b_leaf;
          c->steps[run[q]].chained = q + 1 < best;    // launched at the last member's position
          c->steps[run[q]].chain = (int)c->chains.size();
        }
        const int at = run[best - 1];
        c->steps[at].chain = (int)c->chains.size();
        {
          double t = 0, y = 0;
          for (size_t q = a; q < best; ++q) {
            t += c->steps[run[q]].tcc;
            y += 8.0 * eds[c->steps[run[q]].einsum_idx].N * eds[c->steps[run[q]].einsum_idx].K;
          }
          c->steps[at].chain_tcc = t;
          c->steps[at].chain_tmc = 8.0 * (double)(e0.M * e0.K + eL.M * eL.N) + y;
        }
        chain_tab_at.push_back((int32_t)chain_tab_all.size());
        chain_tab_all.insert(chain_tab_all.end(), btab.begin(), btab.end());
        c->chains.push_back(bd);
        if (c->debug_plan) {
          fprintf(stderr, "[tn] chain:");
          for (size_t q = a; q < best; ++q) fprintf(stderr, " %d", run[q]);
          fprintf(stderr, " (W bits %d..%d, carry tiles 2^%d, smem %zu B)\n", bd.a0, bd.aL, bd.nct,
                  tn::chain_smem_bytes(bd));
        }
        a = best;
      }
    }
  }
  {
    std::vector<int> hint(n_steps, -1);
    for (int q = 0; q < n_steps; ++q)
      if (c->steps[q].chained) {
        int L = q;
        while (L < n_steps && !(c->steps[L].chain == c->steps[q].chain && !c->steps[L].chained)) ++L;
        hint[q] = L;
      }
    const bool any = std::any_of(hint.begin(), hint.end(), [](int x) { return x >= 0; });
    if (c->chain_hint.empty()) {
      if (any) {                       // re-plan with the chains' liveness (tn_set_slices)
        c->chain_hint = hint;
        c->replan = true;
        return TN_OK;
      }
    } else if (hint != c->chain_hint) {
      return fail(TN_ERR_INTERNAL, "skinny chains changed between planning passes");
    }
  }
  if (c->host_only) {
    c->planned = true;
    return TN_OK;
  }
  if (!c->chains.empty()) {
    if (tn_status st3 = dev_alloc(c, &c->d_chain, c->chains.size())) return st3;
    if (tn_status st3 = dev_alloc(c, &c->d_chain_tab, chain_tab_all.size())) return st3;
    TN_CUDA(cudaMemcpyAsync(c->d_chain_tab, chain_tab_all.data(), chain_tab_all.size() * 4,
                            cudaMemcpyHostToDevice, sm));
    for (size_t q = 0; q < c->chains.size(); ++q) c->chains[q].tab = c->d_chain_tab + chain_tab_at[q];
    TN_CUDA(cudaMemcpyAsync(c->d_chain, c->chains.data(), c->chains.size() * sizeof(tn::ChainDesc),
                            cudaMemcpyHostToDevice, sm));
  }
  if (n_einsum) TN_CUDA(cudaMemcpyAsync(c->d_einsum, eds.data(), n_einsum * sizeof(tn::EinsumDesc),
                                        cudaMemcpyHostToDevice, sm));
  if (!gt_all.empty()) {
    tn_status st2 = dev_alloc(c, &c->d_gt, gt_all.size());
    if (st2) return st2;
    TN_CUDA(cudaMemcpyAsync(c->d_gt, gt_all.data(), gt_all.size() * 8, cudaMemcpyHostToDevice, sm));
    for (auto& r : gt_ref) pds[r.first].gt_tab = c->d_gt + r.second;
    for (auto& r : rw_ref) pds[r.first].rowoff = c->d_gt + r.second;
    for (auto& r : bp_ref) pds[r.first].bp_tab = c->d_gt + r.second;
    for (auto& r : gate_ref) pds[r.first].bp_tab = c->d_gt + r.second;
  }
  if (n_prep) TN_CUDA(cudaMemcpyAsync(c->d_prep, pds.data(), n_prep * sizeof(tn::PrepDesc),
                                      cudaMemcpyHostToDevice, sm));
  TN_CUDA(cudaStreamSynchronize(sm));
  c->planned = true;
  return TN_OK;
}

// ---------------------------------------------------------------- execution

struct Timer {
  tn_ctx* c;
  int family;
  double flops, bytes;
  int step;
  cudaEvent_t a{}, b{};
  cudaStream_t sm;
  Timer(tn_ctx* c_, int f, double fl, double by, int st = -1, cudaStream_t s = nullptr)
      : c(c_), family(f), flops(fl), bytes(by), step(st), sm(s ? s : c_->stream) {
    c->stats[f].launches++;
    if (c->profiling) {
      cudaEventCreate(&a);
      cudaEventCreate(&b);
      cudaEventRecord(a, sm);
    }
  }
  ~Timer() {
    if (c->profiling) {
      cudaEventRecord(b, sm);
      c->pending.push_back({a, b, family, flops, bytes, step});
    }
  }
};

// One slice: slice select (a2) then every path step (a3-a8) on stream `sm`.  The
// slice index lives in device memory and advances inside slice_select, so the same
// launch sequence serves every slice (and is what the CUDA graph records).
tn_status launch_slice(tn_ctx* c, const std::vector<int>& passes, cudaStream_t sm) {
  {
    Timer tm(c, 3, 0, 0, -1, sm);
    TN_CUDA(tn::launch_slice_select(c->d_slice_desc, sm));
  }
  for (size_t s = 0; s < c->steps.size(); ++s) {
    StepPlan& sp = c->steps[s];
    if (!sp.tc && sp.folded) continue;      // applied inside its consumer's prep
    if (!sp.tc && sp.chained) continue;     // computed inside its chain's launch
    if (!sp.tc && sp.chain >= 0) {          // fused skinny chain ending at this step
      Timer tm(c, 2, sp.chain_tcc, sp.chain_tmc, (int)s, sm);
      TN_CUDA(tn::launch_chain(c->d_chain + sp.chain, c->chains[sp.chain], c->d_leaf_off, sm));
      continue;
    }
    if (!sp.tc) {
      // first execution of an HBM-bound SIMT step: time every kernel variant on the
      // live operands (the step is idempotent unless it accumulates) and keep the
      // fastest for the following slices
      const int nv = tn::einsum_variants(sp.hdesc);
      if (sp.simt_variant < 0 && c->autotune && c->simt_force < 0 && nv > 1 && !sp.hdesc.acc && sp.tmc > 64e6) {
        cudaEvent_t ev[2 * 8];
        for (int v = 0; v < 2 * nv; ++v) TN_CUDA(cudaEventCreate(&ev[v]));
        for (int v = 0; v < nv; ++v) {
          TN_CUDA(cudaEventRecord(ev[2 * v], sm));
          TN_CUDA(tn::launch_einsum(c->d_einsum + sp.einsum_idx, sp.hdesc, c->d_leaf_off, sm, v));
          TN_CUDA(cudaEventRecord(ev[2 * v + 1], sm));
        }
        TN_CUDA(cudaEventSynchronize(ev[2 * nv - 1]));
        float best = 1e30f;
        for (int v = 0; v < nv; ++v) {
          float ms = 0.f;
          TN_CUDA(cudaEventElapsedTime(&ms, ev[2 * v], ev[2 * v + 1]));
          if (ms < best) { best = ms; sp.simt_variant = v; }
        }
        for (int v = 0; v < 2 * nv; ++v) cudaEventDestroy(ev[v]);
      }
      // untuned (accumulating final steps are never re-run): batched merges with a tiny
      // per-batch output take the warp-per-batch kernel
      int var = sp.simt_variant >= 0 ? sp.simt_variant : (sp.hdesc.mode == 4 && nv >= 3 ? nv - 1 : 0);
      if (c->simt_force >= 0) var = std::min(c->simt_force, nv - 1);
      Timer tm(c, 2, sp.tcc, sp.tmc, (int)s, sm);
      TN_CUDA(tn::launch_einsum(c->d_einsum + sp.einsum_idx, sp.hdesc, c->d_leaf_off, sm, var));
    } else {
      const int ps = passes[s];
      const int planes = ps == 3 ? 4 : 2;
      // the first slice runs unfused: it seeds the delayed-scaling absmax history
      const bool fused = c->tuned;
      for (int side = 0; side < 2; ++side) {
        if (fused && sp.skip_prep[side]) continue;   // planes written by the producer's epilogue
        Timer tm(c, 1, 0, (double)sp.prep_total[side] * (8.0 + 2.0 * planes), (int)s, sm);
        TN_CUDA(tn::launch_prep(c->d_prep + sp.prep_idx + side, sp.prep_total[side], planes,
                                sp.r_fast[side], sp.gtT[side], c->d_leaf_off, sm, sp.gate_k[side],
                                sp.gate_n[side]));
      }
      tn::GemmArgs ga = fused ? sp.gemm : sp.gemm_plain;
      ga.kchunk = ps == 3 ? c->kchunk3 : c->kchunk1;
      // short-K 3-pass GEMMs (K <= 32 * shortk_max): promote every kchunk3_short k-blocks
      // (TN_KCHUNK3_SHORT; A/B knob, default = kchunk3)
      if (ps == 3 && sp.gemm.K <= 32 * c->shortk_max) ga.kchunk = c->kchunk3_short;
      ga.group_m = c->group_m;
      if (fused && sp.planes_consumer >= 0) ga.out_nplanes = passes[sp.planes_consumer] == 3 ? 4 : 2;
      Timer tm(c, 0, sp.tcc, sp.tmc, (int)s, sm);
      TN_CUDA(tn::launch_gemm(ga, ps, c->num_sms, sm));
    }
  }
  return TN_OK;
}

tn_status run_slices(tn_ctx* c, int64_t t0, int64_t t1, tn_precision prec, int topk) {
  cudaStream_t sm = c->stream;
  // mixed precision: the top-k tensor-core steps by T_cc run 1-pass (§4.3, Table 3)
  std::vector<int> passes(c->steps.size(), 3);
  if (prec == TN_PREC_MIXED && topk > 0) {
    std::vector<int> tcs;
    for (size_t s = 0; s < c->steps.size(); ++s) if (c->steps[s].tc) tcs.push_back((int)s);
    std::stable_sort(tcs.begin(), tcs.end(),
                     [&](int a, int b) { return c->steps[a].tcc > c->steps[b].tcc; });
    for (int r = 0; r < (int)tcs.size() && r < topk; ++r) passes[tcs[r]] = 1;
  }
  TN_CUDA(tn::launch_set_counter(c->d_counter, t0, sm));
  for (int64_t t = t0; t < t1; ++t) {
    // After the first slice (kernel attributes set, SIMT variants tuned) the per-slice
    // launch sequence (~500 launches for C4) is recorded once per precision setting
    // into a CUDA graph on a private capture stream and replayed on the caller's stream.
    const bool graph = c->use_graphs && c->tuned && !c->profiling;
    if (!graph) {
      tn_status st = launch_slice(c, passes, sm);
      if (st) return st;
      c->tuned = true;
      continue;
    }
    if (!c->gexec || c->g_prec != (int)prec || c->g_topk != topk) {
      if (c->gexec) { cudaGraphExecDestroy(c->gexec); c->gexec = nullptr; }
      if (!c->cap_stream) TN_CUDA(cudaStreamCreateWithFlags(&c->cap_stream, cudaStreamNonBlocking));
      int64_t before[4];
      for (int f = 0; f < 4; ++f) before[f] = c->stats[f].launches;
      TN_CUDA(cudaStreamBeginCapture(c->cap_stream, cudaStreamCaptureModeRelaxed));
      tn_status st = launch_slice(c, passes, c->cap_stream);
      for (int f = 0; f < 4; ++f) {   // a capture is not an execution: count launches per replay
        c->g_launch[f] = c->stats[f].launches - before[f];
        c->stats[f].launches = before[f];
      }
      cudaGraph_t g = nullptr;
      cudaError_t e = cudaStreamEndCapture(c->cap_stream, &g);
      if (st) { if (g) cudaGraphDestroy(g); return st; }
      if (e != cudaSuccess) return fail(TN_ERR_CUDA, std::string("graph capture: ") + cudaGetErrorString(e));
      e = cudaGraphInstantiate(&c->gexec, g, 0);
      cudaGraphDestroy(g);
      if (e != cudaSuccess) return fail(TN_ERR_CUDA, std::string("graph instantiate: ") + cudaGetErrorString(e));
      c->g_prec = (int)prec;
      c->g_topk = topk;
    }
    TN_CUDA(cudaGraphLaunch(c->gexec, sm));
    c->graph_launches++;
    for (int f = 0; f < 4; ++f) c->stats[f].launches += c->g_launch[f];
  }
  return TN_OK;
}

tn_status check_planned(tn_ctx* c, bool need_device = true) {
  if (!c) return fail(TN_ERR_USAGE, "null context");
  if (!c->planned) return fail(TN_ERR_USAGE, "call tn_set_slices after tn_set_path first");
  if (need_device && c->host_only) return fail(TN_ERR_USAGE, "host-only context (device -1) cannot execute");
  return TN_OK;
}

// leaf layout: [group][remaining labels...] row-major; device element e <- host complex leaf_src[e]
tn_status build_leaves(tn_ctx* c) {
  c->leaf_views.assign(c->n_tensors, View());
  c->leaf_src.clear();
  c->leaf_begin.assign(c->n_tensors, 0);
  int64_t cur = 0;
  for (int t = 0; t < c->n_tensors; ++t) {
    const auto& L = c->labels[t];
    const auto& D = c->dims[t];
    const int r = (int)L.size();
    std::vector<int64_t> hstride(r);
    int64_t s = 1;
    for (int p = r - 1; p >= 0; --p) { hstride[p] = s; s *= D[p]; }
    std::vector<int> open_pos, rest_pos;
    for (int p = 0; p < r; ++p) (c->qubit_of.count(L[p]) ? open_pos : rest_pos).push_back(p);
    std::sort(open_pos.begin(), open_pos.end(),
              [&](int a, int b) { return c->qubit_of[L[a]] < c->qubit_of[L[b]]; });
    View v;
    v.buf = 0;
    v.leaf = t;
    v.off = cur;
    std::vector<uint64_t> table{0};
    if (!open_pos.empty()) {
      for (int p : open_pos) v.q.push_back(c->qubit_of[L[p]]);
      table = table_for(c, v.q);
      v.table = table;
    }
    int64_t rest_elems = 1;
    for (int p : rest_pos) rest_elems *= D[p];
    if (!open_pos.empty()) v.dims.push_back({GROUP, (int64_t)table.size(), 0});
    for (int p : rest_pos) v.dims.push_back({L[p], D[p], 0});
    contiguous_strides(v.dims);
    c->leaf_begin[t] = cur;
    for (size_t g = 0; g < table.size(); ++g) {
      int64_t base = c->data_off[t];
      const int nq = (int)open_pos.size();
      for (int a = 0; a < nq; ++a) base += (int64_t)((table[g] >> (nq - 1 - a)) & 1ull) * hstride[open_pos[a]];
      // enumerate rest digits row-major
      std::vector<int64_t> dig(rest_pos.size(), 0);
      for (int64_t e = 0; e < rest_elems; ++e) {
        int64_t off = base;
        for (size_t a = 0; a < rest_pos.size(); ++a) off += dig[a] * hstride[rest_pos[a]];
        c->leaf_src.push_back(off);
        for (int a = (int)rest_pos.size() - 1; a >= 0; --a) {
          if (++dig[a] < D[rest_pos[a]]) break;
          dig[a] = 0;
        }
      }
    }
    cur += (int64_t)table.size() * rest_elems;
    c->leaf_views[t] = v;
  }
  c->leaf_elems = cur;
  return TN_OK;
}

tn_status upload_leaves(tn_ctx* c, const double* data) {
  if (!c->h_leaf_pinned) TN_CUDA(cudaMallocHost(&c->h_leaf_pinned, std::max<int64_t>(c->leaf_elems, 1) * sizeof(float2)));
  if (!c->d_leaf) {
    void* q = nullptr;
    tn_status st = mem_alloc(c, &q, std::max<int64_t>(c->leaf_elems, 1) * sizeof(float2));
    if (st) return st;
    c->d_leaf = reinterpret_cast<float2*>(q);
  }
  // the previous upload may still be in flight from the pinned buffer
  TN_CUDA(cudaStreamSynchronize(c->stream));
  c->leaf_absmax.assign(c->n_tensors, 0.f);
  for (int t = 0; t < c->n_tensors; ++t) {
    const int64_t b = c->leaf_begin[t];
    const int64_t e = (t + 1 < c->n_tensors) ? c->leaf_begin[t + 1] : c->leaf_elems;
    float m = 0.f;
    for (int64_t x = b; x < e; ++x) {
      const int64_t src = c->leaf_src[x];
      float2 v = make_float2((float)data[2 * src], (float)data[2 * src + 1]);
      c->h_leaf_pinned[x] = v;
      m = std::max(m, std::max(std::fabs(v.x), std::fabs(v.y)));
    }
    c->leaf_absmax[t] = m;
  }
  TN_CUDA(cudaMemcpyAsync(c->d_leaf, c->h_leaf_pinned, c->leaf_elems * sizeof(float2),
                          cudaMemcpyHostToDevice, c->stream));
  if (c->d_absmax) {
    TN_CUDA(cudaMemcpyAsync(c->d_absmax, c->leaf_absmax.data(), c->n_tensors * 4,
                            cudaMemcpyHostToDevice, c->stream));
  }
  return TN_OK;
}

void json_u64_list(std::string& o, const std::vector<int32_t>& v) {
  if (v.size() <= 65536) {
    o += "[";
    for (size_t i = 0; i < v.size(); ++i) { if (i) o += ","; o += std::to_string(v[i]); }
    o += "]";
  } else {
    uint64_t h = 1469598103934665603ull;
    for (int32_t x : v) { h ^= (uint32_t)x; h *= 1099511628211ull; }
    o += "{\"len\":" + std::to_string(v.size()) + ",\"fnv1a\":\"" + std::to_string(h) + "\"}";
  }
}

}  // namespace

// ====================================================================== C ABI

extern "C" {

const char* tn_last_error(void) { return g_err.c_str(); }
const char* tn_version(void) { return "tn-b200 0.1 (sm_100a tcgen05)"; }

tn_status tn_create(tn_ctx** out, int device, const tn_allocator* allocator, void* cuda_stream) {
  if (!out) return fail(TN_ERR_USAGE, "out is NULL");
  *out = nullptr;
  if (allocator && (!allocator->alloc || !allocator->free))
    return fail(TN_ERR_USAGE, "tn_allocator needs both alloc and free");
  tn::refresh_knobs();
  if (device == -1) {
    tn_ctx* c = new tn_ctx();
    c->host_only = true;
    c->debug_plan = env_int("TN_DEBUG_PLAN", 0) != 0;
    c->chain_mode = env_int("TN_CHAIN", 1);
    c->chain_maxbits = env_int("TN_CHAIN_MAXBITS", 8);
    c->chain_min_save = 16.0 * std::ldexp(1.0, env_int("TN_CHAIN_MIN_SAVE_LOG2", 30));
    c->device = -1;
    *out = c;
    return TN_OK;
  }
  int n = 0;
  TN_CUDA(cudaGetDeviceCount(&n));
  if (device < 0 || device >= n) return fail(TN_ERR_USAGE, "bad device index");
  TN_CUDA(cudaSetDevice(device));
  cudaDeviceProp prop;
  TN_CUDA(cudaGetDeviceProperties(&prop, device));
  if (prop.major != 10) return fail(TN_ERR_CUDA, std::string("sm_100a device required, got ") + prop.name);
  tn_ctx* c = new tn_ctx();
  c->device = device;
  c->stream = reinterpret_cast<cudaStream_t>(cuda_stream);
  if (allocator) { c->alloc = *allocator; c->has_alloc = true; }
  c->num_sms = prop.multiProcessorCount;
  c->kchunk3 = env_int("TN_KCHUNK3", 1);
  c->kchunk3_short = env_int("TN_KCHUNK3_SHORT", c->kchunk3);
  c->shortk_max = env_int("TN_SHORTK_MAX", 16);
  // 1-pass: whole K in TMEM (promoting every 4 k-blocks costs 10 % and only moves the
  // all-1-pass C4 error from 2.9e-3 to 2.3e-3: fp16 operand rounding dominates there)
  c->kchunk1 = env_int("TN_KCHUNK1", 0);
  c->autotune = env_int("TN_AUTOTUNE", 1) != 0;
  c->use_graphs = env_int("TN_GRAPHS", 1) != 0;
  c->simt_force = env_int("TN_SIMT_VARIANT", -1);
  c->group_m = env_int("TN_GEMM_GROUP", 8);   // best of {1,8,16,32} on 8192^2 x 16384
  c->debug_plan = env_int("TN_DEBUG_PLAN", 0) != 0;
  c->chain_mode = env_int("TN_CHAIN", 1);
  c->chain_maxbits = env_int("TN_CHAIN_MAXBITS", 8);
  c->chain_min_save = 16.0 * std::ldexp(1.0, env_int("TN_CHAIN_MIN_SAVE_LOG2", 30));
  *out = c;
  return TN_OK;
}

void tn_destroy(tn_ctx* c) {
  if (!c) return;
  if (c->host_only) { delete c; return; }
  cudaSetDevice(c->device);
  cudaStreamSynchronize(c->stream);
  for (auto& p : c->pending) { cudaEventDestroy(p.a); cudaEventDestroy(p.b); }
  free_dev(c);
  if (c->cap_stream) cudaStreamDestroy(c->cap_stream);
  mem_free(c, c->d_leaf);
  if (c->h_leaf_pinned) cudaFreeHost(c->h_leaf_pinned);
  for (auto& kv : std::unordered_map<void*, size_t>(c->owned)) mem_free(c, kv.first);
  delete c;
}

tn_status tn_load_network(tn_ctx* c, int32_t n_tensors, const int32_t* ranks, const int64_t* labels,
                          const int64_t* dims, const double* data, int32_t n_open,
                          const int64_t* open_labels, int64_t n_samples, const uint8_t* samples) {
  if (!c) return fail(TN_ERR_USAGE, "null context");
  if (n_tensors < 1 || !ranks || !data) return fail(TN_ERR_USAGE, "bad network arguments");
  if (!c->host_only) TN_CUDA(cudaSetDevice(c->device));
  free_dev(c);
  c->loaded = c->pathed = false;
  c->n_tensors = n_tensors;
  c->labels.assign(n_tensors, {});
  c->dims.assign(n_tensors, {});
  c->data_off.assign(n_tensors, 0);
  c->dim_of.clear();
  c->count_of.clear();
  c->qubit_of.clear();
  int64_t li = 0, doff = 0;
  for (int t = 0; t < n_tensors; ++t) {
    if (ranks[t] < 0) return fail(TN_ERR_DATA, "negative rank");
    int64_t sz = 1;
    std::unordered_set<int64_t> seen;
    for (int p = 0; p < ranks[t]; ++p, ++li) {
      const int64_t l = labels[li], d = dims[li];
      if (l == GROUP) return fail(TN_ERR_DATA, "reserved label value");
      if (d < 1) return fail(TN_ERR_DATA, "dimension < 1");
      if (!seen.insert(l).second)
        return fail(TN_ERR_DATA, "label " + std::to_string(l) + " repeated in tensor " + std::to_string(t));
      auto it = c->dim_of.find(l);
      if (it != c->dim_of.end() && it->second != d)
        return fail(TN_ERR_DATA, "dimension mismatch on label " + std::to_string(l));
      c->dim_of[l] = d;
      c->count_of[l]++;
      c->labels[t].push_back(l);
      c->dims[t].push_back(d);
      sz *= d;
    }
    c->data_off[t] = doff;
    doff += sz;
  }
  c->n_data = doff;
  if (n_open < 0 || n_open > 64) return fail(TN_ERR_DATA, "n_open must be in [0, 64]");
  c->n_open = n_open;
  c->open_labels.assign(open_labels, open_labels + n_open);
  for (int q = 0; q < n_open; ++q) {
    const int64_t l = open_labels[q];
    if (!c->count_of.count(l) || c->count_of[l] != 1)
      return fail(TN_ERR_DATA, "open label " + std::to_string(l) + " must appear on exactly one tensor");
    if (c->dim_of[l] != 2) return fail(TN_ERR_DATA, "open bonds must have dimension 2");
    if (c->qubit_of.count(l)) return fail(TN_ERR_DATA, "open label listed twice");
    c->qubit_of[l] = q;
  }
  for (auto& kv : c->count_of)
    if (!c->qubit_of.count(kv.first) && kv.second != 2)
      return fail(TN_ERR_DATA, "closed label " + std::to_string(kv.first) + " appears " +
                                   std::to_string(kv.second) + " times (must be 2)");
  c->packed.clear();
  if (!samples) {
    if (n_open > 24) return fail(TN_ERR_DATA, "full-state output limited to n_open <= 24");
    c->full_state = true;
    c->n_samples = n_open > 0 ? (int64_t(1) << n_open) : 1;
    for (int64_t s = 0; s < c->n_samples; ++s) c->packed.push_back((uint64_t)s);
  } else {
    if (n_samples < 1) return fail(TN_ERR_DATA, "n_samples must be >= 1");
    c->full_state = false;
    c->n_samples = n_samples;
    c->packed.resize(n_samples);
    for (int64_t s = 0; s < n_samples; ++s) {
      uint64_t v = 0;
      for (int q = 0; q < n_open; ++q) {
        const uint8_t b = samples[s * n_open + q];
        if (b > 1) return fail(TN_ERR_DATA, "sample bytes must be 0 or 1");
        v = (v << 1) | b;
      }
      c->packed[s] = v;
    }
  }
  tn_status st = build_leaves(c);
  if (st) return st;
  if (c->host_only) {
    c->leaf_absmax.assign(c->n_tensors, 0.f);
    c->loaded = true;
    return TN_OK;
  }
  if (c->d_leaf) { cudaStreamSynchronize(c->stream); mem_free(c, c->d_leaf); c->d_leaf = nullptr; }
  if (c->h_leaf_pinned) { cudaFreeHost(c->h_leaf_pinned); c->h_leaf_pinned = nullptr; }
  st = upload_leaves(c, data);
  if (st) return st;
  c->loaded = true;
  return TN_OK;
}

tn_status tn_upload_tensors(tn_ctx* c, const double* data) {
  if (!c || !c->loaded) return fail(TN_ERR_USAGE, "load a network first");
  if (c->host_only) return fail(TN_ERR_USAGE, "host-only context (device -1) cannot execute");
  if (!data) return fail(TN_ERR_USAGE, "data is NULL");
  const std::vector<float> before = c->leaf_absmax;
  tn_status st = upload_leaves(c, data);
  if (st) return st;
  // a leaf's absmax moved by more than 2x: restart the delayed-scaling history; the
  // next slice runs unfused and re-seeds it (SIMT variants and the captured graph are
  // kept).  Growth would eat the 32x margin; a shrink would leave the history (a
  // running max) stale-large, the planes' exponent too low and the fp16 lo plane
  // (then hi) in subnormals.  Smaller changes keep the history (the margin and the
  // overflow check cover the slice-to-slice variation).
  bool moved = before.size() != c->leaf_absmax.size();
  for (size_t t = 0; t < before.size() && !moved; ++t)
    moved = c->leaf_absmax[t] > 2.f * before[t] || 2.f * c->leaf_absmax[t] < before[t];
  if (c->planned && c->d_hist && moved) {
    TN_CUDA(cudaMemsetAsync(c->d_hist, 0, c->steps.size() * sizeof(unsigned), c->stream));
    c->tuned = false;
  }
  return TN_OK;
}

tn_status tn_set_path(tn_ctx* c, int32_t n_steps, const int32_t* pairs) {
  if (!c || !c->loaded) return fail(TN_ERR_USAGE, "load a network first");
  free_dev(c);
  c->pathed = false;
  if (n_steps != c->n_tensors - 1)
    return fail(TN_ERR_DATA, "path must have N-1 = " + std::to_string(c->n_tensors - 1) + " steps");
  std::vector<char> alive(c->n_tensors, 1);
  c->path.clear();
  for (int s = 0; s < n_steps; ++s) {
    const int i = pairs[2 * s], j = pairs[2 * s + 1];
    if (i < 0 || j < 0 || i >= c->n_tensors || j >= c->n_tensors || i == j || !alive[i] || !alive[j])
      return fail(TN_ERR_DATA, "path step " + std::to_string(s) + " (" + std::to_string(i) + "," +
                                   std::to_string(j) + ") references a retired or unknown id");
    alive[j] = 0;
    c->path.push_back({i, j});
  }
  c->pathed = true;
  return TN_OK;
}

tn_status tn_set_slices(tn_ctx* c, int32_t n_sliced, const int64_t* sliced_labels, int64_t* n_slices_out) {
  if (!c || !c->pathed) return fail(TN_ERR_USAGE, "call tn_set_path first");
  if (!c->host_only) TN_CUDA(cudaSetDevice(c->device));
  std::unordered_set<int64_t> seen;
  c->sliced.clear();
  c->n_slices = 1;
  for (int p = 0; p < n_sliced; ++p) {
    const int64_t l = sliced_labels[p];
    if (!c->dim_of.count(l)) return fail(TN_ERR_DATA, "unknown sliced label " + std::to_string(l));
    if (c->qubit_of.count(l)) return fail(TN_ERR_DATA, "open label " + std::to_string(l) + " cannot be sliced");
    if (!seen.insert(l).second) return fail(TN_ERR_DATA, "sliced label repeated");
    c->sliced.push_back(l);
    if (c->n_slices > INT64_MAX / c->dim_of[l]) return fail(TN_ERR_DATA, "too many slices");
    c->n_slices *= c->dim_of[l];
  }
  // planning runs twice when gate folding applies: the first pass decides the folds,
  // the second keeps the folded steps' inputs live until their consumers (fold_hint)
  c->fold_hint.clear();
  c->chain_hint.clear();
  c->replan = false;
  tn_status st = build_plan(c);
  if (!st && !c->fold_hint.empty()) st = build_plan(c);
  // skinny chains are decided once the folds are: one more pass keeps their inputs live
  if (!st && c->replan) { c->replan = false; st = build_plan(c); }
  if (!st && c->replan) { c->replan = false; st = build_plan(c); }
  if (st || c->replan) {
    free_dev(c);
    c->fold_hint.clear();
    c->chain_hint.clear();
    return st ? st : fail(TN_ERR_INTERNAL, "planning did not converge");
  }
  if (n_slices_out) *n_slices_out = c->n_slices;
  return TN_OK;
}

tn_status tn_contract(tn_ctx* c, int64_t b, int64_t e, tn_precision prec, int32_t topk) {
  tn_status st = check_planned(c);
  if (st) return st;
  if (b < 0 || e > c->n_slices || b > e)
    return fail(TN_ERR_DATA, "slice range [" + std::to_string(b) + "," + std::to_string(e) +
                                 ") outside [0," + std::to_string(c->n_slices) + ")");
  if (prec != TN_PREC_EXTENDED && prec != TN_PREC_MIXED) return fail(TN_ERR_USAGE, "bad precision");
  TN_CUDA(cudaSetDevice(c->device));
  return run_slices(c, b, e, prec, topk);
}

tn_status tn_reset_accumulator(tn_ctx* c) {
  tn_status st = check_planned(c);
  if (st) return st;
  TN_CUDA(cudaMemsetAsync(c->d_acc, 0, c->acc_elems * sizeof(double2), c->stream));
  TN_CUDA(cudaMemsetAsync(c->d_flag, 0, sizeof(int), c->stream));
  return TN_OK;
}

// A fused producer whose delayed-scaling margin (32x over the largest absmax of the
// slices before) was exceeded wrote saturated fp16 planes: fail loudly, never return
// such a sum (rerun with TN_FUSE_PLANES=0).
tn_status check_plane_overflow(tn_ctx* c) {
  int flag = 0;
  TN_CUDA(cudaMemcpyAsync(&flag, c->d_flag, sizeof(int), cudaMemcpyDeviceToHost, c->stream));
  TN_CUDA(cudaStreamSynchronize(c->stream));
  if (flag) return fail(TN_ERR_DATA, "fp16 plane overflow in a fused producer epilogue (delayed-scaling "
                                     "margin exceeded); rerun with TN_FUSE_PLANES=0");
  return TN_OK;
}

tn_status tn_sum_slices(tn_ctx* c, double* out, int64_t n_out) {
  tn_status st = check_planned(c);
  if (st) return st;
  if (n_out != c->n_out) return fail(TN_ERR_USAGE, "n_out must be " + std::to_string(c->n_out));
  if (!out) return fail(TN_ERR_USAGE, "out is NULL");
  TN_CUDA(cudaSetDevice(c->device));
  // asynchronous: the gather itself turns a set overflow flag into NaN output
  TN_CUDA(tn::launch_gather_out(c->d_acc, c->d_out_pos, reinterpret_cast<double2*>(out), n_out, c->d_flag,
                                c->stream));
  return TN_OK;
}

tn_status tn_sum_slices_host(tn_ctx* c, double* out_host, int64_t n_out) {
  tn_status st = check_planned(c);
  if (st) return st;
  if ((st = check_plane_overflow(c))) return st;
  if (n_out != c->n_out) return fail(TN_ERR_USAGE, "n_out must be " + std::to_string(c->n_out));
  if (!out_host) return fail(TN_ERR_USAGE, "out is NULL");
  TN_CUDA(tn::launch_gather_out(c->d_acc, c->d_out_pos, c->d_gather, n_out, nullptr, c->stream));
  TN_CUDA(cudaMemcpyAsync(out_host, c->d_gather, n_out * sizeof(double2), cudaMemcpyDeviceToHost, c->stream));
  TN_CUDA(cudaStreamSynchronize(c->stream));
  return TN_OK;
}

int tn_last_overflow(tn_ctx* c) {
  if (!c || c->host_only || !c->planned) return -1;
  if (cudaSetDevice(c->device) != cudaSuccess) return -1;
  int flag = 0;
  if (cudaMemcpyAsync(&flag, c->d_flag, sizeof(int), cudaMemcpyDeviceToHost, c->stream) != cudaSuccess ||
      cudaStreamSynchronize(c->stream) != cudaSuccess)
    return -1;
  return flag ? 1 : 0;
}

tn_status tn_get_info(tn_ctx* c, tn_info* info) {
  tn_status st = check_planned(c, false);
  if (st) return st;
  info->n_slices = c->n_slices;
  info->n_out = c->n_out;
  info->n_steps = (int32_t)c->steps.size();
  int ntc = 0;
  for (auto& s : c->steps) ntc += s.tc;
  info->n_tc_steps = ntc;
  info->flops_per_slice = c->flops_per_slice;
  info->tc_flops_per_slice = c->tc_flops;
  info->bytes_per_slice = c->bytes_per_slice;
  info->peak_elements = c->peak;
  info->device_bytes = c->device_bytes;
  info->arena_bytes = c->arena_elems * (int64_t)sizeof(float2);
  info->scratch_bytes = c->scratch_bytes;
  info->graph_replays = c->graph_launches;
  return TN_OK;
}

tn_status tn_plan_json(tn_ctx* c, char* buf, size_t cap, size_t* len) {
  tn_status st = check_planned(c, false);
  if (st) return st;
  std::string o = "{\"n_slices\":" + std::to_string(c->n_slices) + ",\"sliced\":[";
  for (size_t p = 0; p < c->sliced.size(); ++p) { if (p) o += ","; o += std::to_string(c->sliced[p]); }
  o += "],\"steps\":[";
  for (size_t s = 0; s < c->steps.size(); ++s) {
    const StepPlan& sp = c->steps[s];
    if (s) o += ",";
    char b[512];
    snprintf(b, sizeof(b),
             "{\"i\":%d,\"j\":%d,\"J\":%lld,\"m\":%lld,\"n\":%lld,\"k\":%lld,\"tcc\":%.17g,"
             "\"tmc\":%.17g,\"route\":\"%s\",\"swap\":%s,\"mode\":%d,\"grouped\":%s,"
             "\"gathered_rows\":%lld,\"out_gen\":%s,\"prep\":[%d,%d],\"planes_out\":%s,\"dense_merge\":%s,\"folded\":%s,\"wd_staged\":%s,\"chain\":%d,\"chained\":%s,\"ia\":",
             sp.i, sp.j, (long long)sp.J, (long long)sp.m, (long long)sp.n, (long long)sp.k, sp.tcc,
             sp.tmc, sp.tc ? "tcgen05" : "simt", sp.swap ? "true" : "false", sp.mode,
             sp.grouped ? "true" : "false", (long long)sp.g_rows, sp.out_gen ? "true" : "false",
             sp.tc ? (sp.skip_prep[0] ? -1 : sp.r_fast[0]) : -1,
             sp.tc ? (sp.skip_prep[1] ? -1 : sp.r_fast[1]) : -1, sp.planes_consumer >= 0 ? "true" : "false",
             sp.dense_merge ? "true" : "false", sp.folded ? "true" : "false",
             (!sp.tc && sp.hdesc.wd_ok) ? "true" : "false", sp.chain, sp.chained ? "true" : "false");
    o += b;
    if (sp.merge) json_u64_list(o, sp.ia); else o += "null";
    o += ",\"ib\":";
    if (sp.merge) json_u64_list(o, sp.ib); else o += "null";
    if (sp.grouped) {
      o += ",\"g_rowmap\":";
      json_u64_list(o, sp.g_rowmap);
      o += ",\"g_blk\":";
      json_u64_list(o, sp.g_blk);
    }
    o += "}";
  }
  o += "],\"reorder\":{\"mode\":" + std::to_string(c->reorder_mode) + ",\"topk\":" +
       std::to_string(c->reorder_topk) + ",\"selected\":[";
  bool first = true;
  for (size_t s = 0; s < c->reorder_sel.size(); ++s)
    if (c->reorder_sel[s]) { o += (first ? "" : ",") + std::to_string(s); first = false; }
  o += "],\"modified\":[";
  first = true;
  for (size_t s = 0; s < c->reorder_mod.size(); ++s)
    if (c->reorder_mod[s]) { o += (first ? "" : ",") + std::to_string(s); first = false; }
  o += "]},\"out_pos\":";
  json_u64_list(o, c->out_pos);
  char b[256];
  snprintf(b, sizeof(b), ",\"flops_per_slice\":%.17g,\"tc_flops_per_slice\":%.17g,\"peak_elements\":%.17g}",
           c->flops_per_slice, c->tc_flops, c->peak);
  o += b;
  if (len) *len = o.size();
  if (buf && cap) {
    size_t n = std::min(cap - 1, o.size());
    memcpy(buf, o.data(), n);
    buf[n] = 0;
  }
  return TN_OK;
}

tn_status tn_set_profiling(tn_ctx* c, int enabled) {
  if (!c) return fail(TN_ERR_USAGE, "null context");
  c->profiling = enabled != 0;
  return TN_OK;
}

static tn_status drain_pending(tn_ctx* c) {
  if (c->pending.empty()) return TN_OK;
  TN_CUDA(cudaStreamSynchronize(c->stream));
  for (auto& v : c->step_ms)
    if (v.size() < c->steps.size()) v.resize(c->steps.size(), 0.0);
  for (auto& p : c->pending) {
    float ms = 0.f;
    cudaEventElapsedTime(&ms, p.a, p.b);
    c->stats[p.family].ms += ms;
    c->stats[p.family].flops += p.flops;
    c->stats[p.family].bytes += p.bytes;
    if (p.step >= 0 && p.step < (int)c->steps.size()) c->step_ms[p.family][p.step] += ms;
    cudaEventDestroy(p.a);
    cudaEventDestroy(p.b);
  }
  c->pending.clear();
  return TN_OK;
}

tn_status tn_get_step_stats(tn_ctx* c, int family, int64_t n, double* ms_out) {
  if (!c || n < 0 || (n > 0 && !ms_out) || family < -1 || family > 3)
    return fail(TN_ERR_USAGE, "bad arguments");
  tn_status st = drain_pending(c);
  if (st) return st;
  for (int64_t s = 0; s < n; ++s) {
    double v = 0.0;
    for (int f = 0; f < 4; ++f)
      if ((family < 0 || family == f) && s < (int64_t)c->step_ms[f].size()) v += c->step_ms[f][s];
    ms_out[s] = v;
  }
  return TN_OK;
}

tn_status tn_get_kernel_stats(tn_ctx* c, int family, tn_kernel_stats* out) {
  if (!c || family < 0 || family > 3 || !out) return fail(TN_ERR_USAGE, "bad arguments");
  tn_status st = drain_pending(c);
  if (st) return st;
  out->launches = c->stats[family].launches;
  out->ms = c->stats[family].ms;
  out->flops = c->stats[family].flops;
  out->bytes = c->stats[family].bytes;
  return TN_OK;
}

tn_status tn_reset_kernel_stats(tn_ctx* c) {
  if (!c) return fail(TN_ERR_USAGE, "null context");
  tn_kernel_stats tmp;
  tn_get_kernel_stats(c, 0, &tmp);
  for (auto& s : c->stats) s = KStats();
  for (auto& v : c->step_ms) v.assign(c->steps.size(), 0.0);
  return TN_OK;
}

tn_status tn_cgemm(tn_ctx* c, const float* A, const float* B, float* C, int64_t J, int64_t m, int64_t n,
                   int64_t k, int64_t ga, int64_t gb, const int32_t* ia, const int32_t* ib, int passes,
                   int force_simt, int format) {
  if (!c) return fail(TN_ERR_USAGE, "null context");
  if (c->host_only) return fail(TN_ERR_USAGE, "host-only context (device -1) cannot execute");
  if (J < 1 || m < 1 || n < 1 || k < 1 || ga < 1 || gb < 1) return fail(TN_ERR_USAGE, "bad sizes");
  if (passes != 1 && passes != 3) return fail(TN_ERR_USAGE, "passes must be 1 or 3");
  if (format < 0 || format > 2) return fail(TN_ERR_USAGE, "format must be 0 (fp16), 1 (bf16) or 2 (tf32)");
  TN_CUDA(cudaSetDevice(c->device));
  cudaStream_t sm = c->stream;
  unsigned* am = nullptr;
  int* sc = nullptr;
  tn_status st0 = mem_alloc(c, reinterpret_cast<void**>(&am), 16);
  if (!st0) st0 = mem_alloc(c, reinterpret_cast<void**>(&sc), 16);
  if (st0) { mem_free(c, am); return st0; }
  TN_CUDA(cudaMemsetAsync(am, 0, 16, sm));
  const float2* A2 = reinterpret_cast<const float2*>(A);
  const float2* B2 = reinterpret_cast<const float2*>(B);
  TN_CUDA(tn::launch_absmax(A2, ga * m * k, am, sm));
  TN_CUDA(tn::launch_absmax(B2, gb * n * k, am + 1, sm));
  tn_status result = TN_OK;
  if (force_simt) {
    tn::EinsumDesc e;
    memset(&e, 0, sizeof(e));
    e.A = A2; e.B = B2; e.C = reinterpret_cast<float2*>(C);
    e.a_leaf = e.b_leaf = -1;
    e.J = J; e.ia = ia; e.ib = ib; e.a_gs = m * k; e.b_gs = n * k;
    e.M = m; e.N = n; e.K = k;
    e.nm = 1; e.m_ext[0] = m; e.m_sa[0] = k;
    e.nn = 1; e.n_ext[0] = n; e.n_sb[0] = k;
    e.nk = 1; e.k_ext[0] = k; e.k_sa[0] = 1; e.k_sb[0] = 1;
    fill_shifts(e);
    tn::EinsumDesc* d = nullptr;
    if (tn_status st1 = mem_alloc(c, reinterpret_cast<void**>(&d), sizeof(e))) return st1;
    TN_CUDA(cudaMemcpyAsync(d, &e, sizeof(e), cudaMemcpyHostToDevice, sm));
    TN_CUDA(tn::launch_einsum(d, e, nullptr, sm));
    TN_CUDA(cudaStreamSynchronize(sm));
    mem_free(c, d);
  } else {
    const int64_t Kpad = (k + 7) / 8 * 8;
    const int64_t esz = format == 2 ? 4 : 2;
    const int64_t b0 = (4 * ga * m * Kpad * esz + 1023) / 1024 * 1024;
    const int64_t b1 = (4 * gb * n * Kpad * esz + 1023) / 1024 * 1024;
    uint8_t* scr = nullptr;
    if (tn_status st1 = mem_alloc(c, reinterpret_cast<void**>(&scr), b0 + b1)) return st1;
    tn::PrepDesc p[2];
    tn::GemmArgs g;
    memset(&g, 0, sizeof(g));
    char err[256];
    for (int side = 0; side < 2; ++side) {
      memset(&p[side], 0, sizeof(tn::PrepDesc));
      const int64_t R = side ? n : m, G = side ? gb : ga;
      p[side].src = side ? B2 : A2;
      p[side].leaf = -1;
      p[side].G = G; p[side].R = R; p[side].K = k; p[side].Kpad = Kpad;
      p[side].g_stride = R * k;
      p[side].nr = 1; p[side].r_ext[0] = R; p[side].r_s[0] = k;
      p[side].nk = 1; p[side].k_ext[0] = k; p[side].k_s[0] = 1;
      p[side].read_r_fast = 0;
      p[side].dst = reinterpret_cast<__half*>(scr + (side ? b0 : 0));
      p[side].plane_elems = G * R * Kpad;
      p[side].absmax_in = am + side;
      p[side].scale_out = sc + side;
      if (!tn::encode_plane_map(side ? &g.mapB : &g.mapA, p[side].dst, Kpad, R, G, 4, 128, err, sizeof(err),
                                format) ||
          (side == 1 && !tn::encode_plane_map(&g.mapB2, p[side].dst, Kpad, R, G, 4, 64, err, sizeof(err),
                                              format))) {
        mem_free(c, scr);
        return fail(TN_ERR_INTERNAL, err);
      }
    }
    tn::PrepDesc* dp = nullptr;
    if (tn_status st1 = mem_alloc(c, reinterpret_cast<void**>(&dp), sizeof(p))) return st1;
    TN_CUDA(cudaMemcpyAsync(dp, p, sizeof(p), cudaMemcpyHostToDevice, sm));
    const int planes = passes == 3 ? 4 : 2;
    if (format == 0) {
      TN_CUDA(tn::launch_prep(dp, p[0].plane_elems, planes, 0, 0, nullptr, sm));
      TN_CUDA(tn::launch_prep(dp + 1, p[1].plane_elems, planes, 0, 0, nullptr, sm));
    } else {
      TN_CUDA(tn::launch_prep_fmt(A2, p[0].dst, ga * m, k, Kpad, planes, format, am, sc, sm));
      TN_CUDA(tn::launch_prep_fmt(B2, p[1].dst, gb * n, k, Kpad, planes, format, am + 1, sc + 1, sm));
    }
    g.J = (int32_t)J; g.M = (int32_t)m; g.N = (int32_t)n; g.K = (int32_t)k;
    g.ia = ia; g.ib = ib;
    g.C = reinterpret_cast<float2*>(C);
    g.scaleA = sc; g.scaleB = sc + 1;
    g.absmax_out = nullptr; g.acc = nullptr;
    g.tiles_m = (int32_t)((m + 127) / 128);
    g.tiles_n = (int32_t)((n + 127) / 128);
    g.n_tiles = (int64_t)g.tiles_m * g.tiles_n * J;
    g.kchunk = passes == 3 ? c->kchunk3 : c->kchunk1;
    g.group_m = c->group_m;
    g.use_pair = (format == 0 && tn::gemm_pair_ok(g, tn::g_knobs.pair_min_m)) ? 1 : 0;
    if (!c->d_wave)
      if (tn_status st1 = mem_alloc(c, reinterpret_cast<void**>(&c->d_wave), sizeof(unsigned long long))) return st1;
    g.wave_ctr = c->d_wave;
    g.wave_sync = (env_int("TN_WAVE_SYNC", 1) && k >= 1024) ? 1 : 0;
    {
      Timer tm(c, 0, 8.0 * (double)J * m * n * k, 8.0 * (double)(ga * m * k + gb * n * k + J * m * n));
      TN_CUDA(tn::launch_gemm(g, passes, c->num_sms, sm, format));
    }
    cudaError_t e = cudaStreamSynchronize(sm);
    mem_free(c, dp);
    mem_free(c, scr);
    if (e != cudaSuccess) result = fail(TN_ERR_CUDA, std::string("cgemm: ") + cudaGetErrorString(e));
  }
  mem_free(c, am);
  mem_free(c, sc);
  return result;
}

}  // extern "C"
