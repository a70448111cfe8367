// Distributed evaluation across G = 2^s0 GPUs, one process (rank) per GPU
// (SURVEY 8(e)).  The reference is single-process (SPEC.md:409 non-goal);
// this is the domain decomposition the north star asks for.
//
// The pyramid is partitioned at split step s0 = log2 G: rank r owns the
// subtree below top-split segment r, i.e. a contiguous box range at every
// level l with 2l >= s0 (Part in engine.h); the levels above are shared and
// computed redundantly.  Phases (each a C-ABI call; the collectives between
// them are issued by the caller through torch.distributed -- NCCL over
// NVLink/NVSwitch -- on the same CUDA stream):
//
//  1. load       shard of the input -> 32-byte records {x, y, g, orig index};
//                local bounding box                     [allreduce MIN]
//  2. top split  s0 median steps, each an exact distributed radix select
//                (8 rounds of 8-bit digits of the order-preserving key)
//                                                       [allreduce SUM x 8]
//                then the tie quota across ranks        [allgather]
//                and a stable local partition (canonical order = ascending
//                original index, because rank r holds indices before rank
//                r+1 and every step is stable)
//  3. exchange   segment t -> rank t                    [all-to-all]
//  4. subtree    run_tree below step s0 with the given root rectangle,
//                writing into global-size tree-order arrays
//  5. geometry   owned boxes of every owned level       [allgather]
//  6. lists      connectivity for owned targets only; import sets: source
//                boxes (M2L, M2P) and source leaves (P2P, P2L) owned by
//                other ranks                            [all-to-all x 2]
//  7. particles  halo leaves                            [all-to-all]
//  8. upward     P2M, P2L, M2M on owned levels; level-ltop multipoles
//                [allgather]; M2M on the shared levels
//  9. multipoles halo boxes                             [all-to-all]
// 10. downward   M2L (owned + shared targets), L2L, L2P/M2P, P2P -> owned
//                values in tree order + their original indices.
//
// Every target is computed by exactly one rank from the same inputs and
// with the same per-target accumulation order as on one GPU; the tree and
// the lists are identical to the single-GPU ones (tests compare them).
#include <cub/device/device_radix_sort.cuh>
#include <cub/device/device_scan.cuh>
#include <cub/device/device_select.cuh>
#include <cub/iterator/counting_input_iterator.cuh>

#include <algorithm>
#include <cmath>
#include <cstdio>

#include "context.h"

namespace fmm {

namespace {

struct Rec {
  double x, y, g;
  long long idx;
};

inline unsigned nblk(long long n, int t) { return (unsigned)((n + t - 1) / t); }

// -------------------------------------------------------------------------
// load: records + local bounding box (min x, -max x, min y, -max y)
__global__ void k_rec_load(long long n, const double2* __restrict__ pos,
                           const double* __restrict__ g, long long idx_base, Rec* rec,
                           unsigned long long* bbkeys) {
  pdl_enter();
  double x0 = INFINITY, x1 = -INFINITY, y0 = INFINITY, y1 = -INFINITY;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n;
       i += (long long)gridDim.x * blockDim.x) {
    const double2 z = pos[i];
    rec[i] = Rec{z.x, z.y, g ? g[i] : 0.0, idx_base + i};
    x0 = fmin(x0, z.x); x1 = fmax(x1, z.x);
    y0 = fmin(y0, z.y); y1 = fmax(y1, z.y);
  }
  for (int d = 16; d; d >>= 1) {
    x0 = fmin(x0, __shfl_xor_sync(0xffffffffu, x0, d));
    x1 = fmax(x1, __shfl_xor_sync(0xffffffffu, x1, d));
    y0 = fmin(y0, __shfl_xor_sync(0xffffffffu, y0, d));
    y1 = fmax(y1, __shfl_xor_sync(0xffffffffu, y1, d));
  }
  if ((threadIdx.x & 31) == 0) {
    atomicMin(bbkeys + 0, ordered_key(x0));
    atomicMin(bbkeys + 1, ordered_key(-x1));
    atomicMin(bbkeys + 2, ordered_key(y0));
    atomicMin(bbkeys + 3, ordered_key(-y1));
  }
}

__device__ __forceinline__ double key_to_double(unsigned long long k) {
  const unsigned long long b = (k & 0x8000000000000000ull) ? (k & 0x7fffffffffffffffull) : ~k;
  return __longlong_as_double((long long)b);
}

__global__ void k_bbox_out(const unsigned long long* bbkeys, double* out4) {
  pdl_enter();
  if (threadIdx.x < 4) out4[threadIdx.x] = key_to_double(bbkeys[threadIdx.x]);
}

// -------------------------------------------------------------------------
// distributed exact k-th smallest per segment: 8 rounds of 8-bit digits of
// the order-preserving 64-bit key of the split coordinate
struct SelState {
  unsigned long long prefix;   // digits found so far (high bits)
  long long k_rem;             // rank still to find inside the prefix bucket (1-based)
  long long less;              // keys strictly below the prefix bucket
};

__global__ void k_sel_init(SelState* sel, const long long* __restrict__ kth, int nseg) {
  pdl_enter();
  const int j = blockIdx.x * blockDim.x + threadIdx.x;
  if (j < nseg) sel[j] = SelState{0ull, kth[j], 0};
}

__device__ __forceinline__ unsigned long long rec_key(const Rec& r, bool along_y) {
  return ordered_key(along_y ? r.y : r.x);
}

// histogram of digit `rho` over the records of every segment whose key matches
// the prefix found so far; block-private SMEM histograms (no hot global bins)
__global__ void __launch_bounds__(256)
k_sel_hist(int rho, int nseg, const Rec* __restrict__ rec, const long long* __restrict__ seg_off,
           const unsigned char* __restrict__ axis, const SelState* __restrict__ sel, int* hist) {
  pdl_enter();
  __shared__ int sh[4][256];
  for (int i = threadIdx.x; i < nseg * 256; i += blockDim.x) sh[i >> 8][i & 255] = 0;
  __syncthreads();
  const int shift = 56 - 8 * rho;
  const long long n = seg_off[nseg];
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n;
       i += (long long)gridDim.x * blockDim.x) {
    int j = 0;
    while (j + 1 < nseg && seg_off[j + 1] <= i) ++j;
    const unsigned long long k = rec_key(rec[i], axis[j]);
    const bool match = rho == 0 || (k >> (shift + 8)) == (sel[j].prefix >> (shift + 8));
    if (match) atomicAdd(&sh[j][(k >> shift) & 255], 1);
  }
  __syncthreads();
  for (int i = threadIdx.x; i < nseg * 256; i += blockDim.x)
    if (sh[i >> 8][i & 255]) atomicAdd(&hist[i], sh[i >> 8][i & 255]);
}

// pick the digit holding the k_rem-th key (same result on every rank: the
// histogram is the allreduced one)
__global__ void k_sel_pick(int rho, int nseg, const int* __restrict__ hist, SelState* sel) {
  pdl_enter();
  const int j = threadIdx.x;
  if (j >= nseg) return;
  const int shift = 56 - 8 * rho;
  SelState s = sel[j];
  long long below = 0;
  int d = 0;
  for (; d < 255; ++d) {
    const long long c = hist[j * 256 + d];
    if (below + c >= s.k_rem) break;
    below += c;
  }
  s.prefix |= (unsigned long long)d << shift;
  s.k_rem -= below;
  s.less += below;
  sel[j] = s;
}

// local count of keys equal to the cut, per segment
__global__ void k_eq_count(int nseg, const Rec* __restrict__ rec,
                           const long long* __restrict__ seg_off,
                           const unsigned char* __restrict__ axis, const SelState* __restrict__ sel,
                           int* eq_local, int* eqflag) {
  pdl_enter();
  const long long n = seg_off[nseg];
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n;
       i += (long long)gridDim.x * blockDim.x) {
    int j = 0;
    while (j + 1 < nseg && seg_off[j + 1] <= i) ++j;
    const bool eq = rec_key(rec[i], axis[j]) == sel[j].prefix;
    eqflag[i] = eq;
    if (eq) atomicAdd(&eq_local[j], 1);
  }
}

// sort key 2j + (goes right): left = key < cut, or key == cut among the first
// `quota` equal keys in canonical order (ranks below first, then local order)
__global__ void k_side_keys(int nseg, int G, int rank, const Rec* __restrict__ rec,
                            const long long* __restrict__ seg_off,
                            const unsigned char* __restrict__ axis,
                            const SelState* __restrict__ sel, const int* __restrict__ eq_all,
                            const int* __restrict__ eqpre, unsigned* skey, int* sval) {
  pdl_enter();
  const long long n = seg_off[nseg];
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n;
       i += (long long)gridDim.x * blockDim.x) {
    int j = 0;
    while (j + 1 < nseg && seg_off[j + 1] <= i) ++j;
    const unsigned long long k = rec_key(rec[i], axis[j]);
    const SelState s = sel[j];
    bool left = k < s.prefix;
    if (k == s.prefix) {
      long long before = eqpre[i] - eqpre[seg_off[j]];     // equal keys before i, locally
      for (int q = 0; q < rank; ++q) before += eq_all[q * nseg + j];
      left = before < s.k_rem;                              // k_rem = quota of equal keys
    }
    skey[i] = 2u * j + (left ? 0u : 1u);
    sval[i] = (int)i;
  }
}

__global__ void k_rec_gather(long long n, const int* __restrict__ perm, const Rec* __restrict__ in,
                             Rec* out) {
  pdl_enter();
  const long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (i < n) out[i] = in[perm[i]];
}

__global__ void k_seg_bounds(long long n, int nseg2, const unsigned* __restrict__ skey,
                             long long* seg_off) {
  pdl_enter();
  const long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (i > n) return;
  const long long prev = i == 0 ? -1 : (long long)skey[i - 1];
  const long long cur = i == n ? nseg2 : (long long)skey[i];
  for (long long b = prev + 1; b <= cur; ++b) seg_off[b] = i;
}

// per-segment local bounding box for the top-level degenerate check
__global__ void k_seg_box(int nseg, const Rec* __restrict__ rec,
                          const long long* __restrict__ seg_off, unsigned long long* keys) {
  pdl_enter();
  const long long n = seg_off[nseg];
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n;
       i += (long long)gridDim.x * blockDim.x) {
    int j = 0;
    while (j + 1 < nseg && seg_off[j + 1] <= i) ++j;
    const Rec r = rec[i];
    atomicMin(keys + 4 * j + 0, ordered_key(r.x));
    atomicMin(keys + 4 * j + 1, ordered_key(-r.x));
    atomicMin(keys + 4 * j + 2, ordered_key(r.y));
    atomicMin(keys + 4 * j + 3, ordered_key(-r.y));
  }
}

__global__ void k_keys_out(const unsigned long long* keys, double* out, int n) {
  pdl_enter();
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) out[i] = key_to_double(keys[i]);
}

__global__ void k_rec_unpack(long long n, const Rec* __restrict__ rec, double2* pos, double* g,
                             int* idx) {
  pdl_enter();
  const long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (i >= n) return;
  const Rec r = rec[i];
  pos[i] = make_double2(r.x, r.y);
  g[i] = r.g;
  idx[i] = (int)r.idx;
}

// -------------------------------------------------------------------------
// geometry of owned boxes: pack / unpack {cx, cy, hw, hh, r}
__device__ __forceinline__ void own_slot(long long u, int ltop, int s0, int* l_out,
                                         long long* k_out) {
  int l = ltop;
  while (true) {
    const long long c = 1ll << (2 * l - s0);
    if (u < c) break;
    u -= c;
    ++l;
  }
  *l_out = l;
  *k_out = u;
}

__global__ void k_geo_pack(long long count, int ltop, int s0, int rank, const double* cx,
                           const double* cy, const double* hw, const double* hh,
                           const double* r, double* out) {
  pdl_enter();
  const long long u = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (u >= count) return;
  int l;
  long long k;
  own_slot(u, ltop, s0, &l, &k);
  const long long gid = level_base(l) + ((long long)rank << (2 * l - s0)) + k;
  double* o = out + 5 * u;
  o[0] = cx[gid]; o[1] = cy[gid]; o[2] = hw[gid]; o[3] = hh[gid]; o[4] = r[gid];
}

__global__ void k_geo_unpack(long long count, int G, int ltop, int s0, const double* in,
                             double* cx, double* cy, double* hw, double* hh, double* r) {
  pdl_enter();
  const long long v = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (v >= count * G) return;
  const int q = (int)(v / count);
  const long long u = v - q * count;
  int l;
  long long k;
  own_slot(u, ltop, s0, &l, &k);
  const long long gid = level_base(l) + ((long long)q << (2 * l - s0)) + k;
  const double* o = in + 5 * v;
  cx[gid] = o[0]; cy[gid] = o[1]; hw[gid] = o[2]; hh[gid] = o[3]; r[gid] = o[4];
}

// -------------------------------------------------------------------------
// import sets: boxes / leaves owned by other ranks that this rank's targets use
__device__ __forceinline__ int box_level(long long gid) {
  int l = 0;
  while (level_base(l + 1) <= gid) ++l;
  return l;
}

__device__ __forceinline__ int owner_of(long long gid, int s0) {   // -1: shared
  const int l = box_level(gid);
  const int t = 2 * l - s0;
  if (t < 0) return -1;
  return (int)((gid - level_base(l)) >> t);
}

__global__ void k_mark_weak(const int* __restrict__ total, const int* __restrict__ w_src,
                            int s0, int rank, unsigned char* flags) {
  pdl_enter();
  const long long n = *total;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n;
       i += (long long)gridDim.x * blockDim.x) {
    const int s = w_src[i];
    const int o = owner_of(s, s0);
    if (o >= 0 && o != rank) flags[s] = 1;
  }
}

// leaf lists (level-local ids) of the owned leaves [b0, b1)
__global__ void k_mark_leaf_lists(long long b0, long long b1, const int* __restrict__ off,
                                  const int* __restrict__ idx, int tshift, int rank,
                                  long long base, unsigned char* flags) {
  pdl_enter();
  const long long b = b0 + ((blockIdx.x * (long long)blockDim.x + threadIdx.x) >> 5);
  const int lane = threadIdx.x & 31;
  if (b >= b1) return;
  for (int q = off[b] + lane; q < off[b + 1]; q += 32) {
    const int a = idx[q];
    if ((a >> tshift) != rank) flags[base + a] = 1;
  }
}

__global__ void k_owner_keys(const int* __restrict__ nsel, const int* __restrict__ ids, int s0,
                             int leaf_level, unsigned* keys) {
  pdl_enter();
  const long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (i >= *nsel) return;
  const int id = ids[i];
  keys[i] = leaf_level >= 0 ? (unsigned)(id >> (2 * leaf_level - s0)) : (unsigned)owner_of(id, s0);
}

// requests per owner q < G from the owner-sorted keys (binary search)
__global__ void k_owner_counts(const int* __restrict__ nsel, const unsigned* __restrict__ keys,
                               int G, int* counts) {
  pdl_enter();
  const int q = threadIdx.x;
  if (q >= G) return;
  const int n = *nsel;
  auto lower = [&](unsigned v) {
    int lo = 0, hi = n;
    while (lo < hi) {
      const int mid = (lo + hi) >> 1;
      if (keys[mid] < v) lo = mid + 1;
      else hi = mid;
    }
    return lo;
  };
  counts[q] = lower((unsigned)q + 1) - lower((unsigned)q);
}

// -------------------------------------------------------------------------
// halo payloads
// particles: every requested leaf travels as nmax records {x, y, g} (padded)
__global__ void k_leaf_pack(long long nids, const int* __restrict__ ids,
                            const int* __restrict__ leaf_off, int nmax,
                            const double2* __restrict__ pos, const double* __restrict__ g,
                            double* out) {
  pdl_enter();
  const long long v = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (v >= nids * nmax) return;
  const long long q = v / nmax;
  const int k = (int)(v - q * nmax);
  const int a = ids[q];
  const int s0 = leaf_off[a], cnt = leaf_off[a + 1] - s0;
  double* o = out + 3 * v;
  if (k < cnt) {
    const double2 z = pos[s0 + k];
    o[0] = z.x; o[1] = z.y; o[2] = g[s0 + k];
  } else {
    o[0] = 0.0; o[1] = 0.0; o[2] = 0.0;
  }
}

__global__ void k_leaf_unpack(long long nids, const int* __restrict__ ids,
                              const int* __restrict__ leaf_off, int nmax,
                              const double* __restrict__ in, double2* pos, double* g) {
  pdl_enter();
  const long long v = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (v >= nids * nmax) return;
  const long long q = v / nmax;
  const int k = (int)(v - q * nmax);
  const int a = ids[q];
  const int s0 = leaf_off[a], cnt = leaf_off[a + 1] - s0;
  if (k >= cnt) return;
  const double* o = in + 3 * v;
  pos[s0 + k] = make_double2(o[0], o[1]);
  g[s0 + k] = o[2];
}

// multipole rows (p+1 complex)
__global__ void k_row_pack(long long nids, const int* __restrict__ ids, int p,
                           const double2* __restrict__ rows, double2* out) {
  pdl_enter();
  const long long v = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (v >= nids * (p + 1)) return;
  const long long q = v / (p + 1);
  const int j = (int)(v - q * (p + 1));
  out[v] = rows[(long long)ids[q] * (p + 1) + j];
}

__global__ void k_row_unpack(long long nids, const int* __restrict__ ids, int p,
                             const double2* __restrict__ in, double2* rows) {
  pdl_enter();
  const long long v = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (v >= nids * (p + 1)) return;
  const long long q = v / (p + 1);
  const int j = (int)(v - q * (p + 1));
  rows[(long long)ids[q] * (p + 1) + j] = in[v];
}

// level-ltop multipoles of every rank (allgather payload)
__global__ void k_level_rows(long long k0, long long cnt, long long lbase, int p,
                             const double2* __restrict__ rows, double2* out, bool pack) {
  pdl_enter();
  const long long v = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (v >= cnt * (p + 1)) return;
  double2* row = const_cast<double2*>(rows) + (lbase + k0) * (p + 1);
  if (pack) out[v] = row[v];
  else row[v] = out[v];
}

__global__ void k_scatter_values(long long n, const double2* __restrict__ vals,
                                 const long long* __restrict__ idx, double2* out) {
  pdl_enter();
  const long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (i < n) out[idx[i]] = vals[i];
}

__global__ void k_fill_owned_idx(long long n, const int* __restrict__ perm, long long* out) {
  pdl_enter();
  const long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (i < n) out[i] = perm[i];
}

// separate evaluation points: destination rank = top-split segment reached by
// coord <= cut (tree.py:210) through the s0 collectively chosen cuts
// (step s, segment j at table entry 2^s - 1 + j)
__global__ void k_eval_dest(long long m, const Rec* __restrict__ rec, int s0,
                            const double* __restrict__ cuts, const unsigned char* __restrict__ axes,
                            unsigned* key, int* val, int* count) {
  pdl_enter();
  const long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (i >= m) return;
  const Rec r = rec[i];
  int seg = 0;
  for (int s = 0; s < s0; ++s) {
    const int t = (1 << s) - 1 + seg;
    seg = 2 * seg + ((axes[t] ? r.y : r.x) <= cuts[t] ? 0 : 1);
  }
  key[i] = (unsigned)seg;
  val[i] = (int)i;
  atomicAdd(count + seg, 1);
}

__global__ void k_erec_unpack(long long m, const Rec* __restrict__ rec, double2* pos, int* idx) {
  pdl_enter();
  const long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (i >= m) return;
  const Rec r = rec[i];
  pos[i] = make_double2(r.x, r.y);
  idx[i] = (int)r.idx;
}

// global-size evaluation leaf offsets: the owned leaves [b0, b0 + nl) carry
// the subtree's local offsets, the others are empty (monotone)
__global__ void k_eoff_global(long long nleaf, long long b0, long long nl,
                              const int* __restrict__ loc, int m, int* out) {
  pdl_enter();
  const long long b = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (b > nleaf) return;
  out[b] = b < b0 ? 0 : (b > b0 + nl ? m : loc[b - b0]);
}

__global__ void k_pick5(const int* a, const int* b, const int* c, const int* d, const int* e,
                        int* out) {
  pdl_enter();
  if (threadIdx.x == 0) {
    out[0] = *a;
    out[1] = *b;
    out[2] = *c;
    out[3] = *d;
    out[4] = *e;
  }
}

__global__ void k_add_base(long long m, const unsigned* __restrict__ in, unsigned base,
                           unsigned* out) {
  pdl_enter();
  const long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (i < m) out[i] = in[i] + base;
}

template <class K, class V>
void sort_pairs(DBuf& tmp, const K* kin, K* kout, const V* vin, V* vout, long long n, int bits,
                cudaStream_t st) {
  size_t bytes = 0;
  FMM_CUDA(cub::DeviceRadixSort::SortPairs(nullptr, bytes, kin, kout, vin, vout, (int)n, 0, bits,
                                           st));
  tmp.reserve(bytes);
  FMM_CUDA(cub::DeviceRadixSort::SortPairs(tmp.p, bytes, kin, kout, vin, vout, (int)n, 0, bits,
                                           st));
}

}  // namespace

}  // namespace fmm

using namespace fmm;

namespace {

DistState& dist(fmm2d_ctx* c) {
  if (!c->D.active) throw ApiError{FMM2D_EBADARG, "no distributed evaluation set up"};
  return c->D;
}

void sync(fmm2d_ctx* c) {
  FMM_CUDA(cudaStreamSynchronize(c->st));
  FMM_CUDA(cudaGetLastError());
}

int top_segments(const DistState& D, int s) { return 1 << s; }

// host mirror of the split-axis rule, geometry.py:57-63
bool split_along_y(const double* r) { return (r[3] - r[2]) / 2 > (r[1] - r[0]) / 2; }

void check_top_degenerate(fmm2d_ctx* c, int s, const double* box4 /* per segment */) {
  DistState& D = c->D;
  if ((s & 1) || (s >> 1) >= D.L) return;
  const int l = s >> 1;
  for (int j = 0; j < top_segments(D, s); ++j) {
    const double* b = box4 + 4 * j;
    if (b[0] == -b[1] && b[2] == -b[3]) {
      const long long cnt = D.off[s][j + 1] - D.off[s][j];
      char buf[512];
      snprintf(buf, sizeof buf,
               "all %lld source points in box %d at level %d coincide at (%.17g, %.17g) but %d "
               "more level(s) are required; reduce the level count or perturb the input",
               cnt, j, l, b[0], b[2], D.L - l);
      c->deg_info[0] = cnt;
      c->deg_info[1] = j;
      c->deg_info[2] = l;
      c->deg_info[3] = D.L - l;
      c->deg_xy[0] = b[0];
      c->deg_xy[1] = b[2];
      throw ApiError{FMM2D_EDEGENERATE, buf};
    }
  }
}

long long own_count(const DistState& D) {
  long long c = 0;
  for (int l = D.part.ltop(); l <= D.L; ++l) c += 1ll << (2 * l - D.part.s0);
  return c;
}

void record(fmm2d_ctx* c, int q) { FMM_CUDA(cudaEventRecord(c->D.ev[q], c->st)); }

}  // namespace

extern "C" {

int fmm2d_dist_setup(fmm2d_ctx* c, int G, int rank, int64_t n_total, int p, double theta, int nd,
                     void* stream, int32_t* n_levels) {
  if (!c) return FMM2D_EBADARG;
  return guarded(c, [&] {
    validate(n_total, n_total, nd, theta, p, true);
    if (G < 1 || (G & (G - 1)) || G > 64) throw ApiError{FMM2D_EBADARG, "world size must be a power of two <= 64"};
    if (rank < 0 || rank >= G) throw ApiError{FMM2D_EBADARG, "bad rank"};
    FMM_CUDA(cudaSetDevice(c->device));
    c->st = stream ? static_cast<cudaStream_t>(stream) : c->own_st;
    DistState& D = c->D;
    D.part = Part{G, rank, 0};
    while ((1 << D.part.s0) < G) ++D.part.s0;
    D.n_total = n_total;
    D.L = plan_levels(n_total, nd);
    D.p = p;
    D.theta = theta;
    D.nd = nd;
    if (2 * D.L < D.part.s0)
      throw ApiError{FMM2D_EBADARG, "too few points for this many ranks (need 4^levels >= ranks)"};
    // data-independent offsets of every global step (tree.py:308-310): kept
    // (host tables and the device leaf offsets) while (n_total, L) repeat
    const int S = 2 * D.L;
    const long long nleaf = 1ll << S;
    if (D.off_key_n != n_total || D.off_key_L != D.L || D.leaf_off.p == nullptr) {
      D.off.assign(S + 1, {});
      D.off[0] = {0, n_total};
      for (int s = 0; s < S; ++s) {
        const auto& o = D.off[s];
        std::vector<long long> nx(2 * (o.size() - 1) + 1);
        nx[0] = 0;
        for (size_t j = 0; j + 1 < o.size(); ++j) {
          const long long cnt = o[j + 1] - o[j];
          nx[2 * j + 1] = o[j] + (cnt + 1) / 2;
          nx[2 * j + 2] = o[j + 1];
        }
        D.off[s + 1] = std::move(nx);
      }
      std::vector<int> lo(nleaf + 1);
      long long mx = 0;
      for (long long k = 0; k <= nleaf; ++k) lo[k] = (int)D.off[S][k];
      for (long long k = 0; k < nleaf; ++k) mx = std::max(mx, D.off[S][k + 1] - D.off[S][k]);
      D.nmax_leaf = std::max(1ll, mx);
      D.leaf_off.reserve(sizeof(int) * (nleaf + 1));
      // on the engine stream (ordered with its kernels); lo lives until the sync
      FMM_CUDA(cudaMemcpyAsync(D.leaf_off.p, lo.data(), sizeof(int) * (nleaf + 1),
                               cudaMemcpyHostToDevice, c->st));
      sync(c);
      D.off_key_n = n_total;
      D.off_key_L = D.L;
    }
    D.g0 = D.off[D.part.s0][rank];
    D.n_r = D.off[D.part.s0][rank + 1] - D.g0;
    // global-size tree-order arrays (halo particles land at their global offsets)
    TreeState& T = c->T;
    T.src_pos.reserve(sizeof(double2) * n_total);
    T.src_g.reserve(sizeof(double) * n_total);
    T.src_perm.reserve(sizeof(int) * n_total);
    const long long nbox = level_base(D.L + 1);
    for (DBuf* b : {&T.box_cx, &T.box_cy, &T.box_hw, &T.box_hh, &T.box_r})
      b->reserve(sizeof(double) * nbox);
    c->E.p = p;
    c->E.mult.reserve(sizeof(double2) * nbox * (p + 1));
    c->E.local.reserve(sizeof(double2) * nbox * (p + 1));
    c->E.phi.reserve(sizeof(double2) * n_total);
    for (auto& e : D.ev)
      if (!e) FMM_CUDA(cudaEventCreate(&e));
    D.active = true;
    D.separate = false;
    D.m_total = D.m_local = D.m_r = 0;
    D.cuts.assign(D.part.s0, {});
    D.axes.assign(D.part.s0, {});
    c->have_tree = c->have_lists = c->have_eval = false;
    if (n_levels) *n_levels = D.L;
    return FMM2D_OK;
  });
}

// shard [idx_base, idx_base + n_local) of the input (device pointers) ->
// records; writes the local box (min x, -max x, min y, -max y) to d_bbox4 for
// an allreduce(MIN)
int fmm2d_dist_load(fmm2d_ctx* c, int64_t n_local, const double* d_pos, const double* d_g,
                    int64_t idx_base, double* d_bbox4) {
  if (!c) return FMM2D_EBADARG;
  return guarded(c, [&] {
    DistState& D = dist(c);
    FMM_CUDA(cudaSetDevice(c->device));
    g_launches = 0;
    reset_status(c);
    record(c, 0);
    D.n_local = n_local;
    D.rec_a.reserve(sizeof(Rec) * std::max<long long>(1, n_local));
    D.bbox.reserve(sizeof(unsigned long long) * 4 * 16);
    FMM_CUDA(cudaMemsetAsync(D.bbox.p, 0xff, sizeof(unsigned long long) * 4, c->st));
    note_launch();
    launch(k_rec_load, std::max(1u, std::min(nblk(n_local, 256), 1184u)), 256, 0, c->st, 
        n_local, reinterpret_cast<const double2*>(d_pos), d_g, idx_base, D.rec_a.as<Rec>(),
        D.bbox.as<unsigned long long>());
    note_launch();
    launch(k_bbox_out, 1, 32, 0, c->st, D.bbox.as<unsigned long long>(), d_bbox4);
    D.seg_off = {0, n_local};
    D.d_seg_off.reserve(sizeof(long long) * 80);
    FMM_CUDA(cudaMemcpyAsync(D.d_seg_off.p, D.seg_off.data(), sizeof(long long) * 2,
                             cudaMemcpyHostToDevice, c->st));
    sync(c);
    return FMM2D_OK;
  });
}

// separate evaluation points (call after fmm2d_dist_load, before the bbox
// allreduce): shard [idx_base, idx_base + m_local) of the M = m_total points
// -> records; the local box written to d_bbox4 now covers sources and
// evaluation points (tree.py:256-259)
int fmm2d_dist_load_evals(fmm2d_ctx* c, int64_t m_total, int64_t m_local, const double* d_epos,
                          int64_t idx_base, double* d_bbox4) {
  if (!c) return FMM2D_EBADARG;
  return guarded(c, [&] {
    DistState& D = dist(c);
    if (m_total < 1 || m_local < 0 || m_total > INT32_MAX)
      throw ApiError{FMM2D_EBADARG, "bad evaluation point count"};
    D.separate = true;
    D.m_total = m_total;
    D.m_local = m_local;
    D.erec_a.reserve(sizeof(Rec) * std::max<long long>(1, m_local));
    if (m_local > 0) {
      note_launch();
      launch(k_rec_load, std::max(1u, std::min(nblk(m_local, 256), 1184u)), 256, 0, c->st,
             (long long)m_local, reinterpret_cast<const double2*>(d_epos), (const double*)nullptr,
             (long long)idx_base, D.erec_a.as<Rec>(), D.bbox.as<unsigned long long>());
    }
    note_launch();
    launch(k_bbox_out, 1, 32, 0, c->st, D.bbox.as<unsigned long long>(), d_bbox4);
    return FMM2D_OK;
  });
}

// after the top split: every local evaluation point's destination rank
// (coord <= cut through the s0 top cuts), records grouped by destination in
// original order; counts (host int64[G]) and the grouped records
int fmm2d_dist_eval_route(fmm2d_ctx* c, int64_t* counts, void** d_records) {
  if (!c) return FMM2D_EBADARG;
  return guarded(c, [&] {
    DistState& D = dist(c);
    const int G = D.part.G, s0 = D.part.s0;
    if (!D.separate) throw ApiError{FMM2D_EBADARG, "no separate evaluation points loaded"};
    const long long m = D.m_local;
    std::vector<double> cut(std::max(1, G - 1));
    std::vector<unsigned char> ax(std::max(1, G - 1));
    for (int s = 0; s < s0; ++s) {
      if ((int)D.cuts[s].size() != (1 << s)) throw ApiError{FMM2D_EBADARG, "top split incomplete"};
      for (int j = 0; j < (1 << s); ++j) {
        cut[(1 << s) - 1 + j] = D.cuts[s][j];
        ax[(1 << s) - 1 + j] = D.axes[s][j];
      }
    }
    D.ecount.reserve(sizeof(int) * G + sizeof(double) * 64 + 64);
    int* dcount = D.ecount.as<int>();
    double* dcut = reinterpret_cast<double*>(D.ecount.as<char>() + ((sizeof(int) * G + 15) & ~15ull));
    unsigned char* dax = reinterpret_cast<unsigned char*>(dcut + 32);
    FMM_CUDA(cudaMemsetAsync(dcount, 0, sizeof(int) * G, c->st));
    FMM_CUDA(cudaMemcpyAsync(dcut, cut.data(), sizeof(double) * cut.size(), cudaMemcpyHostToDevice,
                             c->st));
    FMM_CUDA(cudaMemcpyAsync(dax, ax.data(), ax.size(), cudaMemcpyHostToDevice, c->st));
    std::vector<int> hc(G, 0);
    if (m > 0) {
      for (DBuf* b : {&D.skey, &D.skey2}) b->reserve(sizeof(unsigned) * m);
      for (DBuf* b : {&D.sval, &D.sval2}) b->reserve(sizeof(int) * m);
      note_launch();
      launch(k_eval_dest, nblk(m, 256), 256, 0, c->st, m, D.erec_a.as<Rec>(), s0, dcut, dax,
             D.skey.as<unsigned>(), D.sval.as<int>(), dcount);
      sort_pairs(D.cub_tmp, D.skey.as<unsigned>(), D.skey2.as<unsigned>(), D.sval.as<int>(),
                 D.sval2.as<int>(), m, std::max(1, s0), c->st);
      D.erec_b.reserve(sizeof(Rec) * m);
      note_launch();
      launch(k_rec_gather, nblk(m, 256), 256, 0, c->st, m, D.sval2.as<int>(), D.erec_a.as<Rec>(),
             D.erec_b.as<Rec>());
      D.erec_a.swap(D.erec_b);
      FMM_CUDA(cudaMemcpyAsync(hc.data(), dcount, sizeof(int) * G, cudaMemcpyDeviceToHost, c->st));
    }
    sync(c);   // (cut / ax are host temporaries of the uploads as well)
    for (int q = 0; q < G; ++q) counts[q] = hc[q];
    *d_records = D.erec_a.p;
    return FMM2D_OK;
  });
}

// root rectangle from the allreduced box (tree.py:256-259); level-0 degenerate check
int fmm2d_dist_root(fmm2d_ctx* c, const double* d_bbox4) {
  if (!c) return FMM2D_EBADARG;
  return guarded(c, [&] {
    DistState& D = dist(c);
    double b[4];
    FMM_CUDA(cudaMemcpyAsync(b, d_bbox4, sizeof b, cudaMemcpyDeviceToHost, c->st));
    sync(c);
    D.rect.assign(D.part.s0 + 1, {});
    D.rect[0] = {b[0], -b[1], b[2], -b[3]};
    if (D.L > 0) check_top_degenerate(c, 0, b);
    return FMM2D_OK;
  });
}

// per-segment local boxes for the degenerate check of the level-(s/2) boxes
// (even steps s >= 2 only; allreduce(MIN) over 4 * 2^s doubles)
int fmm2d_dist_segbox(fmm2d_ctx* c, int s, double* d_box) {
  if (!c) return FMM2D_EBADARG;
  return guarded(c, [&] {
    DistState& D = dist(c);
    const int nseg = top_segments(D, s);
    D.bbox.reserve(sizeof(unsigned long long) * 4 * std::max(16, nseg));
    FMM_CUDA(cudaMemsetAsync(D.bbox.p, 0xff, sizeof(unsigned long long) * 4 * nseg, c->st));
    note_launch();
    launch(k_seg_box, std::max(1u, std::min(nblk(D.n_local, 256), 1184u)), 256, 0, c->st, 
        nseg, D.rec_a.as<Rec>(), D.d_seg_off.as<long long>(), D.bbox.as<unsigned long long>());
    note_launch();
    launch(k_keys_out, 1, 128, 0, c->st, D.bbox.as<unsigned long long>(), d_box, 4 * nseg);
    return FMM2D_OK;
  });
}

int fmm2d_dist_check_segbox(fmm2d_ctx* c, int s, const double* d_box) {
  if (!c) return FMM2D_EBADARG;
  return guarded(c, [&] {
    DistState& D = dist(c);
    std::vector<double> b(4 * top_segments(D, s));
    FMM_CUDA(cudaMemcpyAsync(b.data(), d_box, sizeof(double) * b.size(), cudaMemcpyDeviceToHost,
                             c->st));
    sync(c);
    check_top_degenerate(c, s, b.data());
    return FMM2D_OK;
  });
}

// one radix-select round of split step s: d_hist [2^s][256] int32 (zeroed here,
// to be allreduced(SUM) by the caller); rho = 0 also initialises the selection
int fmm2d_dist_hist(fmm2d_ctx* c, int s, int rho, int32_t* d_hist) {
  if (!c) return FMM2D_EBADARG;
  return guarded(c, [&] {
    DistState& D = dist(c);
    const int nseg = top_segments(D, s);
    if (nseg > 4) throw ApiError{FMM2D_EBADARG, "top split supports at most 8 ranks per step"};
    if (rho == 0) {
      std::vector<unsigned char> ax(nseg);
      std::vector<long long> kth(nseg);
      for (int j = 0; j < nseg; ++j) {
        ax[j] = split_along_y(&D.rect[s][4 * j]);
        const long long n = D.off[s][j + 1] - D.off[s][j];
        kth[j] = (n + 1) / 2;                                    // tree.py:108
      }
      D.d_axis.reserve(16);
      D.sel.reserve(sizeof(SelState) * 8 + sizeof(long long) * 8);
      FMM_CUDA(cudaMemcpyAsync(D.d_axis.p, ax.data(), nseg, cudaMemcpyHostToDevice, c->st));
      long long* dk = reinterpret_cast<long long*>(D.sel.as<SelState>() + 8);
      FMM_CUDA(cudaMemcpyAsync(dk, kth.data(), sizeof(long long) * nseg, cudaMemcpyHostToDevice,
                               c->st));
      note_launch();
      launch(k_sel_init, 1, 32, 0, c->st, D.sel.as<SelState>(), dk, nseg);
      sync(c);   // ax / kth are host temporaries
    }
    FMM_CUDA(cudaMemsetAsync(d_hist, 0, sizeof(int) * 256 * nseg, c->st));
    note_launch();
    launch(k_sel_hist, std::max(1u, std::min(nblk(D.n_local, 256), 592u)), 256, 0, c->st, 
        rho, nseg, D.rec_a.as<Rec>(), D.d_seg_off.as<long long>(),
        D.d_axis.as<unsigned char>(), D.sel.as<SelState>(), d_hist);
    return FMM2D_OK;
  });
}

int fmm2d_dist_pick(fmm2d_ctx* c, int s, int rho, const int32_t* d_hist) {
  if (!c) return FMM2D_EBADARG;
  return guarded(c, [&] {
    DistState& D = dist(c);
    note_launch();
    launch(k_sel_pick, 1, 32, 0, c->st, rho, top_segments(D, s), d_hist, D.sel.as<SelState>());
    return FMM2D_OK;
  });
}

// local count of cut-equal keys per segment -> d_eq [2^s] int32 (allgather)
int fmm2d_dist_eqcount(fmm2d_ctx* c, int s, int32_t* d_eq) {
  if (!c) return FMM2D_EBADARG;
  return guarded(c, [&] {
    DistState& D = dist(c);
    const int nseg = top_segments(D, s);
    const long long n = std::max<long long>(1, D.n_local);
    D.eqf.reserve(sizeof(int) * n);
    D.eqpre.reserve(sizeof(int) * (n + 1));
    FMM_CUDA(cudaMemsetAsync(d_eq, 0, sizeof(int) * nseg, c->st));
    note_launch();
    launch(k_eq_count, std::max(1u, std::min(nblk(D.n_local, 256), 1184u)), 256, 0, c->st, 
        nseg, D.rec_a.as<Rec>(), D.d_seg_off.as<long long>(), D.d_axis.as<unsigned char>(),
        D.sel.as<SelState>(), d_eq, D.eqf.as<int>());
    return FMM2D_OK;
  });
}

// stable local partition of step s with the allgathered equal counts
// d_eq_all [G][2^s]; updates the host rectangles of step s+1
int fmm2d_dist_partition(fmm2d_ctx* c, int s, const int32_t* d_eq_all) {
  if (!c) return FMM2D_EBADARG;
  return guarded(c, [&] {
    DistState& D = dist(c);
    const int nseg = top_segments(D, s);
    const long long n = D.n_local;
    if (n > 0) {
      size_t bytes = 0;
      FMM_CUDA(cub::DeviceScan::ExclusiveSum(nullptr, bytes, D.eqf.as<int>(), D.eqpre.as<int>(),
                                             (int)n + 1, c->st));
      D.cub_tmp.reserve(bytes);
      // eqf[n] must be readable: scan n items, eqpre[n] unused
      FMM_CUDA(cub::DeviceScan::ExclusiveSum(D.cub_tmp.p, bytes, D.eqf.as<int>(),
                                             D.eqpre.as<int>(), (int)n, c->st));
      for (DBuf* b : {&D.skey, &D.skey2}) b->reserve(sizeof(unsigned) * n);
      for (DBuf* b : {&D.sval, &D.sval2}) b->reserve(sizeof(int) * n);
      note_launch();
      launch(k_side_keys, std::min(nblk(n, 256), 1184u), 256, 0, c->st, 
          nseg, D.part.G, D.part.rank, D.rec_a.as<Rec>(), D.d_seg_off.as<long long>(),
          D.d_axis.as<unsigned char>(), D.sel.as<SelState>(), d_eq_all, D.eqpre.as<int>(),
          D.skey.as<unsigned>(), D.sval.as<int>());
      sort_pairs(D.cub_tmp, D.skey.as<unsigned>(), D.skey2.as<unsigned>(), D.sval.as<int>(),
                 D.sval2.as<int>(), n, s + 1, c->st);
      D.rec_b.reserve(sizeof(Rec) * n);
      note_launch();
      launch(k_rec_gather, nblk(n, 256), 256, 0, c->st, n, D.sval2.as<int>(), D.rec_a.as<Rec>(),
                                                    D.rec_b.as<Rec>());
      D.rec_a.swap(D.rec_b);
    }
    note_launch();
    launch(k_seg_bounds, nblk(n + 1, 256), 256, 0, c->st, n, 2 * nseg, D.skey2.as<unsigned>(),
                                                      D.d_seg_off.as<long long>());
    // cut values and child rectangles (tree.py:218-222)
    std::vector<SelState> sel(nseg);
    std::vector<int> eq_all((size_t)D.part.G * nseg);
    FMM_CUDA(cudaMemcpyAsync(sel.data(), D.sel.p, sizeof(SelState) * nseg, cudaMemcpyDeviceToHost,
                             c->st));
    FMM_CUDA(cudaMemcpyAsync(eq_all.data(), d_eq_all, sizeof(int) * eq_all.size(),
                             cudaMemcpyDeviceToHost, c->st));
    D.seg_off.assign(2 * nseg + 1, 0);
    FMM_CUDA(cudaMemcpyAsync(D.seg_off.data(), D.d_seg_off.p, sizeof(long long) * (2 * nseg + 1),
                             cudaMemcpyDeviceToHost, c->st));
    sync(c);
    if (n == 0) std::fill(D.seg_off.begin(), D.seg_off.end(), 0);
    // the evaluation points (aliasing the sources) follow coord <= cut
    // (tree.py:210): when more sources equal the cut than the k-th-smallest
    // quota sends left, the reference's evaluation split differs from the
    // source split.  sel and eq_all are identical on every rank, so every
    // rank raises here together (no rank is left waiting in a collective).
    for (int j = 0; j < nseg && !D.separate; ++j) {
      long long eq = 0;
      for (int q = 0; q < D.part.G; ++q) eq += eq_all[(size_t)q * nseg + j];
      if (eq > (long long)sel[j].k_rem)
        throw ApiError{FMM2D_EBADARG,
                       "coordinate ties at a median cut are not supported by the distributed "
                       "engine (evaluate on one GPU)"};
    }
    D.rect[s + 1].assign(8 * nseg, 0.0);
    for (int j = 0; j < nseg; ++j) {
      const double* r = &D.rect[s][4 * j];
      const bool ay = split_along_y(r);
      const unsigned long long k = sel[j].prefix;
      const unsigned long long bits = (k & 0x8000000000000000ull) ? (k & 0x7fffffffffffffffull) : ~k;
      double cut;
      std::memcpy(&cut, &bits, sizeof cut);
      D.cuts[s].resize(nseg);
      D.axes[s].resize(nseg);
      D.cuts[s][j] = cut;
      D.axes[s][j] = ay;
      double* lo = &D.rect[s + 1][8 * j];
      double* hi = lo + 4;
      for (int q = 0; q < 4; ++q) lo[q] = hi[q] = r[q];
      if (ay) { lo[3] = cut; hi[2] = cut; } else { lo[1] = cut; hi[0] = cut; }
    }
    return FMM2D_OK;
  });
}

// records per destination rank after the top split (host int64[G])
int fmm2d_dist_send_counts(fmm2d_ctx* c, int64_t* counts, void** d_records) {
  if (!c) return FMM2D_EBADARG;
  return guarded(c, [&] {
    DistState& D = dist(c);
    const int G = D.part.G;
    if ((int)D.seg_off.size() != G + 1) throw ApiError{FMM2D_EBADARG, "top split incomplete"};
    for (int q = 0; q < G; ++q) counts[q] = D.seg_off[q + 1] - D.seg_off[q];
    *d_records = D.rec_a.p;
    return FMM2D_OK;
  });
}

// build the owned subtree from the received records (n_r of them, canonical
// order) and the owned geometry; returns the owned-box count per rank (the
// geometry allgather is 5 doubles per owned box)
int fmm2d_dist_build(fmm2d_ctx* c, const double* d_recv, int64_t n_recv, const double* d_erecv,
                     int64_t m_recv, int64_t* own_boxes) {
  if (!c) return FMM2D_EBADARG;
  return guarded(c, [&] {
    DistState& D = dist(c);
    if (n_recv != D.n_r) throw ApiError{FMM2D_ECUDA, "exchange delivered a wrong record count"};
    const int s0 = D.part.s0, rank = D.part.rank, L = D.L;
    record(c, 1);
    const long long n = D.n_r;
    D.loc_pos.reserve(sizeof(double2) * n);
    D.loc_g.reserve(sizeof(double) * n);
    D.loc_idx.reserve(sizeof(int) * n);
    note_launch();
    launch(k_rec_unpack, nblk(n, 256), 256, 0, c->st, n, reinterpret_cast<const Rec*>(d_recv),
                                                  D.loc_pos.as<double2>(), D.loc_g.as<double>(),
                                                  D.loc_idx.as<int>());
    TreeState& T = c->T;
    T.n = T.m = n;
    T.L = L;
    T.aliased = true;
    T.pos_p = D.loc_pos.as<double2>();
    T.g_p = D.loc_g.as<double>();
    T.epos_p = nullptr;
    if (D.separate) {
      // the evaluation points this rank owns (original order): its subtree's
      // evaluation split descends the same cut tables (k_descend)
      D.m_r = m_recv;
      D.loc_epos.reserve(sizeof(double2) * std::max<long long>(1, m_recv));
      D.loc_eidx.reserve(sizeof(int) * std::max<long long>(1, m_recv));
      if (m_recv > 0) {
        note_launch();
        launch(k_erec_unpack, nblk(m_recv, 256), 256, 0, c->st, (long long)m_recv,
               reinterpret_cast<const Rec*>(d_erecv), D.loc_epos.as<double2>(),
               D.loc_eidx.as<int>());
      }
      T.m = m_recv;
      T.aliased = false;
      T.epos_p = D.loc_epos.as<double2>();
    }
    T.inputs_ready = nullptr;
    T.spec = TreeSpec{};
    T.spec.s0 = s0;
    T.spec.seg = rank;
    T.spec.out0 = D.g0;
    T.spec.orig = D.loc_idx.as<int>();
    T.spec.eorig = D.separate ? D.loc_eidx.as<int>() : nullptr;
    T.spec.root_given = true;
    for (int q = 0; q < 4; ++q) T.spec.root[q] = D.rect[s0][4 * rank + q];
    for (int attempt = 0;; ++attempt) {
      reset_status(c);
      plan_tree(c->plan, n, n, L, s0);
      run_tree(T, c->plan, c->d_status.as<DevStatus>(), c->st);
      fetch_status(c);
      sync(c);
      const int fl = c->h_status->flags;
      if ((fl & ST_RANK_RETRY) && !T.exact_keys && attempt == 0) {
        T.exact_keys = true;
        continue;
      }
      if (fl & ST_DEGENERATE) {
        const unsigned long long key = c->h_status->degenerate_key;
        char buf[256];
        snprintf(buf, sizeof buf,
                 "all source points in box %lld at level %d coincide but %d more level(s) are "
                 "required; reduce the level count or perturb the input",
                 (long long)(key & ((1ull << 40) - 1)), (int)(key >> 40), L - (int)(key >> 40));
        throw ApiError{FMM2D_EDEGENERATE, buf};
      }
      if ((fl & ST_EVAL_TIES) && !D.separate)
        throw ApiError{FMM2D_EBADARG,
                       "coordinate ties at a median cut are not supported by the distributed "
                       "engine (evaluate on one GPU)"};
      break;
    }
    T.spec = TreeSpec{};
    // every rank sees the whole pyramid through global-size arrays
    T.n = T.m = D.n_total;
    if (D.separate) {
      // evaluation arrays stay local (only the owner evaluates them): local tree
      // order, original indices in eval_perm, global-size leaf offsets and
      // global leaf ids for the downward kernels
      const int S = 2 * L - s0;
      const long long nleaf = 1ll << (2 * L), b0 = (long long)rank << S;
      T.m = D.m_r;
      D.eoff_g.reserve(sizeof(int) * (nleaf + 1));
      note_launch();
      launch(k_eoff_global, nblk(nleaf + 1, 256), 256, 0, c->st, nleaf, b0, 1ll << S,
             T.eval_leaf_off.as<int>(), (int)D.m_r, D.eoff_g.as<int>());
      D.eleaf_g.reserve(sizeof(unsigned) * std::max<long long>(1, D.m_r));
      if (D.m_r > 0 && T.eleaf_t) {
        note_launch();
        launch(k_add_base, nblk(D.m_r, 256), 256, 0, c->st, (long long)D.m_r, T.eleaf_t,
               (unsigned)b0, D.eleaf_g.as<unsigned>());
      }
      T.epos_t = T.eval_pos.as<double2>();
      T.eperm_t = T.eval_perm.as<int>();
      T.eoff_t = D.eoff_g.as<int>();
      T.eleaf_t = D.eleaf_g.as<unsigned>();
      c->E.phi.reserve(sizeof(double2) * std::max<long long>(D.n_total, D.m_r));
    } else {
      T.epos_t = T.src_pos.as<double2>();
      T.eperm_t = T.src_perm.as<int>();
      T.eoff_t = D.leaf_off.as<int>();
      T.eleaf_t = nullptr;
    }
    // shared (top) levels: geometry from the collectively computed rectangles
    // (uploaded on the engine stream, ordered before the connectivity kernels;
    // the staging vectors stay alive until the sync below)
    std::vector<std::vector<double>> stage;
    for (int l = 0; 2 * l < s0 && l <= L; ++l) {
      const int nb = 1 << (2 * l);
      stage.emplace_back(5 * nb);
      std::vector<double>& v = stage.back();
      for (int k = 0; k < nb; ++k) {
        const double* r = &D.rect[2 * l][4 * k];
        v[k] = (r[0] + r[1]) / 2;                     // tree.py:312-314
        v[nb + k] = (r[2] + r[3]) / 2;
        v[2 * nb + k] = (r[1] - r[0]) / 2;
        v[3 * nb + k] = (r[3] - r[2]) / 2;
        v[4 * nb + k] = std::hypot(v[2 * nb + k], v[3 * nb + k]);   // glibc, geometry.py:29
      }
      const long long gb = level_base(l);
      DBuf* arr[5] = {&T.box_cx, &T.box_cy, &T.box_hw, &T.box_hh, &T.box_r};
      for (int f = 0; f < 5; ++f)
        FMM_CUDA(cudaMemcpyAsync(arr[f]->as<double>() + gb, v.data() + f * nb,
                                 sizeof(double) * nb, cudaMemcpyHostToDevice, c->st));
    }
    if (!stage.empty()) sync(c);
    *own_boxes = own_count(D);
    c->have_tree = true;
    return FMM2D_OK;
  });
}

int fmm2d_dist_geom_pack(fmm2d_ctx* c, double* d_send) {
  if (!c) return FMM2D_EBADARG;
  return guarded(c, [&] {
    DistState& D = dist(c);
    const TreeState& T = c->T;
    const long long cnt = own_count(D);
    note_launch();
    launch(k_geo_pack, nblk(cnt, 256), 256, 0, c->st, cnt, D.part.ltop(), D.part.s0, D.part.rank,
                                                  T.box_cx.as<double>(), T.box_cy.as<double>(),
                                                  T.box_hw.as<double>(), T.box_hh.as<double>(),
                                                  T.box_r.as<double>(), d_send);
    return FMM2D_OK;
  });
}

// unpack the geometry allgather, build the owned interaction lists and the
// import sets; req_counts (host int64[2][G]) = boxes / leaves to request from
// every rank, grouped by owner in the request buffers (fmm2d_dist_requests)
int fmm2d_dist_connect(fmm2d_ctx* c, const double* d_geo_all, int64_t* req_counts) {
  if (!c) return FMM2D_EBADARG;
  return guarded(c, [&] {
    DistState& D = dist(c);
    TreeState& T = c->T;
    ListState& Ls = c->Ls;
    const int G = D.part.G, s0 = D.part.s0, rank = D.part.rank, L = D.L;
    const long long cnt = own_count(D);
    note_launch();
    launch(k_geo_unpack, nblk(cnt * G, 256), 256, 0, c->st, 
        cnt, G, D.part.ltop(), s0, d_geo_all, T.box_cx.as<double>(), T.box_cy.as<double>(),
        T.box_hw.as<double>(), T.box_hh.as<double>(), T.box_r.as<double>());
    record(c, 2);
    const long long nbox = level_base(L + 1), nleaf = 1ll << (2 * L);
    for (int attempt = 0;; ++attempt) {
      reset_status(c);
      run_connectivity(T, Ls, D.theta, c->d_status.as<DevStatus>(), c->st, D.part);
      fetch_status(c);
      sync(c);
      if (!(c->h_status->flags & ST_OVERFLOW)) break;
      if (attempt >= 8) throw ApiError{FMM2D_ECUDA, "interaction-list capacity did not converge"};
      Ls.cap_weak *= 2; Ls.cap_strong *= 4; Ls.cap_p2p *= 2; Ls.cap_p2l *= 2; Ls.cap_m2p *= 2;
    }
    record(c, 3);
    // import sets
    D.flags.reserve(nbox + nleaf + 16);
    unsigned char* fb = D.flags.as<unsigned char>();
    unsigned char* fl = fb + nbox;
    FMM_CUDA(cudaMemsetAsync(fb, 0, nbox + nleaf, c->st));
    const long long b0 = D.part.lo(L), b1 = D.part.hi(L);
    const int tshift = 2 * L - s0;
    note_launch();
    launch(k_mark_weak, 1184, 256, 0, c->st, Ls.weak_off.as<int>() + nbox, Ls.weak_idx.as<int>(), s0,
                                         rank, fb);
    note_launch();
    launch(k_mark_leaf_lists, nblk((b1 - b0) * 32, 256), 256, 0, c->st, 
        b0, b1, Ls.m2p_off.as<int>(), Ls.m2p_idx.as<int>(), tshift, rank, level_base(L), fb);
    note_launch();
    launch(k_mark_leaf_lists, nblk((b1 - b0) * 32, 256), 256, 0, c->st, 
        b0, b1, Ls.p2p_off.as<int>(), Ls.p2p_idx.as<int>(), tshift, rank, 0, fl);
    note_launch();
    launch(k_mark_leaf_lists, nblk((b1 - b0) * 32, 256), 256, 0, c->st, 
        b0, b1, Ls.p2l_off.as<int>(), Ls.p2l_idx.as<int>(), tshift, rank, 0, fl);
    // both kinds: flagged ids (boxes at offset 0, leaves at nbox), one count
    // read-back, owner-grouped ids (stable sort by owner key), per-owner
    // request counts on the device, one read-back
    const long long nn[2] = {nbox, nleaf}, base[2] = {0, nbox};
    D.ids.reserve(sizeof(int) * (nbox + nleaf));
    D.keys.reserve(sizeof(unsigned) * (nbox + nleaf));
    D.keys_sorted.reserve(sizeof(unsigned) * (nbox + nleaf));
    D.nsel.reserve(sizeof(int) * (4 + 2 * 64));
    int* nsel_d = D.nsel.as<int>();
    int* cnt_d = nsel_d + 4;
    for (int kind = 0; kind < 2; ++kind) {
      const unsigned char* f = kind == 0 ? fb : fl;
      size_t bytes = 0;
      cub::CountingInputIterator<int> it(0);
      FMM_CUDA(cub::DeviceSelect::Flagged(nullptr, bytes, it, f, D.ids.as<int>() + base[kind],
                                          nsel_d + kind, (int)nn[kind], c->st));
      D.cub_tmp.reserve(bytes);
      FMM_CUDA(cub::DeviceSelect::Flagged(D.cub_tmp.p, bytes, it, f,
                                          D.ids.as<int>() + base[kind], nsel_d + kind,
                                          (int)nn[kind], c->st));
    }
    int nsel[2] = {0, 0};
    FMM_CUDA(cudaMemcpyAsync(nsel, nsel_d, sizeof nsel, cudaMemcpyDeviceToHost, c->st));
    sync(c);
    int bits = 1;
    while ((1 << bits) < G) ++bits;
    for (int kind = 0; kind < 2; ++kind) {
      D.req_ids[kind].reserve(sizeof(int) * std::max(1, nsel[kind]));
      if (nsel[kind] > 0) {
        note_launch();
        launch(k_owner_keys, nblk(nsel[kind], 256), 256, 0, c->st, nsel_d + kind,
               D.ids.as<int>() + base[kind], s0, kind == 0 ? -1 : L,
               D.keys.as<unsigned>() + base[kind]);
        sort_pairs(D.cub_tmp, D.keys.as<unsigned>() + base[kind],
                   D.keys_sorted.as<unsigned>() + base[kind], D.ids.as<int>() + base[kind],
                   D.req_ids[kind].as<int>(), nsel[kind], bits, c->st);
      }
      note_launch();
      launch(k_owner_counts, 1, 64, 0, c->st, nsel_d + kind,
             D.keys_sorted.as<unsigned>() + base[kind], G, cnt_d + kind * 64);
    }
    int cnt_h[2 * 64];
    FMM_CUDA(cudaMemcpyAsync(cnt_h, cnt_d, sizeof(int) * 2 * 64, cudaMemcpyDeviceToHost, c->st));
    sync(c);
    for (int kind = 0; kind < 2; ++kind) {
      D.req_count[kind].assign(G, 0);
      for (int q = 0; q < G; ++q) {
        D.req_count[kind][q] = cnt_h[kind * 64 + q];
        req_counts[kind * G + q] = cnt_h[kind * 64 + q];
      }
    }
    c->have_lists = true;
    return FMM2D_OK;
  });
}

// this rank's requests of `kind` (0 boxes, 1 leaves), grouped by owner
int fmm2d_dist_requests(fmm2d_ctx* c, int kind, const int32_t** d_ids) {
  if (!c || kind < 0 || kind > 1) return FMM2D_EBADARG;
  return guarded(c, [&] {
    *d_ids = dist(c).req_ids[kind].as<int>();
    return FMM2D_OK;
  });
}

// payload sizes in doubles per requested item: kind 0 (box) 2(p+1), kind 1 (leaf) 3 nmax_leaf
int fmm2d_dist_item_doubles(fmm2d_ctx* c, int kind, int64_t* n) {
  if (!c || kind < 0 || kind > 1) return FMM2D_EBADARG;
  return guarded(c, [&] {
    DistState& D = dist(c);
    *n = kind == 0 ? 2ll * (D.p + 1) : 3ll * D.nmax_leaf;
    return FMM2D_OK;
  });
}

// serve requests (ids received from the other ranks) / install the answers to
// this rank's own requests.  kind 1: particles (before the upward pass),
// kind 0: multipoles (after it)
int fmm2d_dist_pack(fmm2d_ctx* c, int kind, const int32_t* d_ids, int64_t nids, double* d_send) {
  if (!c || kind < 0 || kind > 1) return FMM2D_EBADARG;
  return guarded(c, [&] {
    DistState& D = dist(c);
    if (nids <= 0) return FMM2D_OK;
    const TreeState& T = c->T;
    note_launch();
    if (kind == 1)
      launch(k_leaf_pack, nblk(nids * D.nmax_leaf, 256), 256, 0, c->st, 
          nids, d_ids, D.leaf_off.as<int>(), (int)D.nmax_leaf, T.src_pos.as<double2>(),
          T.src_g.as<double>(), d_send);
    else
      launch(k_row_pack, nblk(nids * (D.p + 1), 256), 256, 0, c->st, 
          nids, d_ids, D.p, c->E.mult.as<double2>() + 0, reinterpret_cast<double2*>(d_send));
    return FMM2D_OK;
  });
}

int fmm2d_dist_unpack(fmm2d_ctx* c, int kind, const double* d_recv) {
  if (!c || kind < 0 || kind > 1) return FMM2D_EBADARG;
  return guarded(c, [&] {
    DistState& D = dist(c);
    long long nids = 0;
    for (long long v : D.req_count[kind]) nids += v;
    if (nids <= 0) return FMM2D_OK;
    TreeState& T = c->T;
    note_launch();
    if (kind == 1)
      launch(k_leaf_unpack, nblk(nids * D.nmax_leaf, 256), 256, 0, c->st, 
          nids, D.req_ids[1].as<int>(), D.leaf_off.as<int>(), (int)D.nmax_leaf, d_recv,
          T.src_pos.as<double2>(), T.src_g.as<double>());
    else
      launch(k_row_unpack, nblk(nids * (D.p + 1), 256), 256, 0, c->st, 
          nids, D.req_ids[0].as<int>(), D.p, reinterpret_cast<const double2*>(d_recv),
          c->E.mult.as<double2>());
    return FMM2D_OK;
  });
}

// P2M + P2L on owned leaves, M2M down to the first owned level; packs the
// owned level-ltop multipoles into d_top_send (2(p+1) doubles per box)
int fmm2d_dist_upward(fmm2d_ctx* c, double* d_top_send, int64_t* top_boxes) {
  if (!c) return FMM2D_EBADARG;
  return guarded(c, [&] {
    DistState& D = dist(c);
    const TreeState& T = c->T;
    ExpState& E = c->E;
    const int L = D.L, p = D.p, lt = D.part.ltop();
    record(c, 4);
    FMM_CUDA(cudaMemsetAsync(E.local.p, 0, sizeof(double2) * level_base(L) * (p + 1), c->st));
    run_upward(T, c->Ls, E, D.leaf_off.as<int>(), c->d_status.as<DevStatus>(), c->st, D.part);
    record(c, 5);
    run_m2m(T, E, c->st, D.part, std::max(lt, 1), L - 1);
    const long long k0 = D.part.lo(lt), cnt = D.part.hi(lt) - k0;
    note_launch();
    launch(k_level_rows, nblk(cnt * (p + 1), 256), 256, 0, c->st, 
        k0, cnt, level_base(lt), p, E.mult.as<double2>(), reinterpret_cast<double2*>(d_top_send),
        true);
    *top_boxes = cnt;
    return FMM2D_OK;
  });
}

// install the allgathered level-ltop multipoles; M2M on the shared levels
int fmm2d_dist_upward_top(fmm2d_ctx* c, const double* d_top_all) {
  if (!c) return FMM2D_EBADARG;
  return guarded(c, [&] {
    DistState& D = dist(c);
    const TreeState& T = c->T;
    ExpState& E = c->E;
    const int p = D.p, lt = D.part.ltop();
    const long long nb = 1ll << (2 * lt);
    note_launch();
    launch(k_level_rows, nblk(nb * (p + 1), 256), 256, 0, c->st, 
        0, nb, level_base(lt), p, E.mult.as<double2>(),
        const_cast<double2*>(reinterpret_cast<const double2*>(d_top_all)), false);
    if (lt - 1 >= 1) run_m2m(T, E, c->st, D.part, 1, lt - 1);
    record(c, 6);
    return FMM2D_OK;
  });
}

// M2L, L2L, L2P + M2P and P2P of the owned targets.  Outputs the owned values
// in tree order (d_vals, n_r complex) and their original indices (d_idx,
// int64); rep: this rank's phase times and counts.
int fmm2d_dist_downward(fmm2d_ctx* c, double* d_vals, int64_t* d_idx, fmm2d_report* rep) {
  if (!c) return FMM2D_EBADARG;
  return guarded(c, [&] {
    DistState& D = dist(c);
    TreeState& T = c->T;
    ListState& Ls = c->Ls;
    ExpState& E = c->E;
    const int L = D.L;
    DevStatus* dst = c->d_status.as<DevStatus>();
    record(c, 7);
    run_m2l(T, Ls, E, dst, c->st);
    record(c, 8);
    run_l2l(T, E, dst, c->st, D.part);
    record(c, 9);
    // owned evaluation points: the subtree's sources (aliased, tree-order range
    // [g0, g0 + n_r) of the global arrays) or its separate points (local 0..m_r)
    const long long e0 = D.separate ? 0 : D.g0, ne = D.separate ? D.m_r : D.n_r;
    run_l2p_m2p(T, Ls, E, dst, c->st, e0, e0 + ne, D.part.lo(L), D.part.hi(L));
    record(c, 10);
    run_p2p(T, Ls, E, D.leaf_off.as<int>(), reinterpret_cast<double2*>(d_vals), dst, c->st,
            D.part, e0);
    if (ne > 0) {
      note_launch();
      launch(k_fill_owned_idx, nblk(ne, 256), 256, 0, c->st, ne,
             (D.separate ? T.eval_perm.as<int>() : T.src_perm.as<int>() + D.g0),
             reinterpret_cast<long long*>(d_idx));
    }
    record(c, 11);
    run_stats(T, Ls, dst, c->st, D.part);
    fetch_status(c);
    FMM_CUDA(cudaMemcpyAsync(c->h_hist, Ls.hist.p, sizeof(int) * 4 * HIST_BINS,
                             cudaMemcpyDeviceToHost, c->st));
    sync(c);
    const DevStatus& s = *c->h_status;
    if (s.flags & ST_P2L_SINGULAR)
      throw ApiError{FMM2D_ESINGULAR, "p2l source coincides with the expansion center"};
    if (s.flags & ST_M2L_SINGULAR)
      throw ApiError{FMM2D_ESINGULAR, "m2l shift must be nonzero (boxes are separated)"};
    if (s.flags & ST_M2P_SINGULAR)
      throw ApiError{FMM2D_ESINGULAR, "m2p target coincides with the expansion center"};
    c->have_eval = true;
    if (rep) {
      fmm2d_report r;
      std::memset(&r, 0, sizeof r);
      // sort (load .. subtree) | connect | p2m (+p2l) | m2m | m2l | l2l | l2p | p2p
      r.phase_ms[0] = ev_ms(D.ev[0], D.ev[2]);
      r.phase_ms[1] = ev_ms(D.ev[2], D.ev[3]);
      r.phase_ms[2] = ev_ms(D.ev[4], D.ev[5]);
      r.phase_ms[3] = ev_ms(D.ev[5], D.ev[6]);
      r.phase_ms[4] = ev_ms(D.ev[7], D.ev[8]);
      r.phase_ms[5] = ev_ms(D.ev[8], D.ev[9]);
      r.phase_ms[6] = ev_ms(D.ev[9], D.ev[10]);
      r.phase_ms[7] = ev_ms(D.ev[10], D.ev[11]);
      r.device_ms = ev_ms(D.ev[0], D.ev[11]);
      r.n_levels = L;
      r.n_boxes = level_base(L + 1);
      leaf_stats(D.n_total, L, &r);
      r.p2p_skips = (long long)s.p2p_skips;
      const long long nbox = level_base(L + 1), nleaf = 1ll << (2 * L);
      int tw = 0, sh = 0, tp[3] = {0, 0, 0};
      const int lt = D.part.ltop();
      {
        // the five list totals in one kernel + one copy (the stream is idle here)
        D.totals5.reserve(sizeof(int) * 8);
        note_launch();
        launch(k_pick5, 1, 32, 0, c->st, Ls.weak_off.as<int>() + nbox,
               Ls.weak_off.as<int>() + level_base(lt), Ls.p2p_off.as<int>() + nleaf,
               Ls.p2l_off.as<int>() + nleaf, Ls.m2p_off.as<int>() + nleaf,
               D.totals5.as<int>());
        int v[5];
        FMM_CUDA(cudaMemcpyAsync(v, D.totals5.p, sizeof v, cudaMemcpyDeviceToHost, c->st));
        sync(c);
        tw = v[0];
        sh = v[1];
        tp[0] = v[2];
        tp[1] = v[3];
        tp[2] = v[4];
      }
      // weak pairs of shared targets are computed by every rank: count them on rank 0
      r.list_totals[0] = tw - (D.part.rank == 0 ? 0 : sh);
      r.list_totals[1] = tp[0];
      r.list_totals[2] = tp[1];
      r.list_totals[3] = tp[2];
      for (int q = 0; q < 4; ++q) r.max_len[q] = s.max_len[q];
      r.kernel_launches = g_launches;
      *rep = r;
    }
    return FMM2D_OK;
  });
}

// out[idx[i]] = vals[i] for i < n (device pointers): assembles gathered values
int fmm2d_scatter_values(fmm2d_ctx* c, int64_t n, const double* d_vals, const int64_t* d_idx,
                         double* d_out) {
  if (!c) return FMM2D_EBADARG;
  return guarded(c, [&] {
    if (n <= 0) return FMM2D_OK;
    note_launch();
    launch(k_scatter_values, nblk(n, 256), 256, 0, c->st, 
        n, reinterpret_cast<const double2*>(d_vals), reinterpret_cast<const long long*>(d_idx),
        reinterpret_cast<double2*>(d_out));
    return FMM2D_OK;
  });
}

int fmm2d_dist_end(fmm2d_ctx* c) {
  if (!c) return FMM2D_EBADARG;
  return guarded(c, [&] {
    FMM_CUDA(cudaStreamSynchronize(c->st));
    c->D.active = false;
    c->st = c->own_st;
    return FMM2D_OK;
  });
}

}  // extern "C"
