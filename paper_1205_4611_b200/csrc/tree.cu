// Tree build ("sort" phase): the asymmetric-adaptive pyramid of successive
// median splits, bit-exact with the reference's canonical form.
//
// Reference: tree.py:230-334 (build_tree), :160-177 (partition_median),
// :258-285 (_split_sources/_split_evals/_cut_rect), geometry.py:57-63.
//
// Design (B200): instead of a k-th-element selection per box per split step,
// every source gets its global rank along x and along y once (two 64-bit key
// radix sorts, ties by index).  Each split segment is kept twice, ordered by
// x-rank and by y-rank.  Splitting a segment along x is then free in the
// x-ordered copy (left = first k) and a stable partition "rank_x <= cut rank"
// in the y-ordered copy -- so every step moves one 8-byte (rank_x, rank_y)
// record per source and never selects.  Because every partition is stable
// from the identity order, each segment's members are always in ascending
// original index, which is exactly the canonical tree.  Top steps (large
// segments) run as tiled global partitions; once a segment fits in shared
// memory one CTA finishes its whole subtree in SMEM.  Evaluation points do
// not influence the cuts: each one descends the finished cut table
// (`coord <= cut`, tree.py:210) to its leaf, then a stable radix sort by leaf
// yields eval_perm.
#include <cub/device/device_radix_sort.cuh>

#include "engine.h"
#include "lookback.cuh"

namespace fmm {

namespace {

constexpr int PART_THREADS = 256;
#ifndef TREE_PART_DESC
#define TREE_PART_DESC 1   // split steps read a per-tile descriptor + flag byte
#endif
#ifndef TREE_SUB_PIPE
#define TREE_SUB_PIPE 1   // subtree step tables finished after the partition passes
#endif
#ifndef TREE_PART_ITEMS
#define TREE_PART_ITEMS 4
#endif
#ifndef TREE_SUB_THREADS
#define TREE_SUB_THREADS 512
#endif
#ifndef TREE_KEY_EXTRA
#define TREE_KEY_EXTRA 4   // rank key bits beyond log2 N (rounded up to a radix digit)
#endif
#ifndef TREE_FUSE_RECORDS_MAX
#define TREE_FUSE_RECORDS_MAX (1ll << 22)
#endif
#ifndef TREE_FORK_SORT
#define TREE_FORK_SORT 1   // y-axis rank sort on a side stream
#endif
#ifndef TREE_FORK_MIN
#define TREE_FORK_MIN 4096
#endif
#ifndef TREE_SMEM_BUDGET
#define TREE_SMEM_BUDGET (110 * 1024)
#endif
constexpr int PART_ITEMS = TREE_PART_ITEMS;
constexpr int PART_TILE = PART_THREADS * PART_ITEMS;
constexpr int SUB_THREADS = TREE_SUB_THREADS;
constexpr int SMEM_BUDGET = TREE_SMEM_BUDGET;   // two subtree CTAs per SM
constexpr int LEAF_SMEM_MAX = 512;        // in-SMEM index sort of leaves up to this size

struct Rect {
  double x0, x1, y0, y1;
};

// --------------------------------------------------------------------------
// bounding box of sources and evaluation points (tree.py:256-259)
__device__ __forceinline__ void block_minmax(double& x0, double& x1, double& y0, double& y1,
                                             double (*sw)[32]) {
  for (int d = 16; d; d >>= 1) {
    x0 = fmin(x0, __shfl_xor_sync(0xffffffffu, x0, d));
    x1 = fmax(x1, __shfl_xor_sync(0xffffffffu, x1, d));
    y0 = fmin(y0, __shfl_xor_sync(0xffffffffu, y0, d));
    y1 = fmax(y1, __shfl_xor_sync(0xffffffffu, y1, d));
  }
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5, nw = blockDim.x >> 5;
  __syncthreads();
  if (lane == 0) { sw[0][w] = x0; sw[1][w] = x1; sw[2][w] = y0; sw[3][w] = y1; }
  __syncthreads();
  x0 = lane < nw ? sw[0][lane] : INFINITY;
  x1 = lane < nw ? sw[1][lane] : -INFINITY;
  y0 = lane < nw ? sw[2][lane] : INFINITY;
  y1 = lane < nw ? sw[3][lane] : -INFINITY;
  for (int d = 16; d; d >>= 1) {
    x0 = fmin(x0, __shfl_xor_sync(0xffffffffu, x0, d));
    x1 = fmax(x1, __shfl_xor_sync(0xffffffffu, x1, d));
    y0 = fmin(y0, __shfl_xor_sync(0xffffffffu, y0, d));
    y1 = fmax(y1, __shfl_xor_sync(0xffffffffu, y1, d));
  }
}

// tight bounding rectangle of sources and evaluation points (tree.py:256-259),
// written straight into the root entry of the rectangle table
__global__ void __launch_bounds__(256)
k_bbox(const double2* __restrict__ pos, long long n, const double2* __restrict__ epos,
       long long m, Rect* root, unsigned int* counter, double* partial) {
  pdl_enter();
  double x0 = INFINITY, x1 = -INFINITY, y0 = INFINITY, y1 = -INFINITY;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n + m;
       i += (long long)gridDim.x * blockDim.x) {
    double2 z = i < n ? pos[i] : epos[i - n];
    x0 = fmin(x0, z.x); x1 = fmax(x1, z.x);
    y0 = fmin(y0, z.y); y1 = fmax(y1, z.y);
  }
  __shared__ double sw[4][32];
  __shared__ bool last;
  block_minmax(x0, x1, y0, y1, sw);
  if (threadIdx.x == 0) {
    partial[4 * blockIdx.x + 0] = x0; partial[4 * blockIdx.x + 1] = x1;
    partial[4 * blockIdx.x + 2] = y0; partial[4 * blockIdx.x + 3] = y1;
    __threadfence();
    last = atomicAdd(counter, 1u) == gridDim.x - 1;
  }
  __syncthreads();
  if (!last) return;
  __threadfence();
  x0 = INFINITY; x1 = -INFINITY; y0 = INFINITY; y1 = -INFINITY;
  for (unsigned q = threadIdx.x; q < gridDim.x; q += blockDim.x) {
    x0 = fmin(x0, __ldcg(partial + 4 * q + 0)); x1 = fmax(x1, __ldcg(partial + 4 * q + 1));
    y0 = fmin(y0, __ldcg(partial + 4 * q + 2)); y1 = fmax(y1, __ldcg(partial + 4 * q + 3));
  }
  block_minmax(x0, x1, y0, y1, sw);
  if (threadIdx.x == 0) {
    *root = Rect{x0, x1, y0, y1};
    *counter = 0;
  }
}

// --------------------------------------------------------------------------
// rank keys
__global__ void k_make_keys(const double2* __restrict__ pos, long long n, int axis,
                            unsigned long long* keys, int* vals) {
  pdl_enter();
  long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (i >= n) return;
  double2 z = pos[i];
  keys[i] = ordered_key(axis ? z.y : z.x);
  vals[i] = (int)i;
}

// 32-bit monotone key: fixed point of (c - lo) / (hi - lo) over the root
// rectangle.  Non-decreasing in c (every step rounds monotonically), so a
// stable sort by it orders the points up to runs of equal keys, which
// k_fix_ties then orders exactly by (coordinate, index).
__global__ void k_make_keys32(const double2* __restrict__ pos, long long n,
                              const Rect* __restrict__ root, unsigned* keys, int* vals,
                              int shift) {
  pdl_enter();
  const long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (i >= n) return;
  const Rect r = *root;
  const double2 z = pos[i];
  // both axes in one pass: x keys in keys[0, n), y keys in keys[n, 2n)
#pragma unroll
  for (int axis = 0; axis < 2; ++axis) {
    const double lo = axis ? r.y0 : r.x0, span = axis ? r.y1 - r.y0 : r.x1 - r.x0;
    const double c = axis ? z.y : z.x;
    unsigned k = 0;
    if (span > 0.0) {
      const double u = (c - lo) / span * 4294967296.0;
      k = u >= 4294967295.0 ? 0xffffffffu : (unsigned)u;
    }
    keys[axis * n + i] = k >> shift;   // key_bits = 32 - shift (ties fixed exactly by k_fix_ties)
  }
  vals[i] = (int)i;
}

constexpr int TIE_RUN_MAX = 64;

// order every run of equal 32-bit keys by (coordinate, original index) and
// write the inverse permutation (rank of every point along the axis) in the
// same pass: singletons scatter their rank directly, a run's head thread
// sorts the run and scatters its members' ranks.  A run longer than
// TIE_RUN_MAX (pathologically clustered input) raises ST_RANK_RETRY and the
// host reruns with exact 64-bit keys.
//
// The y pass (X != null) writes the split records directly instead of
// rank_y: a point of y rank r and x rank rx is (rx, r) at Y[r] and X[rx]
// (what k_init_arrays builds from both rank arrays in the exact-key path).
struct RankOut {
  int* rank;                 // x pass: rank along the axis
  const int* rank_x;         // y pass: x ranks ...
  int2* X;                   // ... and the two record copies
  int2* Y;
  unsigned char* xpar;
  unsigned char* ypar;
};
__device__ __forceinline__ void emit_rank(const RankOut& o, int idx, int r, long long n) {
  if (o.X) {
    const int rx = o.rank_x[idx];
    o.Y[r] = make_int2(rx, r);
    // rank_x is incomplete only when the x pass raised ST_RANK_RETRY (the
    // build is then redone with exact keys): never scatter out of range
    if ((unsigned long long)rx < (unsigned long long)n) o.X[rx] = make_int2(rx, r);
  } else {
    o.rank[idx] = r;
  }
}

__global__ void k_fix_ties(const unsigned* __restrict__ keys, int* perm,
                           const double2* __restrict__ pos, int axis, long long n, RankOut o,
                           DevStatus* st) {
  pdl_enter();
  const long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (i >= n) return;
  if (i == 0 && o.X) { o.xpar[0] = 0; o.ypar[0] = 0; }
  const unsigned k = keys[i];
  if (i > 0 && keys[i - 1] == k) return;                 // run member: the head writes it
  if (i + 1 >= n || keys[i + 1] != k) {                  // singleton
    emit_rank(o, perm[i], (int)i, n);
    return;
  }
  long long e = i + 1;
  while (e < n && keys[e] == k) {
    if (++e - i > TIE_RUN_MAX) {
      atomicOr(&st->flags, ST_RANK_RETRY);
      // still emit a valid (if not exactly ordered) permutation, so the rest
      // of this attempt indexes in bounds before the host reruns it
      while (e < n && keys[e] == k) ++e;
      for (long long q = i; q < e; ++q) emit_rank(o, perm[q], (int)q, n);
      return;
    }
  }
  const int cnt = (int)(e - i);
  int idx[TIE_RUN_MAX];
  double crd[TIE_RUN_MAX];
  for (int q = 0; q < cnt; ++q) {
    idx[q] = perm[i + q];
    const double2 z = pos[idx[q]];
    crd[q] = axis ? z.y : z.x;
  }
  for (int q = 1; q < cnt; ++q) {      // insertion sort, stable in index
    const int vi = idx[q];
    const double vc = crd[q];
    int r = q - 1;
    while (r >= 0 && (crd[r] > vc || (crd[r] == vc && idx[r] > vi))) {
      idx[r + 1] = idx[r];
      crd[r + 1] = crd[r];
      --r;
    }
    idx[r + 1] = vi;
    crd[r + 1] = vc;
  }
  for (int q = 0; q < cnt; ++q) {
    perm[i + q] = idx[q];
    emit_rank(o, idx[q], (int)(i + q), n);
  }
  // x pass: exactly equal x are adjacent now; equal y as well means two
  // sources coincide, so P2P must test r2 == 0 per pair (ST_DUPLICATES)
  if (axis == 0) {
    bool dup = false;
    for (int q = 1; q < cnt && !dup; ++q)
      for (int r = q - 1; r >= 0 && crd[r] == crd[q] && !dup; --r)
        dup = pos[idx[r]].y == pos[idx[q]].y;
    if (dup) atomicOr(&st->flags, ST_DUPLICATES);
  }
}

// inverse permutation: rank of every point along the sorted axis (an
// L2-resident scatter; the coordinates are looked up only at the cuts)
__global__ void k_rank_scatter(long long n, const int* __restrict__ perm, int* rank) {
  pdl_enter();
  const long long r = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (r < n) rank[perm[r]] = (int)r;
}

__global__ void k_init_arrays(long long n, const int* __restrict__ perm_x,
                              const int* __restrict__ perm_y, const int* __restrict__ rank_x,
                              const int* __restrict__ rank_y, int2* X, int2* Y,
                              unsigned char* xpar, unsigned char* ypar) {
  pdl_enter();
  long long r = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (r == 0) { xpar[0] = 0; ypar[0] = 0; }
  if (r >= n) return;
  X[r] = make_int2((int)r, rank_y[perm_x[r]]);
  Y[r] = make_int2(rank_x[perm_y[r]], (int)r);
}

// --------------------------------------------------------------------------
// one split step, per segment: axis, cut, child rectangles, degenerate check
struct StepArgs {
  const int* off;           // step offsets table
  Rect* rect_tab;
  double* cut_tab;
  unsigned char* axis_tab;
  const double2* pos;       // input positions (original order)
  const int* perm_x;        // original index at every x rank
  const int* perm_y;        // ... and y rank
  int L;
  int s0;                   // global step of local step 0 (subtree builds)
  long long seg;            // global index of the local root segment at step s0
};

// The dependent global reads are issued in two waves instead of a chain of
// seven: (1) the rectangle and every permutation entry either axis could
// need, (2) the coordinates of the selected entries -- the ranks are known,
// only the axis comes from the rectangle.  Every caller waits on this at a
// barrier or a look-back, so the round trips are the step's critical path.
__device__ __forceinline__ void prepare_segment(const StepArgs& a, int s, long long j, int s0,
                                                int n, int2 x_first, int2 x_last, int2 y_first,
                                                int2 y_last, int2 x_kth, int2 y_kth, int2 x_next,
                                                int2 y_next, DevStatus* st, int* cut_rank_out,
                                                bool* along_y_out) {
  const int sg = s + a.s0;                                          // global step
  const bool deg = (sg & 1) == 0 && (sg >> 1) < a.L;                // tree.py:285
  const int k = (n + 1) / 2;
  // wave 1
  const Rect r = a.rect_tab[step_base(s) + j];
  const int ikx = a.perm_x[x_kth.x], iky = a.perm_y[y_kth.y];
  const int inx = a.perm_x[x_next.x], iny = a.perm_y[y_next.y];
  const int ixa = a.perm_x[x_first.x], ixb = a.perm_x[x_last.x];
  const int iya = a.perm_y[y_first.y], iyb = a.perm_y[y_last.y];
  const bool along_y = (r.y1 - r.y0) / 2 > (r.x1 - r.x0) / 2;      // geometry.py:63
  // wave 2: coordinate of rank cr along the axis (tree.py:202), the next
  // one, and the four extremes of the degenerate check
  const double2 pc = a.pos[along_y ? iky : ikx];
  const double2 pn = a.pos[along_y ? iny : inx];
  const double2 pxa = a.pos[ixa], pxb = a.pos[ixb], pya = a.pos[iya], pyb = a.pos[iyb];
  const int cr = along_y ? y_kth.y : x_kth.x;
  const double cut = along_y ? pc.y : pc.x;
  if (deg && pxa.x == pxb.x && pya.y == pyb.y) {
    unsigned long long key = ((unsigned long long)(sg >> 1) << 40) |
                             (unsigned long long)((a.seg << s) + j);
    atomicMin(&st->degenerate_key, key);
    atomicOr(&st->flags, ST_DEGENERATE);
  }
  // evaluation points split by coord <= cut (tree.py:210): they follow the
  // sources' median split exactly unless the (k+1)-th coordinate equals the cut
  if (k < n && (along_y ? pn.y : pn.x) == cut) atomicOr(&st->flags, ST_EVAL_TIES);
  a.cut_tab[step_base(s) + j] = cut;
  a.axis_tab[step_base(s) + j] = along_y;
  Rect lo = r, hi = r;                                              // tree.py:218-222
  if (along_y) { lo.y1 = cut; hi.y0 = cut; } else { lo.x1 = cut; hi.x0 = cut; }
  a.rect_tab[step_base(s + 1) + 2 * j] = lo;
  a.rect_tab[step_base(s + 1) + 2 * j + 1] = hi;
  *cut_rank_out = cr;
  *along_y_out = along_y;
  (void)s0;
}

// per-tile descriptors of a split step (TREE_PART_DESC): static {segment,
// tile start, segment start, end}, the flag bytes of this step (null: the
// first step, read the segment tables) and of the next (null: the subtree
// kernel takes over), and the next step's first tile per segment
struct PartDesc {
  const int* desc;
  const unsigned char* flag_in;
  unsigned char* flag_out;
  const int* segt_next;
};

// stable partition of the moving copy, tiles aligned to segments
__device__ __forceinline__ bool part_flag(int2 e, bool along_y, int cr) {
  return (along_y ? e.y : e.x) <= cr;
}

// One global split step in ONE pass (replaces prepare / count / scan /
// scatter): tiles are segment-aligned and taken in ticket order; every tile
// derives its segment's axis and cut rank, the segment's first tile also
// writes the step tables (cut, axis, child rectangles, parities, checks); a
// segmented decoupled look-back gives each tile the number of left-going
// elements of its segment before it; the stable partition is then written.
__global__ void __launch_bounds__(PART_THREADS)
k_part_step(StepArgs a, int s, const int* __restrict__ tile_seg,
            const int* __restrict__ tile_start, int2* X0, int2* X1, int2* Y0, int2* Y1,
            const unsigned char* xpar, const unsigned char* ypar, unsigned char* xpar_next,
            unsigned char* ypar_next, LookbackPacked lbs, unsigned ntiles, DevStatus* st,
            PartDesc pd) {
  pdl_enter();
  __shared__ unsigned s_tile;
  __shared__ int sw[PART_THREADS / 32];
  __shared__ long long s_excl;
  if (threadIdx.x == 0) s_tile = lb_ticket(lbs, ntiles);
  __syncthreads();
  const unsigned t = s_tile;
#if TREE_PART_DESC
  // one round trip for everything the partition needs: the static tile
  // descriptor and the flag byte the previous step's head tile wrote
  // (parities and axis); only the first step reads the segment tables
  const int4 td = reinterpret_cast<const int4*>(pd.desc)[t];
  const unsigned fl = pd.flag_in ? pd.flag_in[t] : 0u;
  const int j = td.x, tstart = td.y, s0 = td.z, end = td.w, n = end - s0, k = (n + 1) / 2;
  unsigned char xp, yp;
  bool along_y;
  if (pd.flag_in) {
    xp = fl & 1u;
    yp = (fl >> 1) & 1u;
    along_y = (fl >> 2) & 1u;
  } else {
    xp = xpar[j];
    yp = ypar[j];
    const Rect r = a.rect_tab[step_base(s) + j];
    along_y = (r.y1 - r.y0) / 2 > (r.x1 - r.x0) / 2;              // geometry.py:63
  }
  const int2* X = xp ? X1 : X0;
  const int2* Y = yp ? Y1 : Y0;
  const bool head = tstart == s0;
#else
  const int j = tile_seg[t];
  const int* off = a.off + off_base(s);
  const int s0 = off[j], end = off[j + 1], n = end - s0, k = (n + 1) / 2;
  const unsigned char xp = xpar[j], yp = ypar[j];
  const int2* X = xp ? X1 : X0;
  const int2* Y = yp ? Y1 : Y0;
  const int tstart = tile_start[t];
  const bool head = tstart == s0;
  const Rect r = a.rect_tab[step_base(s) + j];
  const bool along_y = (r.y1 - r.y0) / 2 > (r.x1 - r.x0) / 2;      // geometry.py:63
#endif
  const int cr = along_y ? Y[s0 + k - 1].y : X[s0 + k - 1].x;
  const int2* M = along_y ? X : Y;
  int2* D = along_y ? (xp ? X0 : X1) : (yp ? Y0 : Y1);
  const int tend = min(end, tstart + PART_TILE);
  const int base = tstart + threadIdx.x * PART_ITEMS;
  int2 e[PART_ITEMS];
  bool f[PART_ITEMS];
  int c = 0;
#pragma unroll
  for (int q = 0; q < PART_ITEMS; ++q) {
    const int i = base + q;
    f[q] = false;
    if (i < tend) {
      e[q] = M[i];
      f[q] = part_flag(e[q], along_y, cr);
      c += f[q];
    }
  }
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  int incl = c;
#pragma unroll
  for (int d = 1; d < 32; d <<= 1) {
    const int o = __shfl_up_sync(0xffffffffu, incl, d);
    if (lane >= d) incl += o;
  }
  if (lane == 31) sw[w] = incl;
  __syncthreads();
  if (w == 0) {
    unsigned agg = 0;
    for (int q = 0; q < PART_THREADS / 32; ++q) agg += sw[q];
    const unsigned excl = lb_prefix_packed(lbs, t, agg, head);
    if (lane == 0) s_excl = excl;
  }
  __syncthreads();
  int wpre = 0;
  for (int q = 0; q < w; ++q) wpre += sw[q];
  int lp = (int)s_excl + wpre + incl - c;   // left elements of this segment before `base`
#pragma unroll
  for (int q = 0; q < PART_ITEMS; ++q) {
    const int i = base + q;
    if (i < tend) {
      const int dst = f[q] ? s0 + lp : s0 + k + (i - s0) - lp;
      D[dst] = e[q];
      lp += f[q];
    }
  }
  // the segment's first tile writes the next step's tables -- after its own
  // scatter, off the look-back chain that every later tile of the segment
  // waits on (the next step reads them after this launch completes)
  if (head && threadIdx.x == 0) {
    int cr2;
    bool ay2;
    const int kn = k < n ? k : k - 1;
    prepare_segment(a, s, j, s0, n, X[s0], X[s0 + n - 1], Y[s0], Y[s0 + n - 1], X[s0 + k - 1],
                    Y[s0 + k - 1], X[s0 + kn], Y[s0 + kn], st, &cr2, &ay2);
    // the copy ordered along the split axis stays put; the other one moves
    const unsigned char nxp = along_y ? (unsigned char)(1 - xp) : xp;
    const unsigned char nyp = along_y ? yp : (unsigned char)(1 - yp);
    xpar_next[2 * j] = nxp; xpar_next[2 * j + 1] = nxp;
    ypar_next[2 * j] = nyp; ypar_next[2 * j + 1] = nyp;
#if TREE_PART_DESC
    if (pd.flag_out) {
      // children's flag bytes, one per tile of the next step (axis from the
      // child rectangles prepare_segment just wrote)
      const Rect lo = a.rect_tab[step_base(s + 1) + 2 * j];
      const Rect hi = a.rect_tab[step_base(s + 1) + 2 * j + 1];
      const unsigned base = nxp | (nyp << 1);
      const unsigned f0 = base | (((lo.y1 - lo.y0) / 2 > (lo.x1 - lo.x0) / 2) ? 4u : 0u);
      const unsigned f1 = base | (((hi.y1 - hi.y0) / 2 > (hi.x1 - hi.x0) / 2) ? 4u : 0u);
      const int c0 = pd.segt_next[2 * j], c1 = pd.segt_next[2 * j + 1],
                c2 = pd.segt_next[2 * j + 2];
      for (int q = c0; q < c1; ++q) pd.flag_out[q] = (unsigned char)f0;
      for (int q = c1; q < c2; ++q) pd.flag_out[q] = (unsigned char)f1;
    }
#endif
  }
}

// --------------------------------------------------------------------------
// subtree kernel: all remaining split steps of one segment inside SMEM
struct SubArgs {
  StepArgs a;
  int sb, S;
  const int2 *X0, *X1, *Y0, *Y1;
  const unsigned char *xpar, *ypar;
  const int* perm_x;
  const double2* pos;
  const double* g;
  double2* src_pos;
  double* src_g;
  int* src_perm;
  int* leaf_of;           // fallback: leaf id per original index
  bool in_smem_finalize;
  int nmax;
  long long out0;         // tree-order offset of the outputs (subtree builds)
  const int* orig;        // original index of every input point (null: identity)
};

__global__ void __launch_bounds__(SUB_THREADS)
k_subtree(SubArgs A, DevStatus* st) {
  pdl_enter();
  extern __shared__ unsigned char smem_raw[];
  const long long j0 = blockIdx.x;
  const int* off_sb = A.a.off + off_base(A.sb);
  const int g0 = off_sb[j0];
  const int n = off_sb[j0 + 1] - g0;
  const int nmax = A.nmax;
  const int nseg_max = 1 << (A.S - A.sb);
#if TREE_SUB_PIPE
  Rect* s_rect = reinterpret_cast<Rect*>(smem_raw);       // this CTA's segment rectangles
  int2* sx = reinterpret_cast<int2*>(s_rect + nseg_max);
#else
  int2* sx = reinterpret_cast<int2*>(smem_raw);
#endif
  int2* sy = sx + nmax;
  int2* scr = sy + nmax;
  unsigned short* segid = reinterpret_cast<unsigned short*>(scr + nmax);
  int* q_s0 = reinterpret_cast<int*>(segid + ((nmax + 1) & ~1));
  int* q_k = q_s0 + nseg_max;
  int* q_cr = q_k + nseg_max;
  int* q_P = q_cr + nseg_max;
  unsigned char* q_ax = reinterpret_cast<unsigned char*>(q_P + nseg_max);

  {
    const int2* X = A.xpar[j0] ? A.X1 : A.X0;
    const int2* Y = A.ypar[j0] ? A.Y1 : A.Y0;
    for (int i = threadIdx.x; i < n; i += blockDim.x) {
      sx[i] = X[g0 + i];
      sy[i] = Y[g0 + i];
      segid[i] = 0;
    }
  }
  __syncthreads();

  // every warp owns a contiguous, 32-aligned element range; lanes take
  // consecutive elements (coalesced, bank-conflict-free SMEM) and the stable
  // partition positions come from ballots: prefix = warp base + popc(lower lanes)
  constexpr int NW = SUB_THREADS / 32;
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int wchunk = ((n + NW - 1) / NW + 31) & ~31;
  const int w0 = min(n, w * wchunk), w1 = min(n, w0 + wchunk);
  const unsigned lt_mask = (1u << lane) - 1u;
  __shared__ int s_wpre[NW];
  int* q_loc = q_P;                      // per segment: local prefix at its start ...
  unsigned char* q_w = reinterpret_cast<unsigned char*>(q_ax + nseg_max);  // ... and its warp

  for (int s = A.sb; s < A.S; ++s) {
    const int nloc = 1 << (s - A.sb);
    const int* off = A.a.off + off_base(s);
#if TREE_SUB_PIPE
    // segment q = threadIdx.x (nloc <= SUB_THREADS, checked by the host):
    // the axis comes from the rectangle this CTA computed one step earlier
    // (SMEM) and the cut rank from the SMEM records, so the partition starts
    // after one round trip (the rank -> original index lookups); the
    // coordinate loads behind them land during the two partition passes and
    // the step tables are finished after them (prepare_segment's work, split)
    const int q = threadIdx.x;
    const bool qa = q < nloc;
    const long long j = j0 * nloc + q;
    int s0 = 0, nn = 0, k = 0;
    Rect r{0.0, 0.0, 0.0, 0.0};
    bool along_y = false;
    double2 pc{}, pn{}, pxa{}, pxb{}, pya{}, pyb{};
    if (qa) {
      s0 = off[j] - g0;
      nn = off[j + 1] - off[j];
      k = (nn + 1) / 2;
      r = s == A.sb ? A.a.rect_tab[step_base(s) + j] : s_rect[q];
      along_y = (r.y1 - r.y0) / 2 > (r.x1 - r.x0) / 2;      // geometry.py:63
      const int kn = k < nn ? k : k - 1;
      const int ik = along_y ? A.a.perm_y[sy[s0 + k - 1].y] : A.a.perm_x[sx[s0 + k - 1].x];
      const int in = along_y ? A.a.perm_y[sy[s0 + kn].y] : A.a.perm_x[sx[s0 + kn].x];
      const int ixa = A.a.perm_x[sx[s0].x], ixb = A.a.perm_x[sx[s0 + nn - 1].x];
      const int iya = A.a.perm_y[sy[s0].y], iyb = A.a.perm_y[sy[s0 + nn - 1].y];
      pc = A.a.pos[ik];
      pn = A.a.pos[in];
      pxa = A.a.pos[ixa];
      pxb = A.a.pos[ixb];
      pya = A.a.pos[iya];
      pyb = A.a.pos[iyb];
      q_s0[q] = s0;
      q_k[q] = k;
      q_cr[q] = along_y ? sy[s0 + k - 1].y : sx[s0 + k - 1].x;
      q_ax[q] = along_y;
    }
#else
    for (int q = threadIdx.x; q < nloc; q += blockDim.x) {
      const long long j = j0 * nloc + q;
      const int s0 = off[j] - g0, nn = off[j + 1] - off[j], k = (nn + 1) / 2;
      int cr;
      bool along_y;
      const int kn = k < nn ? k : k - 1;
      prepare_segment(A.a, s, j, s0, nn, sx[s0], sx[s0 + nn - 1], sy[s0], sy[s0 + nn - 1],
                      sx[s0 + k - 1], sy[s0 + k - 1], sx[s0 + kn], sy[s0 + kn], st, &cr,
                      &along_y);
      q_s0[q] = s0;
      q_k[q] = k;
      q_cr[q] = cr;
      q_ax[q] = along_y;
    }
#endif
    __syncthreads();
    // pass 1: flags of the moving copy; record the in-warp prefix at segment starts
    int run = 0;
    for (int i0 = w0; i0 < w1; i0 += 32) {
      const int i = i0 + lane;
      bool f = false;
      int q = 0;
      if (i < w1) {
        q = segid[i];
        const bool ay = q_ax[q];
        f = part_flag(ay ? sx[i] : sy[i], ay, q_cr[q]);
      }
      const unsigned bal = __ballot_sync(0xffffffffu, f);
      if (i < w1 && q_s0[q] == i) {
        q_loc[q] = run + __popc(bal & lt_mask);
        q_w[q] = (unsigned char)w;
      }
      run += __popc(bal);
    }
    if (lane == 0) s_wpre[w] = run;
    __syncthreads();
    if (threadIdx.x == 0) {
      int acc = 0;
      for (int q = 0; q < NW; ++q) {
        const int v = s_wpre[q];
        s_wpre[q] = acc;
        acc += v;
      }
    }
    __syncthreads();
    for (int q = threadIdx.x; q < nloc; q += blockDim.x) q_loc[q] += s_wpre[q_w[q]];
    __syncthreads();
    // pass 2: scatter the moving copy into scratch (stable in both halves)
    run = s_wpre[w];
    for (int i0 = w0; i0 < w1; i0 += 32) {
      const int i = i0 + lane;
      bool f = false;
      int q = 0;
      int2 e = make_int2(0, 0);
      if (i < w1) {
        q = segid[i];
        const bool ay = q_ax[q];
        e = ay ? sx[i] : sy[i];
        f = part_flag(e, ay, q_cr[q]);
      }
      const unsigned bal = __ballot_sync(0xffffffffu, f);
      if (i < w1) {
        const int lp = run + __popc(bal & lt_mask) - q_loc[q];   // left elements of q before i
        const int s0 = q_s0[q];
        scr[f ? s0 + lp : s0 + q_k[q] + (i - s0) - lp] = e;
      }
      run += __popc(bal);
    }
    __syncthreads();
    for (int i = threadIdx.x; i < n; i += blockDim.x) {
      int q = segid[i];
      if (q_ax[q]) sx[i] = scr[i]; else sy[i] = scr[i];
      segid[i] = (unsigned short)(2 * q + (i - q_s0[q] >= q_k[q]));
    }
#if TREE_SUB_PIPE
    if (qa) {   // the step tables (prepare_segment's second wave, same values)
      const int sg = s + A.a.s0;                                   // global step
      const bool deg = (sg & 1) == 0 && (sg >> 1) < A.a.L;         // tree.py:285
      const double cut = along_y ? pc.y : pc.x;
      if (deg && pxa.x == pxb.x && pya.y == pyb.y) {
        const unsigned long long key = ((unsigned long long)(sg >> 1) << 40) |
                                       (unsigned long long)((A.a.seg << s) + j);
        atomicMin(&st->degenerate_key, key);
        atomicOr(&st->flags, ST_DEGENERATE);
      }
      if (k < nn && (along_y ? pn.y : pn.x) == cut) atomicOr(&st->flags, ST_EVAL_TIES);
      A.a.cut_tab[step_base(s) + j] = cut;
      A.a.axis_tab[step_base(s) + j] = along_y;
      Rect lo = r, hi = r;                                         // tree.py:218-222
      if (along_y) { lo.y1 = cut; hi.y0 = cut; } else { lo.x1 = cut; hi.x0 = cut; }
      A.a.rect_tab[step_base(s + 1) + 2 * j] = lo;
      A.a.rect_tab[step_base(s + 1) + 2 * j + 1] = hi;
      s_rect[2 * q] = lo;
      s_rect[2 * q + 1] = hi;
    }
#endif
    __syncthreads();
  }

  // leaves: members sorted by original index (canonical order)
  const int nleaf = 1 << (A.S - A.sb);
  const int* offL = A.a.off + off_base(A.S);
  int* sidx = reinterpret_cast<int*>(scr);
  for (int i = threadIdx.x; i < n; i += blockDim.x) sidx[i] = A.perm_x[sx[i].x];
  __syncthreads();
  if (A.in_smem_finalize) {
    for (int i = threadIdx.x; i < n; i += blockDim.x) {
      const int q = segid[i];
      const long long jl = j0 * nleaf + q;
      const int l0 = offL[jl] - g0, l1 = offL[jl + 1] - g0;
      const int me = sidx[i];
      int rank = 0;
      for (int t = l0; t < l1; ++t) rank += sidx[t] < me;
      // canonical position of local point `me`; the point data itself is
      // gathered afterwards by a full-occupancy kernel (k_gather_points)
      A.leaf_of[g0 + l0 + rank] = me;
    }
  } else {
    for (int i = threadIdx.x; i < n; i += blockDim.x)
      A.leaf_of[sidx[i]] = (int)(j0 * nleaf + segid[i]);
  }
}

// --------------------------------------------------------------------------
// fallback finalize / evaluation points: leaf ids then stable sort by leaf
__global__ void k_global_leaf_of(int S, const int* __restrict__ offS, const int2* X0,
                                 const int2* X1, const unsigned char* __restrict__ xpar,
                                 const int* __restrict__ perm_x, long long n, int* leaf_of) {
  pdl_enter();
  // used when every split ran globally: leaf = segment of the final step
  long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (i >= n) return;
  long long lo = 0, hi = (1ll << S);
  while (hi - lo > 1) {
    long long mid = (lo + hi) >> 1;
    if (offS[mid] <= i) lo = mid; else hi = mid;
  }
  const int2* X = xpar[lo] ? X1 : X0;
  leaf_of[perm_x[X[i].x]] = (int)lo;
}

__global__ void k_iota_perm(int* v, long long n) {
  pdl_enter();
  long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (i < n) v[i] = (int)i;
}

__global__ void k_descend(const double2* __restrict__ pts, long long m, int S,
                          const double* __restrict__ cut_tab,
                          const unsigned char* __restrict__ axis_tab, unsigned int* keys,
                          int* vals) {
  pdl_enter();
  long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (e >= m) return;
  const double2 z = pts[e];
  long long seg = 0;
  for (int s = 0; s < S; ++s) {
    const long long t = step_base(s) + seg;
    const double c = axis_tab[t] ? z.y : z.x;
    seg = 2 * seg + (c <= cut_tab[t] ? 0 : 1);     // tree.py:210 (coords <= cut)
  }
  keys[e] = (unsigned int)seg;
  vals[e] = (int)e;
}

__global__ void k_iota_keys(const int* __restrict__ leaf_of, long long n, unsigned int* keys,
                            int* vals) {
  pdl_enter();
  long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (i >= n) return;
  keys[i] = (unsigned int)leaf_of[i];
  vals[i] = (int)i;
}

__global__ void k_gather_points(const int* __restrict__ perm, long long m,
                                const double2* __restrict__ pts, const double* __restrict__ g,
                                double2* out_pos, double* out_g, int* out_perm,
                                long long out0, const int* __restrict__ orig) {
  pdl_enter();
  long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (i >= m) return;
  int e = perm[i];
  out_perm[out0 + i] = orig ? orig[e] : e;
  out_pos[out0 + i] = pts[e];
  if (g) out_g[out0 + i] = g[e];
}

// leaf offsets from leaf-sorted keys (handles empty leaves)
__global__ void k_leaf_offsets(const unsigned int* __restrict__ skeys, long long m, long long nleaf,
                               int* leaf_off) {
  pdl_enter();
  long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (i > m) return;
  long long prev = i == 0 ? -1 : (long long)skeys[i - 1];
  long long cur = i == m ? nleaf : (long long)skeys[i];
  for (long long b = prev + 1; b <= cur; ++b) leaf_off[b] = (int)i;
}

__global__ void k_leaf_offsets_identity(int* leaf_off, long long m) {
  pdl_enter();
  leaf_off[0] = 0;
  leaf_off[1] = (int)m;
}

// per-level box geometry from the rectangles of even steps (tree.py:312-314)
__global__ void k_level_geometry(int L, const Rect* __restrict__ rect_tab, double* cx, double* cy,
                                 double* hw, double* hh, double* r, int s0, long long seg) {
  pdl_enter();
  long long gid = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  const long long total = level_base(L + 1);
  if (gid >= total) return;
  int l = 0;
  while (level_base(l + 1) <= gid) ++l;
  const long long k = gid - level_base(l);
  // subtree builds own boxes k in [seg << t, (seg + 1) << t) of level l, t = 2l - s0
  const int t = 2 * l - s0;
  if (t < 0 || (k >> t) != seg) return;
  const Rect rc = rect_tab[step_base(t) + (k - (seg << t))];
  cx[gid] = (rc.x0 + rc.x1) / 2;
  cy[gid] = (rc.y0 + rc.y1) / 2;
  const double w = (rc.x1 - rc.x0) / 2, h = (rc.y1 - rc.y0) / 2;
  hw[gid] = w;
  hh[gid] = h;
  r[gid] = glibc_hypot(w, h);
}

inline unsigned nblk(long long n, int t) { return (unsigned)((n + t - 1) / t); }

template <class K, class V>
void radix_sort_pairs(DBuf& tmp, const K* kin, K* kout, const V* vin, V* vout, long long n,
                      int end_bit, cudaStream_t st) {
  size_t bytes = 0;
  FMM_CUDA(cub::DeviceRadixSort::SortPairs(nullptr, bytes, kin, kout, vin, vout, (int)n, 0,
                                           end_bit, st));
  tmp.reserve(bytes);
  FMM_CUDA(cub::DeviceRadixSort::SortPairs(tmp.p, bytes, kin, kout, vin, vout, (int)n, 0,
                                           end_bit, st));
}

int smem_need(long long nmax, int nseg) {
  return (int)((TREE_SUB_PIPE ? (long long)sizeof(Rect) * nseg : 0) + 3 * 8 * nmax +
               2 * ((nmax + 1) & ~1ll) + 18ll * nseg + 64);
}

}  // namespace

int plan_levels(int64_t n, int nd) {
  // Eq. (6), tree.py:86-94, clamped so that 4^L <= n (tree.py:186-192)
  double raw = 0.5 * std::log2(0.625 * (double)n / (double)nd);
  int lev = raw > 0 ? (int)std::ceil(raw) : 0;
  while (lev > 0 && (int64_t(1) << (2 * lev)) > n) --lev;
  return lev;
}

void plan_tree(TreePlan& P, int64_t n, int64_t m, int L, int s0) {
  if (P.n == n && P.m == m && P.L == L && P.s0 == s0) return;
  P.n = n; P.m = m; P.L = L; P.s0 = s0; P.S = 2 * L - s0;
  const int S = P.S;
  // choose the first step whose segments fit one subtree CTA in SMEM
  auto nmax_at = [&](int s) { return (n + (int64_t(1) << s) - 1) >> s; };
  int sb = S;
  bool fits_any = false;
  // the pipelined subtree step gives each segment of a step its own thread
  auto seg_ok = [&](int s) { return !TREE_SUB_PIPE || (1ll << (S - s)) <= SUB_THREADS; };
  for (int s = 0; s <= S; ++s) {
    if (seg_ok(s) && smem_need(nmax_at(s), 1 << (S - s)) <= SMEM_BUDGET) {
      sb = s;
      fits_any = true;
      break;
    }
  }
  if (!fits_any) {
    for (int s = 0; s <= S; ++s)
      if (seg_ok(s) && smem_need(nmax_at(s), 1 << (S - s)) <= 220 * 1024) {
        sb = s;
        fits_any = true;
        break;
      }
  }
  const int64_t leaf_max = nmax_at(S);
  P.global_leaf_finalize = !fits_any || leaf_max > LEAF_SMEM_MAX;
  if (!fits_any) sb = S;
  P.sb = sb;
  P.smem_bytes = fits_any ? smem_need(nmax_at(sb), 1 << (S - sb)) : 0;

  // data-independent offsets for all steps (host mirror for the tile tables)
  std::vector<std::vector<int64_t>> off(S + 1);
  off[0] = {0, n};
  for (int s = 0; s < S; ++s) {
    const auto& o = off[s];
    std::vector<int64_t> nx(2 * (o.size() - 1) + 1);
    nx[0] = 0;
    for (size_t j = 0; j + 1 < o.size(); ++j) {
      int64_t cnt = o[j + 1] - o[j], left = (cnt + 1) / 2;
      nx[2 * j + 1] = o[j] + left;
      nx[2 * j + 2] = o[j + 1];
    }
    off[s + 1] = std::move(nx);
  }
  std::vector<int> tseg, tstart;
  P.tile_base.assign(sb, 0);
  P.tile_count.assign(sb, 0);
  for (int s = 0; s < sb; ++s) {
    P.tile_base[s] = (int)tseg.size();
    for (size_t j = 0; j + 1 < off[s].size(); ++j) {
      for (int64_t b = off[s][j]; b < off[s][j + 1]; b += PART_TILE) {
        tseg.push_back((int)j);
        tstart.push_back((int)b);
      }
    }
    P.tile_count[s] = (int)tseg.size() - P.tile_base[s];
  }
  const int64_t off_entries = off_base(S + 1);
  P.d_off.reserve(sizeof(int) * off_entries);
  {
    std::vector<int> flat(off_entries);
    for (int s = 0; s <= S; ++s)
      for (size_t j = 0; j < off[s].size(); ++j) flat[off_base(s) + j] = (int)off[s][j];
    FMM_CUDA(cudaMemcpy(P.d_off.p, flat.data(), sizeof(int) * off_entries,
                        cudaMemcpyHostToDevice));
  }
  {
    // per-tile descriptors, first tile of every segment per step, flag bytes
    std::vector<int> desc(4 * tseg.size() + 4), st0;
    P.segt_base.assign(sb + 1, 0);
    for (int s = 0; s < sb; ++s) {
      P.segt_base[s] = (int)st0.size();
      const int tb = P.tile_base[s];
      int t = 0;
      for (size_t j = 0; j + 1 < off[s].size(); ++j) {
        st0.push_back(t);
        for (int64_t b = off[s][j]; b < off[s][j + 1]; b += PART_TILE, ++t) {
          desc[4 * (tb + t)] = (int)j;
          desc[4 * (tb + t) + 1] = (int)b;
          desc[4 * (tb + t) + 2] = (int)off[s][j];
          desc[4 * (tb + t) + 3] = (int)off[s][j + 1];
        }
      }
      st0.push_back(t);
    }
    P.segt_base[sb] = (int)st0.size();
    st0.push_back(0);
    P.d_tile_desc.reserve(sizeof(int) * desc.size());
    P.d_seg_tile0.reserve(sizeof(int) * st0.size());
    P.d_tile_flag.reserve(tseg.size() + 16);
    FMM_CUDA(cudaMemcpy(P.d_tile_desc.p, desc.data(), sizeof(int) * desc.size(),
                        cudaMemcpyHostToDevice));
    FMM_CUDA(cudaMemcpy(P.d_seg_tile0.p, st0.data(), sizeof(int) * st0.size(),
                        cudaMemcpyHostToDevice));
  }
  P.d_tile_seg.reserve(sizeof(int) * (tseg.size() + 1));
  P.d_tile_start.reserve(sizeof(int) * (tstart.size() + 1));
  if (!tseg.empty()) {
    FMM_CUDA(cudaMemcpy(P.d_tile_seg.p, tseg.data(), sizeof(int) * tseg.size(),
                        cudaMemcpyHostToDevice));
    FMM_CUDA(cudaMemcpy(P.d_tile_start.p, tstart.data(), sizeof(int) * tstart.size(),
                        cudaMemcpyHostToDevice));
  }
}

void run_tree(TreeState& T, TreePlan& P, DevStatus* dstat, cudaStream_t st) {
  const long long n = T.n, m = T.m;
  const TreeSpec& spec = T.spec;
  const int L = T.L, S = 2 * L - spec.s0, sb = P.sb;
  const double2* pos = T.pos_p;
  const double2* epos = T.aliased ? pos : T.epos_p;
  const long long nseg_total = step_base(S + 1);
  T.dup_checked = false;

  T.src_pos.reserve(sizeof(double2) * (spec.out0 + n));
  T.src_g.reserve(sizeof(double) * (spec.out0 + n));
  T.src_perm.reserve(sizeof(int) * (spec.out0 + n));
  T.eval_pos.reserve(sizeof(double2) * m);
  T.eval_perm.reserve(sizeof(int) * m);
  T.eval_leaf_off.reserve(sizeof(int) * ((1ll << S) + 1));
  T.rect_tab.reserve(sizeof(Rect) * nseg_total);
  T.cut_tab.reserve(sizeof(double) * (step_base(S) + 1));
  T.axis_tab.reserve(step_base(S) + 1);
  const long long nbox = level_base(L + 1);
  for (DBuf* b : {&T.box_cx, &T.box_cy, &T.box_hw, &T.box_hh, &T.box_r})
    b->reserve(sizeof(double) * nbox);
  T.bbox.reserve(sizeof(double) * (4 + 4 * 1024) + 64);
  const long long nmx = std::max(n, m);
  T.keys_in.reserve(sizeof(unsigned long long) * nmx);
  T.keys_out.reserve(sizeof(unsigned long long) * nmx);
  T.vals_in.reserve(sizeof(int) * nmx);
  T.vals_out.reserve(sizeof(int) * nmx);

  // strengths / evaluation points uploaded on the copy stream: wait before their
  // first use (the bounding box when evaluation points are separate)
  bool inputs_waited = false;
  auto wait_inputs = [&] {
    if (T.inputs_ready && !inputs_waited && !capture_cut(ACT_WAIT_INPUTS))
      FMM_CUDA(cudaStreamWaitEvent(st, T.inputs_ready, 0));
    inputs_waited = true;
  };
  if (!T.aliased) wait_inputs();
  // root rectangle: given (subtree of a distributed top split) or the tight bbox
  if (spec.root_given) {
    const Rect rr{spec.root[0], spec.root[1], spec.root[2], spec.root[3]};
    FMM_CUDA(cudaMemcpyAsync(T.rect_tab.p, &rr, sizeof(Rect), cudaMemcpyHostToDevice, st));
    FMM_CUDA(cudaStreamSynchronize(st));   // rr lives on this stack frame
  } else {
    double* bb = T.bbox.as<double>();
    unsigned int* counter = reinterpret_cast<unsigned int*>(bb + 4 + 4 * 1024);
    FMM_CUDA(cudaMemsetAsync(counter, 0, sizeof(unsigned int), st));
    unsigned blocks = (unsigned)std::min<long long>(1024, std::max<long long>(1, nblk(n + m, 256)));
    note_launch();
    launch(k_bbox, blocks, 256, 0, st, pos, n, epos, T.aliased ? 0 : m, T.rect_tab.as<Rect>(),
                                   counter, bb + 4);
  }

  if (S > 0) {
    // global ranks along x and y (ties by original index: stable radix sort)
    for (DBuf* b : {&T.perm_x, &T.perm_y, &T.rank_x, &T.rank_y}) b->reserve(sizeof(int) * n);
    for (DBuf* b : {&T.X0, &T.X1, &T.Y0, &T.Y1}) b->reserve(sizeof(int2) * n);
    const long long pmax = (1ll << std::max(sb, 1)) + 2;
    for (DBuf* b : {&T.xpar0, &T.xpar1, &T.ypar0, &T.ypar1}) b->reserve(pmax);
    // small N: the y tie pass scatters the split records itself (all arrays
    // L2-resident); large N: rank arrays + one gather pass (k_init_arrays),
    // whose random reads hit a 4-byte rank array instead of scattering 8-byte
    // records across a DRAM-sized copy
    const bool fuse_records = n <= TREE_FUSE_RECORDS_MAX;
    for (int axis = 0; axis < 2; ++axis) {
      int* perm = axis ? T.perm_y.as<int>() : T.perm_x.as<int>();
      if (T.exact_keys) {
        auto* kin = T.keys_in.as<unsigned long long>();
        auto* kout = T.keys_out.as<unsigned long long>();
        note_launch();
        launch(k_make_keys, nblk(n, 256), 256, 0, st, pos, n, axis, kin, T.vals_in.as<int>());
        radix_sort_pairs(T.cub_tmp, kin, kout, T.vals_in.as<int>(), perm, n, 64, st);
      } else {
        auto* kin = reinterpret_cast<unsigned*>(T.keys_in.p) + axis * n;   // 2n u32 fit
        auto* kout = reinterpret_cast<unsigned*>(T.keys_out.p);
        // key resolution ~16x finer than the mean point spacing: a radix pass less
        // for small N, equal-key runs stay short (k_fix_ties orders them exactly)
        int nb = 0;
        while ((1ll << nb) < n) ++nb;
        const int key_bits = std::min(32, std::max(16, (nb + TREE_KEY_EXTRA + 7) / 8 * 8));
        const bool fork = TREE_FORK_SORT && n >= TREE_FORK_MIN;
        if (axis == 0) {
          note_launch();
          launch(k_make_keys32, nblk(n, 256), 256, 0, st, pos, n, T.rect_tab.as<Rect>(), kin,
                 T.vals_in.as<int>(), 32 - key_bits);
          if (fork) {
            // the y-axis sort runs on the side stream while x sorts and fixes ties
            T.aux.ensure();
            FMM_CUDA(cudaEventRecord(T.aux.fork, st));
            FMM_CUDA(cudaStreamWaitEvent(T.aux.s, T.aux.fork, 0));
            radix_sort_pairs(T.cub_tmp2, kin + n, kout + n, T.vals_in.as<int>(),
                             T.perm_y.as<int>(), n, key_bits, T.aux.s);
            FMM_CUDA(cudaEventRecord(T.aux.join, T.aux.s));
          }
        }
        if (fork) {
          kout += axis * n;
          if (axis == 1) FMM_CUDA(cudaStreamWaitEvent(st, T.aux.join, 0));
        }
        if (!fork || axis == 0)
          radix_sort_pairs(T.cub_tmp, kin, kout, T.vals_in.as<int>(), perm, n, key_bits, st);
        note_launch();
        RankOut o{axis ? T.rank_y.as<int>() : T.rank_x.as<int>(), nullptr, nullptr, nullptr,
                  nullptr, nullptr};
        if (axis == 1 && fuse_records)
          o = RankOut{nullptr, T.rank_x.as<int>(), T.X0.as<int2>(), T.Y0.as<int2>(),
                      T.xpar0.as<unsigned char>(), T.ypar0.as<unsigned char>()};
        launch(k_fix_ties, nblk(n, 256), 256, 0, st, kout, perm, pos, axis, n, o, dstat);
        if (axis == 0) T.dup_checked = true;
        continue;
      }
      note_launch();
      launch(k_rank_scatter, nblk(n, 256), 256, 0, st, n, perm, axis ? T.rank_y.as<int>() : T.rank_x.as<int>());
    }
    if (T.exact_keys || !fuse_records) {
      note_launch();
      launch(k_init_arrays, nblk(n, 256), 256, 0, st, n, T.perm_x.as<int>(), T.perm_y.as<int>(),
             T.rank_x.as<int>(), T.rank_y.as<int>(), T.X0.as<int2>(), T.Y0.as<int2>(),
             T.xpar0.as<unsigned char>(), T.ypar0.as<unsigned char>());
    }
    StepArgs a{P.d_off.as<int>(), T.rect_tab.as<Rect>(), T.cut_tab.as<double>(),
               T.axis_tab.as<unsigned char>(), pos, T.perm_x.as<int>(), T.perm_y.as<int>(),
               L, spec.s0, spec.seg};
    unsigned char *xp = T.xpar0.as<unsigned char>(), *yp = T.ypar0.as<unsigned char>();
    unsigned char *xq = T.xpar1.as<unsigned char>(), *yq = T.ypar1.as<unsigned char>();
    int maxtiles = 1;
    for (int s = 0; s < sb; ++s) maxtiles = std::max(maxtiles, P.tile_count[s]);
    const int2 *X0 = T.X0.as<int2>(), *X1 = T.X1.as<int2>(), *Y0 = T.Y0.as<int2>(),
               *Y1 = T.Y1.as<int2>();
    // look-back state of the fused step kernel (grow-only, epoch-tagged)
    T.lb_epoch = 0;
    lb_advance(lb_base_prepare(T.lb_base, T.lb_base_ready, st), st);
    if (T.lb_tiles < maxtiles + 1) {
      T.lb_vals.reserve(sizeof(unsigned long long) * (maxtiles + 1));
      T.lb_ticket.reserve(sizeof(unsigned) * 4);
      FMM_CUDA(cudaMemsetAsync(T.lb_vals.p, 0, sizeof(unsigned long long) * (maxtiles + 1), st));
      FMM_CUDA(cudaMemsetAsync(T.lb_ticket.p, 0, sizeof(unsigned) * 4, st));
      T.lb_tiles = maxtiles + 1;
    }
    for (int s = 0; s < sb; ++s) {
      const int nt = P.tile_count[s];
      const int* tseg = P.d_tile_seg.as<int>() + P.tile_base[s];
      const int* tstart = P.d_tile_start.as<int>() + P.tile_base[s];
      ++T.lb_epoch;
      const LookbackPacked lbs{T.lb_vals.as<unsigned long long>(), T.lb_ticket.as<unsigned>(),
                               T.lb_epoch, T.lb_base.as<unsigned>()};
      note_launch();
      unsigned char* flags = P.d_tile_flag.as<unsigned char>();
      const PartDesc pd{P.d_tile_desc.as<int>() + 4ll * P.tile_base[s],
                        s > 0 ? flags + P.tile_base[s] : nullptr,
                        s + 1 < sb ? flags + P.tile_base[s + 1] : nullptr,
                        s + 1 < sb ? P.d_seg_tile0.as<int>() + P.segt_base[s + 1] : nullptr};
      launch(k_part_step, nt, PART_THREADS, 0, st, a, s, tseg, tstart, T.X0.as<int2>(),
                                               T.X1.as<int2>(), T.Y0.as<int2>(), T.Y1.as<int2>(),
                                               xp, yp, xq, yq, lbs, (unsigned)nt, dstat, pd);
      std::swap(xp, xq);
      std::swap(yp, yq);
    }
    T.leaf_of.reserve(sizeof(int) * std::max(n, m));
    wait_inputs();
    if (P.smem_bytes > 0) {
      SubArgs A{a, sb, S, X0, X1, Y0, Y1, xp, yp, T.perm_x.as<int>(), pos, T.g_p,
                T.src_pos.as<double2>(), T.src_g.as<double>(), T.src_perm.as<int>(),
                T.leaf_of.as<int>(), !P.global_leaf_finalize,
                (int)((n + (1ll << sb) - 1) >> sb), spec.out0, spec.orig};
      FMM_CUDA(cudaFuncSetAttribute(k_subtree, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                    P.smem_bytes));
      note_launch();
      launch(k_subtree, (unsigned)(1ll << sb), SUB_THREADS, P.smem_bytes, st, A, dstat);
      if (!P.global_leaf_finalize) {
        note_launch();
        launch(k_gather_points, nblk(n, 256), 256, 0, st, T.leaf_of.as<int>(), n, pos, T.g_p,
                                                      T.src_pos.as<double2>(),
                                                      T.src_g.as<double>(),
                                                      T.src_perm.as<int>(), spec.out0,
                                                      spec.orig);
      }
    } else {
      // every split ran as a global step: leaves are segments of the global copies
      note_launch();
      launch(k_global_leaf_of, nblk(n, 256), 256, 0, st, S, P.d_off.as<int>() + off_base(S), X0, X1,
                                                     xp, T.perm_x.as<int>(), n,
                                                     T.leaf_of.as<int>());
    }
    if (P.global_leaf_finalize) {
      auto* kin = reinterpret_cast<unsigned int*>(T.keys_in.p);
      auto* kout = reinterpret_cast<unsigned int*>(T.keys_out.p);
      note_launch();
      launch(k_iota_keys, nblk(n, 256), 256, 0, st, T.leaf_of.as<int>(), n, kin, T.vals_in.as<int>());
      radix_sort_pairs(T.cub_tmp, kin, kout, T.vals_in.as<int>(), T.vals_out.as<int>(), n, S, st);
      note_launch();
      launch(k_gather_points, nblk(n, 256), 256, 0, st, T.vals_out.as<int>(), n, pos, T.g_p,
                                                    T.src_pos.as<double2>(), T.src_g.as<double>(),
                                                    T.src_perm.as<int>(), spec.out0, spec.orig);
    }
    if (T.aliased && !T.eval_full) {
      // evaluation points = sources, same partition (ties re-run the full path)
      T.eleaf_t = nullptr;
      T.epos_t = T.src_pos.as<double2>();
      T.eperm_t = T.src_perm.as<int>();
      T.eoff_t = P.d_off.as<int>() + off_base(S);
    } else {
      // evaluation points: descend the cut table, stable sort by leaf
      auto* kin = reinterpret_cast<unsigned int*>(T.keys_in.p);
      auto* kout = reinterpret_cast<unsigned int*>(T.keys_out.p);
      note_launch();
      launch(k_descend, nblk(m, 256), 256, 0, st, epos, m, S, T.cut_tab.as<double>(),
                                              T.axis_tab.as<unsigned char>(), kin,
                                              T.vals_in.as<int>());
      radix_sort_pairs(T.cub_tmp, kin, kout, T.vals_in.as<int>(), T.vals_out.as<int>(), m, S, st);
      note_launch();
      launch(k_gather_points, nblk(m, 256), 256, 0, st, T.vals_out.as<int>(), m, epos, nullptr,
                                                    T.eval_pos.as<double2>(), nullptr,
                                                    T.eval_perm.as<int>(), 0ll, spec.eorig);
      note_launch();
      launch(k_leaf_offsets, nblk(m + 1, 256), 256, 0, st, kout, m, 1ll << S, T.eval_leaf_off.as<int>());
      T.epos_t = T.eval_pos.as<double2>();
      T.eperm_t = T.eval_perm.as<int>();
      T.eoff_t = T.eval_leaf_off.as<int>();
      T.eleaf_t = kout;
    }
  } else {
    // L == 0: a single box, identity permutations (tree.py:253-254)
    wait_inputs();
    note_launch();
    launch(k_iota_perm, nblk(n, 256), 256, 0, st, T.vals_in.as<int>(), n);
    note_launch();
    launch(k_gather_points, nblk(n, 256), 256, 0, st, T.vals_in.as<int>(), n, pos, T.g_p,
                                                  T.src_pos.as<double2>(), T.src_g.as<double>(),
                                                  T.src_perm.as<int>(), spec.out0, spec.orig);
    if (T.aliased) {
      T.epos_t = T.src_pos.as<double2>();
      T.eperm_t = T.src_perm.as<int>();
    } else {
      note_launch();
      launch(k_iota_perm, nblk(m, 256), 256, 0, st, T.vals_in.as<int>(), m);
      note_launch();
      launch(k_gather_points, nblk(m, 256), 256, 0, st, T.vals_in.as<int>(), m, epos, nullptr,
                                                    T.eval_pos.as<double2>(), nullptr,
                                                    T.eval_perm.as<int>(), 0ll, nullptr);
      T.epos_t = T.eval_pos.as<double2>();
      T.eperm_t = T.eval_perm.as<int>();
    }
    note_launch();
    launch(k_leaf_offsets_identity, 1, 1, 0, st, T.eval_leaf_off.as<int>(), m);
    T.eoff_t = T.eval_leaf_off.as<int>();
  }
  note_launch();
  launch(k_level_geometry, nblk(nbox, 256), 256, 0, st, L, T.rect_tab.as<Rect>(), T.box_cx.as<double>(),
                                                    T.box_cy.as<double>(), T.box_hw.as<double>(),
                                                    T.box_hh.as<double>(), T.box_r.as<double>(),
                                                    spec.s0, spec.seg);
}

}  // namespace fmm
