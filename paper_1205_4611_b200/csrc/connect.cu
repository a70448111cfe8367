// Connectivity ("connect" phase): θ-criterion interaction lists, bit-exact.
//
// Reference: connectivity.py:47-68 (classify_level), :71-96
// (reclassify_finest), :99-114 (build_connectivity); predicates
// geometry.py:27-54 restated bit-exactly in common.cuh.
//
// One warp per target box.  Candidates of box b are the children of the
// boxes strongly coupled to its parent, generated in ascending order, so the
// ballot/popc compaction below writes every list already sorted ascending
// (the property connectivity.py:10-12 promises).  One launch per level:
// predicates -> decoupled look-back offsets -> fill; the weak lists of all
// levels form one global CSR (global box ids),
// which is also the pair list the single M2L launch consumes.  No host sync:
// list buffers are sized from capacities kept in the context, and a fill that
// would overflow only raises ST_OVERFLOW (the host then regrows and reruns).
#include <cstdlib>

#include "engine.h"
#include "lookback.cuh"

namespace fmm {

namespace {


struct LevelGeo {
  const double* cx;
  const double* cy;
  const double* r;
};

constexpr int CL_WARPS = 8;     // warps per CTA
constexpr int CL_PPW = 1;       // classify: parents (4 sibling targets each) per warp
constexpr int CL_TPW = 8;       // reclassify: finest targets per warp
constexpr int CL_MAXM = 16;     // ballot masks cached per target (512 candidates)
#ifndef CL_GRID_CAP
#define CL_GRID_CAP (8u * 148u)   // predicate / fill grids (warp per parent, grid-stride)
#endif
#ifndef CL_SPLIT_MIN
#define CL_SPLIT_MIN 1024       // parents per level from which the split classify runs
#endif
#ifndef CL_HEAVY_MIN
#define CL_HEAVY_MIN 64         // strong-list length from which a parent counts as heavy
#endif
#ifndef CL_HEAVY_RATIO
#define CL_HEAVY_RATIO 4        // ... and only if it exceeds this multiple of the mean
#endif
// load-balanced chunked predicate/fill kernels unless FMM2D_CL_CHUNKED=0
bool cl_chunked() {
  static bool v = [] {
    const char* e = getenv("FMM2D_CL_CHUNKED");
    return !(e && e[0] == '0');
  }();
  return v;
}
// split classify (predicates, then look-back + fill) unless FMM2D_CL_SPLIT=0
bool cl_split() {
  static bool v = [] {
    const char* e = getenv("FMM2D_CL_SPLIT");
    return !(e && e[0] == '0');
  }();
  return v;
}

// One level of classify_level (connectivity.py:47-68) in ONE pass.  A warp
// walks CL_PPW parent boxes; for each it evaluates the four children against
// the children of the parent's strong list (the siblings share that candidate
// set, so each candidate's geometry is loaded once for four predicates); the
// far/near ballot masks stay in SMEM; one decoupled look-back per CTA
// (CL_WARPS * CL_PPW parents) gives every target its offsets in the global
// weak CSR and in the level's strong CSR; the lists are then written
// compacted, ascending.  Children outside the owned window [tb, te) get empty
// lists (distributed ranks).  A CTA that finds the lists already overflowed
// publishes zero counts (never stalls its successors) and writes nothing.
__global__ void __launch_bounds__(CL_WARPS * 32)
k_classify(int l, LevelGeo geo, double theta, const int* __restrict__ ps_off,
           const int* __restrict__ ps_idx, int* so, int* sidx, long long scap, int* woff,
           int* widx, int* wtgt, long long wcap, LookbackState lbs, unsigned ntiles,
           long long P0, long long P1, long long tb, long long te, int* maxs, DevStatus* st) {
  pdl_enter();
  __shared__ unsigned s_mask[CL_WARPS][CL_PPW][4][CL_MAXM];
  __shared__ int s_cnt[CL_WARPS][CL_PPW][4][2];
  __shared__ long long s_excl[2];
  __shared__ unsigned s_tile;
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  if (threadIdx.x == 0) s_tile = lb_ticket(lbs, ntiles);
  __syncthreads();
  const unsigned tile = s_tile;
  const bool dead = lists_overflowed(st);
  const long long lb = level_base(l);
  const long long Pw = P0 + ((long long)tile * CL_WARPS + w) * CL_PPW;   // this warp's first parent
  auto cand_of = [&](int a0, int c) { return 4 * ps_idx[a0 + (c >> 2)] + (c & 3); };
  // phase 1: predicates -> masks + counts
  for (int u = 0; u < CL_PPW; ++u) {
    const long long P = Pw + u;
    const bool live = P < P1 && !dead;
    int a0 = 0, ncand = 0;
    if (live) {
      a0 = ps_off[P];
      ncand = 4 * (ps_off[P + 1] - a0);
    }
    double rt[4], xt[4], yt[4];
    bool own[4];
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      own[j] = live && 4 * P + j >= tb && 4 * P + j < te;
      const long long gb = lb + 4 * (live ? P : 0) + j;
      rt[j] = geo.r[gb];
      xt[j] = geo.cx[gb];
      yt[j] = geo.cy[gb];
    }
    int nw[4] = {0, 0, 0, 0}, ns[4] = {0, 0, 0, 0};
    for (int c0 = 0; c0 < ncand; c0 += 32) {
      const int c = c0 + lane;
      const bool valid = c < ncand;
      const long long gc = lb + (valid ? cand_of(a0, c) : 0);
      const double xc = geo.cx[gc], yc = geo.cy[gc], rc = geo.r[gc];
      const unsigned vm = __ballot_sync(0xffffffffu, valid);
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        if (!own[j]) continue;                                   // warp-uniform
        // d = |c_target - c_source| (geometry.py:40), then the θ-test (:41)
        const bool far =
            valid && well_separated_dz(rt[j], rc, xt[j] - xc, yt[j] - yc, theta);
        const unsigned m = __ballot_sync(0xffffffffu, far);
        if (lane == 0 && (c0 >> 5) < CL_MAXM) s_mask[w][u][j][c0 >> 5] = m;
        nw[j] += __popc(m);
        ns[j] += __popc(vm & ~m);
      }
    }
    if (lane == 0) {
      int mx = 0;
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        s_cnt[w][u][j][0] = nw[j];
        s_cnt[w][u][j][1] = ns[j];
        mx = max(mx, ns[j]);
      }
      if (mx) atomicMax(maxs, mx);      // longest strong list of the level (cl_heavy)
    }
  }
  __syncthreads();
  if (w == 0) {
    long long agg[2] = {0, 0}, excl[2];
    for (int q = 0; q < CL_WARPS * CL_PPW * 4; ++q) {
      agg[0] += (&s_cnt[0][0][0][0])[2 * q];
      agg[1] += (&s_cnt[0][0][0][0])[2 * q + 1];
    }
    lb_prefix<2>(lbs, tile, agg, excl);
    if (lane == 0) {
      s_excl[0] = excl[0];
      s_excl[1] = excl[1];
    }
  }
  __syncthreads();
  // out[0] may alias the base; it is rewritten with the same value, so racing reads agree
  const long long wbase0 = woff[lb];
  long long wb = wbase0 + s_excl[0], sb = s_excl[1];
  for (int q = 0; q < w; ++q)
    for (int u = 0; u < CL_PPW; ++u)
      for (int j = 0; j < 4; ++j) {
        wb += s_cnt[q][u][j][0];
        sb += s_cnt[q][u][j][1];
      }
  if (tile == ntiles - 1 && w == CL_WARPS - 1 && lane == 0) {   // totals: end of this level
    long long wt = wb, stt = sb;
    for (int u = 0; u < CL_PPW; ++u)
      for (int j = 0; j < 4; ++j) {
        wt += s_cnt[w][u][j][0];
        stt += s_cnt[w][u][j][1];
      }
    so[4 * P1] = (int)stt;
    woff[lb + 4 * P1] = (int)wt;
    woff[level_base(l + 1)] = (int)wt;     // next level's base (same slot when P1 = 4^(l-1))
  }
  // phase 2: offsets and compacted lists
  const unsigned below = (1u << lane) - 1u;
  for (int u = 0; u < CL_PPW; ++u) {
    const long long P = Pw + u;
    if (P >= P1) break;
    long long wpos[4], spos[4];
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      wpos[j] = wb;
      spos[j] = sb;
      wb += s_cnt[w][u][j][0];
      sb += s_cnt[w][u][j][1];
    }
    if (lane == 0) {
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        so[4 * P + j] = (int)spos[j];
        woff[lb + 4 * P + j] = (int)wpos[j];
      }
    }
    if (dead) continue;
    if (wb > wcap || sb > scap) {
      if (lane == 0) {
        atomicOr(&st->flags, ST_OVERFLOW);
        atomicOr(&st->overflow_where, 1);
      }
      continue;
    }
    const int a0 = ps_off[P];
    const int ncand = 4 * (ps_off[P + 1] - a0);
    bool own[4];
#pragma unroll
    for (int j = 0; j < 4; ++j) own[j] = 4 * P + j >= tb && 4 * P + j < te;
    for (int c0 = 0; c0 < ncand; c0 += 32) {
      const int c = c0 + lane;
      const bool valid = c < ncand;
      const int cand = valid ? cand_of(a0, c) : 0;
      const unsigned vm = __ballot_sync(0xffffffffu, valid);
      double xc = 0.0, yc = 0.0, rc = 0.0;
      if ((c0 >> 5) >= CL_MAXM) {
        const long long gc = lb + cand;
        xc = geo.cx[gc];
        yc = geo.cy[gc];
        rc = geo.r[gc];
      }
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        if (!own[j]) continue;
        unsigned m;
        if ((c0 >> 5) < CL_MAXM) {
          m = s_mask[w][u][j][c0 >> 5];
        } else {
          const long long gb = lb + 4 * P + j;
          const bool far = valid && well_separated_dz(geo.r[gb], rc, geo.cx[gb] - xc,
                                                      geo.cy[gb] - yc, theta);
          m = __ballot_sync(0xffffffffu, far);
        }
        const unsigned sm = vm & ~m;
        if ((m >> lane) & 1u) {
          const long long o = wpos[j] + __popc(m & below);
          widx[o] = (int)(lb + cand);
          wtgt[o] = (int)(lb + 4 * P + j);
        }
        if ((sm >> lane) & 1u) sidx[spos[j] + __popc(sm & below)] = cand;
        wpos[j] += __popc(m);
        spos[j] += __popc(sm);
      }
    }
  }
}

// Split form of one classify_level (default): the predicate pass and the
// list fill are separate launches, so the look-back that places every
// target's lists runs on counts that are already known.  In the one-pass
// kernel above a tile can only publish its count after its own predicates,
// and on clustered inputs (long, uneven candidate lists) a slow tile stalls
// every later tile in the look-back; here each fill tile publishes at once.
//
// k_classify_pred: one warp per parent (grid-stride), the four siblings'
// far masks for each 32-candidate chunk go to global planes (word base of
// parent P: (P - P0) + 4 * (ps_off[P] - ps_off[P0]) / 32, disjoint because
// a parent needs at most 1 + floor(4 n_P / 32) words), counts to cnt[].
__device__ __forceinline__ long long cl_wbase(const int* ps_off, long long P, long long P0) {
  return (P - P0) + (4ll * (ps_off[P] - ps_off[P0])) / 32;
}

__device__ __forceinline__ void classify_pred_parents(
    int l, LevelGeo geo, double theta, const int* __restrict__ ps_off,
    const int* __restrict__ ps_idx, long long P0, long long P1, long long tb, long long te,
    int2* cnt, unsigned* masks, long long mplane, DevStatus* st) {
  const int lane = threadIdx.x & 31;
  const long long lb = level_base(l);
  const bool dead = lists_overflowed(st);
  const long long nwarps = ((long long)gridDim.x * blockDim.x) >> 5;
  for (long long P = P0 + ((blockIdx.x * (long long)blockDim.x + threadIdx.x) >> 5); P < P1;
       P += nwarps) {
    const int a0 = ps_off[P];
    const int ncand = dead ? 0 : 4 * (ps_off[P + 1] - a0);
    const long long wb = cl_wbase(ps_off, P, P0);
    double rt[4], xt[4], yt[4];
    bool own[4];
    unsigned ownm = 0;
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      own[j] = 4 * P + j >= tb && 4 * P + j < te;
      ownm |= (unsigned)own[j] << j;
      const long long gb = lb + 4 * P + j;
      rt[j] = geo.r[gb];
      xt[j] = geo.cx[gb];
      yt[j] = geo.cy[gb];
    }
    int nw[4] = {0, 0, 0, 0}, ns[4] = {0, 0, 0, 0};
    for (int c0 = 0; c0 < ncand; c0 += 32) {
      const int c = c0 + lane;
      const bool valid = c < ncand;
      const long long gc = lb + (valid ? 4 * ps_idx[a0 + (c >> 2)] + (c & 3) : 0);
      const double xc = geo.cx[gc], yc = geo.cy[gc], rc = geo.r[gc];
      const unsigned vm = __ballot_sync(0xffffffffu, valid);
      unsigned mk = 0;
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        if (!own[j]) continue;                                   // warp-uniform
        const bool far =
            valid && well_separated_dz(rt[j], rc, xt[j] - xc, yt[j] - yc, theta);
        const unsigned m = __ballot_sync(0xffffffffu, far);
        if (lane == j) mk = m;
        nw[j] += __popc(m);
        ns[j] += __popc(vm & ~m);
      }
      if (lane < 4 && ((ownm >> lane) & 1)) masks[lane * mplane + wb + (c0 >> 5)] = mk;
    }
    if (lane < 4) {
      int w = 0, s = 0;
#pragma unroll
      for (int j = 0; j < 4; ++j)
        if (j == lane) { w = nw[j]; s = ns[j]; }
      cnt[4 * (P - P0) + lane] = make_int2(w, s);     // zero for targets not owned
    }
  }
}

// Load-balanced split classify (default for the large levels).  The unit of
// work is a 32-candidate CHUNK of one parent's candidate list (chunk ids are
// the mask-word ids cl_wbase above: parent P owns ids [wbase(P), wbase(P+1))
// and uses the first ceil(4 n_P / 32)), and every warp takes a contiguous
// range of chunk ids.  A parent with thousands of candidates (clustered
// inputs: weak lists up to 2894) is then spread over many warps instead of
// serialising one warp, which bounded the old per-parent kernels' tail.
// Counts are integer atomics per target (exact, order independent); the fill
// recovers each chunk's in-list position from the popcounts of the parent's
// earlier mask words.
__device__ __forceinline__ long long cl_chunks_total(const int* ps_off, long long P0,
                                                     long long P1) {
  return cl_wbase(ps_off, P1, P0);
}
// the parent owning chunk id c: largest P in [P0, P1) with wbase(P) <= c
// (whole warp, 32-ary search)
__device__ __forceinline__ long long cl_parent_of(const int* ps_off, long long P0, long long P1,
                                                  long long c) {
  const int lane = threadIdx.x & 31;
  long long lo = P0, hi = P1;
  while (hi - lo > 1) {
    const long long step = (hi - lo + 31) / 32;
    const long long probe = lo + (long long)lane * step;
    const bool ok = probe < hi && cl_wbase(ps_off, probe, P0) <= c;
    const unsigned b = __ballot_sync(0xffffffffu, ok);
    const int last = 31 - __clz(b);                 // lane 0 (probe = lo) is always ok
    lo = lo + (long long)last * step;
    hi = min(hi, lo + step);
  }
  return lo;
}

__device__ __forceinline__ void classify_pred_chunks(
    int l, LevelGeo geo, double theta, const int* __restrict__ ps_off,
    const int* __restrict__ ps_idx, long long P0, long long P1, long long tb, long long te,
    int2* cnt, unsigned* masks, long long mplane, DevStatus* st) {
  if (lists_overflowed(st)) return;
  const int lane = threadIdx.x & 31;
  const long long lb = level_base(l);
  const long long nwarps = ((long long)gridDim.x * blockDim.x) >> 5;
  const long long wid = (blockIdx.x * (long long)blockDim.x + threadIdx.x) >> 5;
  const long long C = cl_chunks_total(ps_off, P0, P1);
  const long long per = (C + nwarps - 1) / nwarps;
  const long long c_begin = wid * per, c_end = min(C, c_begin + per);
  if (c_begin >= c_end) return;
  long long P = cl_parent_of(ps_off, P0, P1, c_begin);
  long long wb = cl_wbase(ps_off, P, P0), wnext = cl_wbase(ps_off, P + 1, P0);
  int a0 = ps_off[P], ncand = 4 * (ps_off[P + 1] - a0);
  double rt[4], xt[4], yt[4];
  bool own[4];
  auto load_targets = [&]() {
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      own[j] = 4 * P + j >= tb && 4 * P + j < te;
      const long long gb = lb + 4 * P + j;
      rt[j] = geo.r[gb];
      xt[j] = geo.cx[gb];
      yt[j] = geo.cy[gb];
    }
  };
  load_targets();
  int nw[4] = {0, 0, 0, 0}, ns[4] = {0, 0, 0, 0};
  auto flush = [&]() {
    if (lane < 4) {
      int w = 0, s2 = 0;
#pragma unroll
      for (int j = 0; j < 4; ++j)
        if (j == lane) { w = nw[j]; s2 = ns[j]; }
      if (w) atomicAdd(&cnt[4 * (P - P0) + lane].x, w);
      if (s2) atomicAdd(&cnt[4 * (P - P0) + lane].y, s2);
    }
#pragma unroll
    for (int j = 0; j < 4; ++j) nw[j] = ns[j] = 0;
  };
  for (long long c = c_begin; c < c_end; ++c) {
    if (c >= wnext) {                       // next parent(s): chunk ids are monotone in P
      flush();
      do {
        ++P;
        wb = wnext;
        wnext = cl_wbase(ps_off, P + 1, P0);
      } while (c >= wnext);
      a0 = ps_off[P];
      ncand = 4 * (ps_off[P + 1] - a0);
      load_targets();
    }
    const int c0 = 32 * (int)(c - wb);
    if (c0 >= ncand) continue;              // unused id of this parent
    const int cc = c0 + lane;
    const bool valid = cc < ncand;
    const long long gc = lb + (valid ? 4 * ps_idx[a0 + (cc >> 2)] + (cc & 3) : 0);
    const double xc = geo.cx[gc], yc = geo.cy[gc], rc = geo.r[gc];
    const unsigned vm = __ballot_sync(0xffffffffu, valid);
    unsigned mk = 0;
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      if (!own[j]) continue;                // warp-uniform
      const bool far = valid && well_separated_dz(rt[j], rc, xt[j] - xc, yt[j] - yc, theta);
      const unsigned m = __ballot_sync(0xffffffffu, far);
      if (lane == j) mk = m;
      nw[j] += __popc(m);
      ns[j] += __popc(vm & ~m);
    }
    if (lane < 4 && own[lane & 3]) masks[lane * mplane + c] = mk;
  }
  flush();
}

__device__ __forceinline__ void classify_fill_chunks(
    int l, const int* __restrict__ ps_off, const int* __restrict__ ps_idx,
    const int* __restrict__ so, int* sidx, long long scap, const int* __restrict__ woff,
    int* widx, int* wtgt, long long wcap, long long P0, long long P1, long long tb, long long te,
    const unsigned* __restrict__ masks, long long mplane, DevStatus* st) {
  if (lists_overflowed(st)) return;
  const int lane = threadIdx.x & 31;
  const long long lb = level_base(l);
  const unsigned below = (1u << lane) - 1u;
  if (woff[lb + 4 * P1] > wcap || so[4 * P1] > scap) {   // level totals past capacity
    if (blockIdx.x == 0 && threadIdx.x == 0) {
      atomicOr(&st->flags, ST_OVERFLOW);
      atomicOr(&st->overflow_where, 1);
    }
    return;
  }
  const long long nwarps = ((long long)gridDim.x * blockDim.x) >> 5;
  const long long wid = (blockIdx.x * (long long)blockDim.x + threadIdx.x) >> 5;
  const long long C = cl_chunks_total(ps_off, P0, P1);
  const long long per = (C + nwarps - 1) / nwarps;
  const long long c_begin = wid * per, c_end = min(C, c_begin + per);
  if (c_begin >= c_end) return;
  long long P = cl_parent_of(ps_off, P0, P1, c_begin);
  long long wb = 0, wnext = cl_wbase(ps_off, P, P0);
  int a0 = 0, ncand = 0;
  bool own[4] = {false, false, false, false};
  long long wpos[4], spos[4];
  bool first = true;
  for (long long c = c_begin; c < c_end; ++c) {
    if (c >= wnext || first) {              // (re)enter a parent: list bases + earlier chunks
      if (!first) ++P;
      while (c >= cl_wbase(ps_off, P + 1, P0)) ++P;
      wb = cl_wbase(ps_off, P, P0);
      wnext = cl_wbase(ps_off, P + 1, P0);
      a0 = ps_off[P];
      ncand = 4 * (ps_off[P + 1] - a0);
      const int wl = lane < 4 ? woff[lb + 4 * P + lane] : 0;
      const int sl = lane < 4 ? so[4 * P + lane] : 0;
      // far entries of the parent's chunks before c (warp-parallel popcounts)
      const long long kc = c - wb;
      int far[4] = {0, 0, 0, 0};
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        own[j] = 4 * P + j >= tb && 4 * P + j < te;
        if (!own[j]) continue;
        int f = 0;
        for (long long k = lane; k < kc; k += 32) f += __popc(masks[j * mplane + wb + k]);
#pragma unroll
        for (int d = 16; d; d >>= 1) f += __shfl_xor_sync(0xffffffffu, f, d);
        far[j] = f;
      }
      const int before = (int)min(32 * kc, (long long)ncand);   // candidates before chunk c
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        wpos[j] = __shfl_sync(0xffffffffu, wl, j) + far[j];
        spos[j] = __shfl_sync(0xffffffffu, sl, j) + (before - far[j]);
      }
      first = false;
    }
    const int c0 = 32 * (int)(c - wb);
    if (c0 >= ncand) continue;
    const int cc = c0 + lane;
    const bool valid = cc < ncand;
    const int cand = valid ? 4 * ps_idx[a0 + (cc >> 2)] + (cc & 3) : 0;
    const unsigned vm = __ballot_sync(0xffffffffu, valid);
    const unsigned mine = lane < 4 && own[lane & 3] ? masks[lane * mplane + c] : 0u;
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      if (!own[j]) continue;
      const unsigned m = __shfl_sync(0xffffffffu, mine, j);
      const unsigned sm = vm & ~m;
      if ((m >> lane) & 1u) {
        const long long q = wpos[j] + __popc(m & below);
        widx[q] = (int)(lb + cand);
        wtgt[q] = (int)(lb + 4 * P + j);
      }
      if ((sm >> lane) & 1u) sidx[spos[j] + __popc(sm & below)] = cand;
      wpos[j] += __popc(m);
      spos[j] += __popc(sm);
    }
  }
}

// Exclusive scan of NC per-entry counters (entry stride CS ints) into the
// CSR offset arrays out[k][0..n] (+ *base for counter 0; the total also to
// *tot_extra).  Large tiles (SCAN_TILE entries) keep the look-back chain short;
// the counts are already known, so every tile publishes at once.
constexpr int SCAN_THREADS = 256, SCAN_ITEMS = 8, SCAN_TILE = SCAN_THREADS * SCAN_ITEMS;
struct ScanOut {
  int* out[3];
  const int* base;          // added to counter 0 (null: 0)
  int* tot_extra;           // also receives counter 0's total (null: none)
};
template <int NC, int CS>
__global__ void __launch_bounds__(SCAN_THREADS)
k_scan_counts(const int* cnt, long long n, ScanOut o, LookbackState lbs,
              unsigned ntiles, int* maxs, DevStatus* st) {
  pdl_enter();
  __shared__ long long s_w[SCAN_THREADS / 32][NC];
  __shared__ long long s_excl[NC];
  __shared__ unsigned s_tile;
  if (threadIdx.x == 0) s_tile = lb_ticket(lbs, ntiles);
  __syncthreads();
  const unsigned tile = s_tile;
  const bool dead = lists_overflowed(st);
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const long long i0 = (long long)tile * SCAN_TILE + threadIdx.x * SCAN_ITEMS;
  int v[SCAN_ITEMS][NC];
  long long tsum[NC];
#pragma unroll
  for (int k = 0; k < NC; ++k) tsum[k] = 0;
#pragma unroll
  for (int q = 0; q < SCAN_ITEMS; ++q)
#pragma unroll
    for (int k = 0; k < NC; ++k) {
      v[q][k] = (i0 + q < n && !dead) ? cnt[(i0 + q) * CS + k] : 0;
      tsum[k] += v[q][k];
    }

  if (maxs && NC > 1) {                 // longest strong list (counter 1), for cl_heavy
    int mx = 0;
#pragma unroll
    for (int q = 0; q < SCAN_ITEMS; ++q) mx = max(mx, v[q][NC > 1 ? 1 : 0]);
#pragma unroll
    for (int d = 16; d; d >>= 1) mx = max(mx, __shfl_xor_sync(0xffffffffu, mx, d));
    if (lane == 0 && mx) atomicMax(maxs, mx);
  }
  long long incl[NC];
#pragma unroll
  for (int k = 0; k < NC; ++k) {
    incl[k] = tsum[k];
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
      const long long t = __shfl_up_sync(0xffffffffu, incl[k], d);
      if (lane >= d) incl[k] += t;
    }
    if (lane == 31) s_w[w][k] = incl[k];
  }
  __syncthreads();
  if (w == 0) {
    long long agg[NC], excl[NC];
#pragma unroll
    for (int k = 0; k < NC; ++k) {
      agg[k] = 0;
      for (int q = 0; q < SCAN_THREADS / 32; ++q) agg[k] += s_w[q][k];
    }
    lb_prefix<NC>(lbs, tile, agg, excl);
    if (lane == 0) {
      const long long b0 = o.base ? *o.base : 0;
#pragma unroll
      for (int k = 0; k < NC; ++k) s_excl[k] = excl[k] + (k == 0 ? b0 : 0);
      if (tile == ntiles - 1) {
#pragma unroll
        for (int k = 0; k < NC; ++k) o.out[k][n] = (int)(s_excl[k] + agg[k]);
        if (o.tot_extra) *o.tot_extra = (int)(s_excl[0] + agg[0]);
      }
    }
  }
  __syncthreads();
#pragma unroll
  for (int k = 0; k < NC; ++k) {
    long long run = s_excl[k] + incl[k] - tsum[k];
    for (int q = 0; q < w; ++q) run += s_w[q][k];
#pragma unroll
    for (int q = 0; q < SCAN_ITEMS; ++q) {
      if (i0 + q < n) o.out[k][i0 + q] = (int)run;
      run += v[q][k];
    }
  }
}

// k_classify_fill: one warp per parent (grid-stride, no look-back): the
// offsets come from the scan, the compacted lists from the stored masks
// (ascending candidate order, as before).
__device__ __forceinline__ void classify_fill_parents(
    int l, const int* __restrict__ ps_off, const int* __restrict__ ps_idx,
    const int* __restrict__ so, int* sidx, long long scap, const int* __restrict__ woff,
    int* widx, int* wtgt, long long wcap, long long P0, long long P1, long long tb, long long te,
    const unsigned* __restrict__ masks, long long mplane, DevStatus* st) {
  if (lists_overflowed(st)) return;
  const int lane = threadIdx.x & 31;
  const long long lb = level_base(l);
  const unsigned below = (1u << lane) - 1u;
  if (woff[lb + 4 * P1] > wcap || so[4 * P1] > scap) {   // level totals past capacity
    if (blockIdx.x == 0 && threadIdx.x == 0) {
      atomicOr(&st->flags, ST_OVERFLOW);
      atomicOr(&st->overflow_where, 1);
    }
    return;
  }
  const long long nwarps = ((long long)gridDim.x * blockDim.x) >> 5;
  for (long long P = P0 + ((blockIdx.x * (long long)blockDim.x + threadIdx.x) >> 5); P < P1;
       P += nwarps) {
    long long wpos[4], spos[4];
    const int wl = lane < 4 ? woff[lb + 4 * P + lane] : 0;
    const int sl = lane < 4 ? so[4 * P + lane] : 0;
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      wpos[j] = __shfl_sync(0xffffffffu, wl, j);
      spos[j] = __shfl_sync(0xffffffffu, sl, j);
    }
    const int a0 = ps_off[P];
    const int ncand = 4 * (ps_off[P + 1] - a0);
    const long long mw = cl_wbase(ps_off, P, P0);
    bool own[4];
    unsigned ownm = 0;
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      own[j] = 4 * P + j >= tb && 4 * P + j < te;
      ownm |= (unsigned)own[j] << j;
    }
    for (int c0 = 0; c0 < ncand; c0 += 32) {
      const int c = c0 + lane;
      const bool valid = c < ncand;
      const int cand = valid ? 4 * ps_idx[a0 + (c >> 2)] + (c & 3) : 0;
      const unsigned vm = __ballot_sync(0xffffffffu, valid);
      const unsigned mine =
          lane < 4 && ((ownm >> lane) & 1) ? masks[lane * mplane + mw + (c0 >> 5)] : 0u;
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        if (!own[j]) continue;
        const unsigned m = __shfl_sync(0xffffffffu, mine, j);
        const unsigned sm = vm & ~m;
        if ((m >> lane) & 1u) {
          const long long q = wpos[j] + __popc(m & below);
          widx[q] = (int)(lb + cand);
          wtgt[q] = (int)(lb + 4 * P + j);
        }
        if ((sm >> lane) & 1u) sidx[spos[j] + __popc(sm & below)] = cand;
        wpos[j] += __popc(m);
        spos[j] += __popc(sm);
      }
    }
  }
}

// Which body runs a split level: the chunked (load-balanced) one when some
// parent's strong list is far longer than the mean -- clustered inputs -- and
// the warp-per-parent one otherwise (fewer dependent loads per chunk: faster
// on uniform inputs).  maxs = the longest strong list among the parents
// (recorded by the previous level's count pass); decided on the device so
// the choice needs no host round trip and replays inside a CUDA graph.
__device__ __forceinline__ bool cl_heavy(const int* ps_off, long long P0, long long P1,
                                         const int* maxs) {
  const long long tot = ps_off[P1] - ps_off[P0];
  const long long mx = *maxs;
  return mx > CL_HEAVY_MIN && mx * (P1 - P0) > CL_HEAVY_RATIO * tot;
}

__global__ void __launch_bounds__(256, 3)   // keep the per-parent body's occupancy
k_classify_pred(int l, LevelGeo geo, double theta, const int* __restrict__ ps_off,
                const int* __restrict__ ps_idx, long long P0, long long P1, long long tb,
                long long te, int2* cnt, unsigned* masks, long long mplane, const int* maxs,
                DevStatus* st) {
  pdl_enter();
  if (cl_heavy(ps_off, P0, P1, maxs))
    classify_pred_chunks(l, geo, theta, ps_off, ps_idx, P0, P1, tb, te, cnt, masks, mplane, st);
  else
    classify_pred_parents(l, geo, theta, ps_off, ps_idx, P0, P1, tb, te, cnt, masks, mplane, st);
}

__global__ void __launch_bounds__(256, 5)
k_classify_fill(int l, const int* __restrict__ ps_off, const int* __restrict__ ps_idx,
                const int* __restrict__ so, int* sidx, long long scap, const int* __restrict__ woff,
                int* widx, int* wtgt, long long wcap, long long P0, long long P1, long long tb,
                long long te, const unsigned* __restrict__ masks, long long mplane,
                const int* maxs, int2* cnt, DevStatus* st) {
  pdl_enter();
  // the scan has consumed the counters: zero them for the next level's atomics
  // (the chunked predicate body accumulates into them; no memset per level)
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < 4 * (P1 - P0);
       i += (long long)gridDim.x * blockDim.x)
    cnt[i] = make_int2(0, 0);
  if (cl_heavy(ps_off, P0, P1, maxs))
    classify_fill_chunks(l, ps_off, ps_idx, so, sidx, scap, woff, widx, wtgt, wcap, P0, P1, tb,
                         te, masks, mplane, st);
  else
    classify_fill_parents(l, ps_off, ps_idx, so, sidx, scap, woff, widx, wtgt, wcap, P0, P1,
                          tb, te, masks, mplane, st);
}

// reclassify_finest (connectivity.py:71-96) in one pass: a warp walks CL_TPW
// finest targets, kinds cached as ballot masks, three-counter look-back per
// CTA, compacted ascending p2p / p2l / m2p lists.
__global__ void __launch_bounds__(CL_WARPS * 32)
k_reclassify(int L, LevelGeo geo, double theta, const int* __restrict__ s_off,
             const int* __restrict__ s_idx, int* o_p2p, int* i_p2p, long long cap_p2p,
             int* o_p2l, int* i_p2l, long long cap_p2l, int* o_m2p, int* i_m2p,
             long long cap_m2p, LookbackState lbs, unsigned ntiles, long long tb, long long te,
             DevStatus* st) {
  pdl_enter();
  __shared__ unsigned s_mask[CL_WARPS][CL_TPW][2][CL_MAXM];   // p2l, m2p (p2p = rest)
  __shared__ int s_cnt[CL_WARPS][CL_TPW][3];
  __shared__ long long s_excl[3];
  __shared__ unsigned s_tile;
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  if (threadIdx.x == 0) s_tile = lb_ticket(lbs, ntiles);
  __syncthreads();
  const unsigned tile = s_tile;
  const bool dead = lists_overflowed(st);
  const long long lb = level_base(L);
  const long long bw = tb + ((long long)tile * CL_WARPS + w) * CL_TPW;
  auto kinds = [&](long long b, double rt, double xt, double yt, int c, int a1, unsigned& ml,
                   unsigned& mm, unsigned& vm, int& src) {
    const bool valid = c < a1;
    int kind = 0;   // 0 p2p, 1 p2l (larger source), 2 m2p (smaller source)
    src = valid ? s_idx[c] : 0;
    if (valid) {
      const double rs = geo.r[lb + src];
      const bool sw = well_separated_swapped_dz(rt, rs, xt - geo.cx[lb + src],
                                                yt - geo.cy[lb + src], theta);
      const bool moved = sw && src != b && rs != rt;
      kind = moved ? (rs > rt ? 1 : 2) : 0;
    }
    vm = __ballot_sync(0xffffffffu, valid);
    ml = __ballot_sync(0xffffffffu, kind == 1);
    mm = __ballot_sync(0xffffffffu, kind == 2);
  };
  for (int u = 0; u < CL_TPW; ++u) {
    const long long b = bw + u;
    const bool live = b < te && !dead;
    int a0 = 0, a1 = 0;
    if (live) {
      a0 = s_off[b];
      a1 = s_off[b + 1];
    }
    const long long gt = lb + (live ? b : 0);
    const double rt = geo.r[gt], xt = geo.cx[gt], yt = geo.cy[gt];
    int n0 = 0, n1 = 0, n2 = 0;
    for (int c0 = a0; c0 < a1; c0 += 32) {
      unsigned ml, mm, vm;
      int src;
      kinds(b, rt, xt, yt, c0 + lane, a1, ml, mm, vm, src);
      const int ch = (c0 - a0) >> 5;
      if (lane == 0 && ch < CL_MAXM) {
        s_mask[w][u][0][ch] = ml;
        s_mask[w][u][1][ch] = mm;
      }
      n0 += __popc(vm & ~(ml | mm));
      n1 += __popc(ml);
      n2 += __popc(mm);
    }
    if (lane == 0) {
      s_cnt[w][u][0] = n0;
      s_cnt[w][u][1] = n1;
      s_cnt[w][u][2] = n2;
    }
  }
  __syncthreads();
  if (w == 0) {
    long long agg[3] = {0, 0, 0}, excl[3];
    for (int q = 0; q < CL_WARPS * CL_TPW; ++q)
      for (int k = 0; k < 3; ++k) agg[k] += (&s_cnt[0][0][0])[3 * q + k];
    lb_prefix<3>(lbs, tile, agg, excl);
    if (lane == 0)
      for (int k = 0; k < 3; ++k) s_excl[k] = excl[k];
  }
  __syncthreads();
  long long pos[3] = {s_excl[0], s_excl[1], s_excl[2]};
  for (int q = 0; q < w; ++q)
    for (int u = 0; u < CL_TPW; ++u)
      for (int k = 0; k < 3; ++k) pos[k] += s_cnt[q][u][k];
  if (tile == ntiles - 1 && w == CL_WARPS - 1 && lane == 0) {
    long long tot[3] = {pos[0], pos[1], pos[2]};
    for (int u = 0; u < CL_TPW; ++u)
      for (int k = 0; k < 3; ++k) tot[k] += s_cnt[w][u][k];
    o_p2p[te] = (int)tot[0];
    o_p2l[te] = (int)tot[1];
    o_m2p[te] = (int)tot[2];
  }
  const unsigned below = (1u << lane) - 1u;
  for (int u = 0; u < CL_TPW; ++u) {
    const long long b = bw + u;
    if (b >= te) break;
    if (lane == 0) {
      o_p2p[b] = (int)pos[0];
      o_p2l[b] = (int)pos[1];
      o_m2p[b] = (int)pos[2];
    }
    const int n0 = s_cnt[w][u][0], n1 = s_cnt[w][u][1], n2 = s_cnt[w][u][2];
    if (!dead && pos[0] + n0 <= cap_p2p && pos[1] + n1 <= cap_p2l && pos[2] + n2 <= cap_m2p) {
      const int a0 = s_off[b], a1 = s_off[b + 1];
      const long long gt = lb + b;
      long long q0 = pos[0], q1 = pos[1], q2 = pos[2];
      for (int c0 = a0; c0 < a1; c0 += 32) {
        unsigned ml, mm, vm;
        int src;
        const int ch = (c0 - a0) >> 5;
        if (ch < CL_MAXM) {
          const int c = c0 + lane;
          src = c < a1 ? s_idx[c] : 0;
          vm = __ballot_sync(0xffffffffu, c < a1);
          ml = s_mask[w][u][0][ch];
          mm = s_mask[w][u][1][ch];
        } else {
          kinds(b, geo.r[gt], geo.cx[gt], geo.cy[gt], c0 + lane, a1, ml, mm, vm, src);
        }
        const unsigned mp = vm & ~(ml | mm);
        if ((mp >> lane) & 1u) i_p2p[q0 + __popc(mp & below)] = src;
        if ((ml >> lane) & 1u) i_p2l[q1 + __popc(ml & below)] = src;
        if ((mm >> lane) & 1u) i_m2p[q2 + __popc(mm & below)] = src;
        q0 += __popc(mp);
        q1 += __popc(ml);
        q2 += __popc(mm);
      }
    } else if (!dead && lane == 0) {
      atomicOr(&st->flags, ST_OVERFLOW);
      atomicOr(&st->overflow_where, 2);
    }
    pos[0] += n0;
    pos[1] += n1;
    pos[2] += n2;
  }
}

// Split form of reclassify_finest (default, same reason as the split
// classify): k_reclassify_pred stores the p2l / m2p kind masks of every
// 32-source chunk (word base of target b: (b - tb) + (s_off[b] - s_off[tb]) /
// 32) and the three counts; k_reclassify_fill publishes its tile's counts to
// the look-back first and then writes the three compacted lists.
__device__ __forceinline__ void reclassify_pred_targets(
    int L, LevelGeo geo, double theta, const int* __restrict__ s_off,
    const int* __restrict__ s_idx, long long tb, long long te, int4* cnt, unsigned* masks,
    long long mplane, DevStatus* st) {
  const int lane = threadIdx.x & 31;
  const long long lb = level_base(L);
  const bool dead = lists_overflowed(st);
  const long long nwarps = ((long long)gridDim.x * blockDim.x) >> 5;
  for (long long b = tb + ((blockIdx.x * (long long)blockDim.x + threadIdx.x) >> 5); b < te;
       b += nwarps) {
    const int a0 = s_off[b], a1 = dead ? a0 : s_off[b + 1];
    const long long wb = (b - tb) + (s_off[b] - s_off[tb]) / 32;
    const long long gt = lb + b;
    const double rt = geo.r[gt], xt = geo.cx[gt], yt = geo.cy[gt];
    int n0 = 0, n1 = 0, n2 = 0;
    for (int c0 = a0; c0 < a1; c0 += 32) {
      const int c = c0 + lane;
      const bool valid = c < a1;
      int kind = 0;   // 0 p2p, 1 p2l (larger source), 2 m2p (smaller source)
      if (valid) {
        const int src = s_idx[c];
        const double rs = geo.r[lb + src];
        const bool sw = well_separated_swapped_dz(rt, rs, xt - geo.cx[lb + src],
                                                  yt - geo.cy[lb + src], theta);
        const bool moved = sw && src != b && rs != rt;
        kind = moved ? (rs > rt ? 1 : 2) : 0;
      }
      const unsigned vm = __ballot_sync(0xffffffffu, valid);
      const unsigned ml = __ballot_sync(0xffffffffu, kind == 1);
      const unsigned mm = __ballot_sync(0xffffffffu, kind == 2);
      const int ch = (c0 - a0) >> 5;
      if (lane == 0) masks[wb + ch] = ml;
      if (lane == 1) masks[mplane + wb + ch] = mm;
      n0 += __popc(vm & ~(ml | mm));
      n1 += __popc(ml);
      n2 += __popc(mm);
    }
    if (lane == 0) cnt[b - tb] = make_int4(n0, n1, n2, 0);
  }
}

__device__ __forceinline__ void reclassify_fill_targets(
    const int* __restrict__ s_off, const int* __restrict__ s_idx, const int* __restrict__ o_p2p,
    int* i_p2p, const int* __restrict__ o_p2l, int* i_p2l, const int* __restrict__ o_m2p,
    int* i_m2p, long long tb, long long te, const unsigned* __restrict__ masks,
    long long mplane) {
  const int lane = threadIdx.x & 31;
  const unsigned below = (1u << lane) - 1u;
  const long long nwarps = ((long long)gridDim.x * blockDim.x) >> 5;
  for (long long b = tb + ((blockIdx.x * (long long)blockDim.x + threadIdx.x) >> 5); b < te;
       b += nwarps) {
    long long q0 = o_p2p[b], q1 = o_p2l[b], q2 = o_m2p[b];
    const int a0 = s_off[b], a1 = s_off[b + 1];
    const long long wb = (b - tb) + (a0 - s_off[tb]) / 32;
    for (int c0 = a0; c0 < a1; c0 += 32) {
      const int c = c0 + lane;
      const int ch = (c0 - a0) >> 5;
      const int src = c < a1 ? s_idx[c] : 0;
      const unsigned vm = __ballot_sync(0xffffffffu, c < a1);
      const unsigned ml = masks[wb + ch], mm = masks[mplane + wb + ch];
      const unsigned mp = vm & ~(ml | mm);
      if ((mp >> lane) & 1u) i_p2p[q0 + __popc(mp & below)] = src;
      if ((ml >> lane) & 1u) i_p2l[q1 + __popc(ml & below)] = src;
      if ((mm >> lane) & 1u) i_m2p[q2 + __popc(mm & below)] = src;
      q0 += __popc(mp);
      q1 += __popc(ml);
      q2 += __popc(mm);
    }
  }
}

// off[i] for i outside the written window [lo, hi]: off[lo] before, off[hi] after
// chunked (load-balanced) reclassify: chunk ids over targets as in the
// per-target form (target b owns [(b - tb) + (s_off[b] - s_off[tb]) / 32, ...));
// counts by integer atomics, fill positions from earlier chunks' popcounts
__device__ __forceinline__ long long rc_wbase(const int* s_off, long long b, long long tb) {
  return (b - tb) + (s_off[b] - s_off[tb]) / 32;
}
__device__ __forceinline__ long long rc_target_of(const int* s_off, long long tb, long long te,
                                                  long long c) {
  const int lane = threadIdx.x & 31;
  long long lo = tb, hi = te;
  while (hi - lo > 1) {
    const long long step = (hi - lo + 31) / 32;
    const long long probe = lo + (long long)lane * step;
    const bool ok = probe < hi && rc_wbase(s_off, probe, tb) <= c;
    const unsigned bm = __ballot_sync(0xffffffffu, ok);
    lo = lo + (long long)(31 - __clz(bm)) * step;
    hi = min(hi, lo + step);
  }
  return lo;
}

__device__ __forceinline__ void reclassify_pred_chunks(
    int L, LevelGeo geo, double theta, const int* __restrict__ s_off,
    const int* __restrict__ s_idx, long long tb, long long te, int4* cnt, unsigned* masks,
    long long mplane, DevStatus* st) {
  if (lists_overflowed(st)) return;
  const int lane = threadIdx.x & 31;
  const long long lb = level_base(L);
  const long long nwarps = ((long long)gridDim.x * blockDim.x) >> 5;
  const long long wid = (blockIdx.x * (long long)blockDim.x + threadIdx.x) >> 5;
  const long long C = rc_wbase(s_off, te, tb);
  const long long per = (C + nwarps - 1) / nwarps;
  const long long c_begin = wid * per, c_end = min(C, c_begin + per);
  if (c_begin >= c_end) return;
  long long b = rc_target_of(s_off, tb, te, c_begin);
  long long wb = rc_wbase(s_off, b, tb), wnext = rc_wbase(s_off, b + 1, tb);
  int a0 = s_off[b], a1 = s_off[b + 1];
  double rt = geo.r[lb + b], xt = geo.cx[lb + b], yt = geo.cy[lb + b];
  int n0 = 0, n1 = 0, n2 = 0;
  auto flush = [&]() {
    if (lane == 0) {
      if (n0) atomicAdd(&cnt[b - tb].x, n0);
      if (n1) atomicAdd(&cnt[b - tb].y, n1);
      if (n2) atomicAdd(&cnt[b - tb].z, n2);
    }
    n0 = n1 = n2 = 0;
  };
  for (long long c = c_begin; c < c_end; ++c) {
    if (c >= wnext) {
      flush();
      do {
        ++b;
        wb = wnext;
        wnext = rc_wbase(s_off, b + 1, tb);
      } while (c >= wnext);
      a0 = s_off[b];
      a1 = s_off[b + 1];
      rt = geo.r[lb + b];
      xt = geo.cx[lb + b];
      yt = geo.cy[lb + b];
    }
    const int c0 = a0 + 32 * (int)(c - wb);
    if (c0 >= a1) continue;
    const int cc = c0 + lane;
    const bool valid = cc < a1;
    int kind = 0;
    if (valid) {
      const int src = s_idx[cc];
      const double rs = geo.r[lb + src];
      const bool sw = well_separated_swapped_dz(rt, rs, xt - geo.cx[lb + src],
                                                yt - geo.cy[lb + src], theta);
      const bool moved = sw && src != b && rs != rt;
      kind = moved ? (rs > rt ? 1 : 2) : 0;
    }
    const unsigned vm = __ballot_sync(0xffffffffu, valid);
    const unsigned ml = __ballot_sync(0xffffffffu, kind == 1);
    const unsigned mm = __ballot_sync(0xffffffffu, kind == 2);
    if (lane == 0) masks[c] = ml;
    if (lane == 1) masks[mplane + c] = mm;
    n0 += __popc(vm & ~(ml | mm));
    n1 += __popc(ml);
    n2 += __popc(mm);
  }
  flush();
}

__device__ __forceinline__ void reclassify_fill_chunks(
    const int* __restrict__ s_off, const int* __restrict__ s_idx, const int* __restrict__ o_p2p,
    int* i_p2p, const int* __restrict__ o_p2l, int* i_p2l, const int* __restrict__ o_m2p,
    int* i_m2p, long long tb, long long te, const unsigned* __restrict__ masks,
    long long mplane) {
  const int lane = threadIdx.x & 31;
  const unsigned below = (1u << lane) - 1u;
  const long long nwarps = ((long long)gridDim.x * blockDim.x) >> 5;
  const long long wid = (blockIdx.x * (long long)blockDim.x + threadIdx.x) >> 5;
  const long long C = rc_wbase(s_off, te, tb);
  const long long per = (C + nwarps - 1) / nwarps;
  const long long c_begin = wid * per, c_end = min(C, c_begin + per);
  if (c_begin >= c_end) return;
  long long b = rc_target_of(s_off, tb, te, c_begin);
  long long wb = 0, wnext = -1;
  int a0 = 0, a1 = 0;
  long long q0 = 0, q1 = 0, q2 = 0;
  for (long long c = c_begin; c < c_end; ++c) {
    if (c >= wnext) {                       // (re)enter a target: bases + earlier chunks
      if (wnext >= 0) ++b;
      while (c >= rc_wbase(s_off, b + 1, tb)) ++b;
      wb = rc_wbase(s_off, b, tb);
      wnext = rc_wbase(s_off, b + 1, tb);
      a0 = s_off[b];
      a1 = s_off[b + 1];
      const long long kc = c - wb;
      int fl = 0, fm = 0;
      for (long long k = lane; k < kc; k += 32) {
        fl += __popc(masks[wb + k]);
        fm += __popc(masks[mplane + wb + k]);
      }
#pragma unroll
      for (int d = 16; d; d >>= 1) {
        fl += __shfl_xor_sync(0xffffffffu, fl, d);
        fm += __shfl_xor_sync(0xffffffffu, fm, d);
      }
      const int before = (int)min(32 * kc, (long long)(a1 - a0));
      q0 = o_p2p[b] + (before - fl - fm);
      q1 = o_p2l[b] + fl;
      q2 = o_m2p[b] + fm;
    }
    const int c0 = a0 + 32 * (int)(c - wb);
    if (c0 >= a1) continue;
    const int cc = c0 + lane;
    const int src = cc < a1 ? s_idx[cc] : 0;
    const unsigned vm = __ballot_sync(0xffffffffu, cc < a1);
    const unsigned ml = masks[c], mm = masks[mplane + c];
    const unsigned mp = vm & ~(ml | mm);
    if ((mp >> lane) & 1u) i_p2p[q0 + __popc(mp & below)] = src;
    if ((ml >> lane) & 1u) i_p2l[q1 + __popc(ml & below)] = src;
    if ((mm >> lane) & 1u) i_m2p[q2 + __popc(mm & below)] = src;
    q0 += __popc(mp);
    q1 += __popc(ml);
    q2 += __popc(mm);
  }
}

__global__ void __launch_bounds__(256, 4)
k_reclassify_pred(int L, LevelGeo geo, double theta, const int* __restrict__ s_off,
                  const int* __restrict__ s_idx, long long tb, long long te, int4* cnt,
                  unsigned* masks, long long mplane, const int* maxs, DevStatus* st) {
  pdl_enter();
  if (cl_heavy(s_off, tb, te, maxs))
    reclassify_pred_chunks(L, geo, theta, s_off, s_idx, tb, te, cnt, masks, mplane, st);
  else
    reclassify_pred_targets(L, geo, theta, s_off, s_idx, tb, te, cnt, masks, mplane, st);
}

__global__ void __launch_bounds__(256, 7)
k_reclassify_fill(const int* __restrict__ s_off, const int* __restrict__ s_idx,
                  const int* __restrict__ o_p2p, int* i_p2p, long long cap_p2p,
                  const int* __restrict__ o_p2l, int* i_p2l, long long cap_p2l,
                  const int* __restrict__ o_m2p, int* i_m2p, long long cap_m2p, long long tb,
                  long long te, const unsigned* __restrict__ masks, long long mplane,
                  const int* maxs, int4* cnt, DevStatus* st) {
  pdl_enter();
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < te - tb;
       i += (long long)gridDim.x * blockDim.x)
    cnt[i] = make_int4(0, 0, 0, 0);
  if (lists_overflowed(st)) return;
  if (o_p2p[te] > cap_p2p || o_p2l[te] > cap_p2l || o_m2p[te] > cap_m2p) {
    if (blockIdx.x == 0 && threadIdx.x == 0) {
      atomicOr(&st->flags, ST_OVERFLOW);
      atomicOr(&st->overflow_where, 2);
    }
    return;
  }
  if (cl_heavy(s_off, tb, te, maxs))
    reclassify_fill_chunks(s_off, s_idx, o_p2p, i_p2p, o_p2l, i_p2l, o_m2p, i_m2p, tb, te, masks,
                           mplane);
  else
    reclassify_fill_targets(s_off, s_idx, o_p2p, i_p2p, o_p2l, i_p2l, o_m2p, i_m2p, tb, te,
                            masks, mplane);
}

__global__ void k_csr_pad(int* off, long long n, long long lo, long long hi) {
  pdl_enter();
  const long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (i > n) return;
  if (i < lo) off[i] = off[lo];
  else if (i > hi) off[i] = off[hi];
}

__global__ void k_root_lists(int* weak_off, int* s_off, int* s_idx, unsigned* lb_base,
                             int* lvl_max, int nlvl) {
  pdl_enter();
  for (int i = threadIdx.x; i < nlvl; i += blockDim.x) lvl_max[i] = 0;
  if (threadIdx.x) return;
  lb_advance_base(lb_base);   // this evaluation's look-back epoch base (lookback.cuh)
  weak_off[0] = 0;
  weak_off[1] = 0;     // the root has no far field (connectivity.py:106)
  s_off[0] = 0;
  s_off[1] = 1;
  s_idx[0] = 0;        // strong[0] = [0] (connectivity.py:107)
}

__global__ void k_radius(const double* hw, const double* hh, double* r, long long n) {
  pdl_enter();
  long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (i < n) r[i] = glibc_hypot(hw[i], hh[i]);
}

// list-length histograms and maxima for EngineReport (engine.py:185-204):
// warp-aggregated (match_any) into a block-private SMEM histogram, then one
// global add per non-empty bin
__global__ void __launch_bounds__(256)
k_histogram(const int* __restrict__ off, long long n, int kind, int* hist, DevStatus* st) {
  pdl_enter();
  __shared__ int sh[HIST_BINS];
  __shared__ int smax;
  if (lists_overflowed(st)) return;
  for (int i = threadIdx.x; i < HIST_BINS; i += blockDim.x) sh[i] = 0;
  if (threadIdx.x == 0) smax = 0;
  __syncthreads();
  int mx = 0;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i - threadIdx.x < n;
       i += (long long)gridDim.x * blockDim.x) {
    const bool valid = i < n;
    const int len = valid ? off[i + 1] - off[i] : -1;
    const int bin = min(len, HIST_BINS - 1);
    const unsigned peers = __match_any_sync(0xffffffffu, bin);
    if (valid && (threadIdx.x & 31) == __ffs(peers) - 1) atomicAdd(&sh[bin], __popc(peers));
    mx = max(mx, len);
  }
  for (int d = 16; d; d >>= 1) mx = max(mx, __shfl_xor_sync(0xffffffffu, mx, d));
  if ((threadIdx.x & 31) == 0) atomicMax(&smax, mx);
  __syncthreads();
  for (int i = threadIdx.x; i < HIST_BINS; i += blockDim.x)
    if (sh[i]) atomicAdd(&hist[kind * HIST_BINS + i], sh[i]);
  if (threadIdx.x == 0) atomicMax(&st->max_len[kind], smax);
}

inline unsigned nblk(long long n, int t) { return (unsigned)((n + t - 1) / t); }

}  // namespace

void compute_radius(TreeState& T, cudaStream_t st) {
  const long long nbox = level_base(T.L + 1);
  note_launch();
  launch(k_radius, nblk(nbox, 256), 256, 0, st, T.box_hw.as<double>(), T.box_hh.as<double>(),
                                            T.box_r.as<double>(), nbox);
}

void run_connectivity(const TreeState& T, ListState& Ls, double theta, DevStatus* dstat,
                      cudaStream_t st, const Part& part) {
  const int L = T.L;
  const long long nbox = level_base(L + 1);
  const long long nleaf = 1ll << (2 * L);
  // capacities: at least a generous estimate for this tree, else the high-water mark
  Ls.cap_weak = std::max<long long>(Ls.cap_weak, std::max<long long>(4096, 64 * nbox));
  Ls.cap_strong = std::max<long long>(Ls.cap_strong, std::max<long long>(4096, 48 * nleaf));
  Ls.cap_p2p = std::max<long long>(Ls.cap_p2p, std::max<long long>(4096, 32 * nleaf));
  Ls.cap_p2l = std::max<long long>(Ls.cap_p2l, std::max<long long>(4096, 8 * nleaf));
  Ls.cap_m2p = std::max<long long>(Ls.cap_m2p, std::max<long long>(4096, 8 * nleaf));
  Ls.weak_off.reserve(sizeof(int) * (nbox + 1));
  Ls.weak_idx.reserve(sizeof(int) * Ls.cap_weak);
  Ls.weak_tgt.reserve(sizeof(int) * Ls.cap_weak);
  for (int q = 0; q < 2; ++q) {
    Ls.s_off[q].reserve(sizeof(int) * (nleaf + 1));
    Ls.s_idx[q].reserve(sizeof(int) * std::max<long long>(Ls.cap_strong, 1));
  }
  for (DBuf* b : {&Ls.p2p_off, &Ls.p2l_off, &Ls.m2p_off}) b->reserve(sizeof(int) * (nleaf + 1));
  Ls.p2p_idx.reserve(sizeof(int) * Ls.cap_p2p);
  Ls.p2l_idx.reserve(sizeof(int) * Ls.cap_p2l);
  Ls.m2p_idx.reserve(sizeof(int) * Ls.cap_m2p);
  Ls.hist.reserve(sizeof(int) * 4 * HIST_BINS);

  // look-back state: flags + 3 counters per tile, grow-only, epoch-tagged
  const long long max_tiles = (nleaf + CL_WARPS - 1) / CL_WARPS + 1;   // >= tiles of any launch
  if (Ls.lb_tiles < max_tiles) {
    Ls.lb_flags.reserve(sizeof(unsigned) * max_tiles);
    Ls.lb_vals.reserve(sizeof(long long) * 6 * max_tiles);
    Ls.lb_ticket.reserve(sizeof(unsigned) * 4);
    FMM_CUDA(cudaMemsetAsync(Ls.lb_flags.p, 0, sizeof(unsigned) * max_tiles, st));
    FMM_CUDA(cudaMemsetAsync(Ls.lb_ticket.p, 0, sizeof(unsigned) * 4, st));
    Ls.lb_tiles = max_tiles;
  }
  unsigned* lb_base = lb_base_prepare(Ls.lb_base, Ls.lb_base_ready, st);
  Ls.lb_epoch = 0;
  auto lbstate = [&]() {
    ++Ls.lb_epoch;
    long long* v = Ls.lb_vals.as<long long>();
    return LookbackState{Ls.lb_flags.as<unsigned>(), v, v + 3 * max_tiles,
                         Ls.lb_ticket.as<unsigned>(), Ls.lb_epoch, lb_base};
  };

  const LevelGeo geo{T.box_cx.as<double>(), T.box_cy.as<double>(), T.box_r.as<double>()};
  int* woff = Ls.weak_off.as<int>();
  // split classify scratch: counts per target, four far-mask planes per level
  const long long mplane = nleaf / 4 + Ls.cap_strong / 8 + 4;      // classify planes (4)
  const long long rplane = nleaf + Ls.cap_strong / 32 + 4;          // reclassify planes (2)
  if (cl_split()) {
    Ls.cl_cnt.reserve(sizeof(int4) * (nleaf + 4));
    if (Ls.cl_cnt_zeroed != (long long)Ls.cl_cnt.bytes) {   // fresh buffer: zero once; each
      FMM_CUDA(cudaMemsetAsync(Ls.cl_cnt.p, 0, Ls.cl_cnt.bytes, st));   // scan re-zeroes it
      Ls.cl_cnt_zeroed = (long long)Ls.cl_cnt.bytes;
    }
    Ls.cl_mask.reserve(sizeof(unsigned) * std::max(4 * mplane, 2 * rplane));
  }
  // longest strong list per level (cl_heavy); slot L+1 is a permanent zero
  Ls.lvl_max.reserve(sizeof(int) * (L + 2));
  int* lvl_max = Ls.lvl_max.as<int>();
  note_launch();
  launch(k_root_lists, 1, 32, 0, st, woff, Ls.s_off[0].as<int>(), Ls.s_idx[0].as<int>(), lb_base,
         lvl_max, L + 2);
  int cur = 0;
  for (int l = 1; l <= L; ++l) {
    const long long tb = part.lo(l), te = part.hi(l);
    const long long P0 = tb >> 2, P1 = (te + 3) >> 2;
    if (cl_split() && P1 - P0 >= CL_SPLIT_MIN) {
      const long long nt = 4 * (P1 - P0);
      const unsigned stiles = (unsigned)((nt + SCAN_TILE - 1) / SCAN_TILE);
      // parents' longest strong list (recorded by level l-1); slot L+1 stays 0
      const int* maxs_prev = cl_chunked() ? lvl_max + (l - 1) : lvl_max + (L + 1);
      note_launch();
      launch(k_classify_pred, CL_GRID_CAP, 256, 0, st, l, geo, theta, Ls.s_off[cur].as<int>(),
             Ls.s_idx[cur].as<int>(), P0, P1, tb, te, Ls.cl_cnt.as<int2>(),
             Ls.cl_mask.as<unsigned>(), mplane, maxs_prev, dstat);
      const ScanOut so{{woff + level_base(l) + 4 * P0, Ls.s_off[1 - cur].as<int>() + 4 * P0,
                        nullptr},
                       woff + level_base(l), woff + level_base(l + 1)};
      note_launch();
      launch(k_scan_counts<2, 2>, stiles, SCAN_THREADS, 0, st,
             reinterpret_cast<const int*>(Ls.cl_cnt.as<int2>()), nt, so, lbstate(), stiles,
             lvl_max + l, dstat);
      note_launch();
      launch(k_classify_fill, CL_GRID_CAP, 256, 0, st, l, Ls.s_off[cur].as<int>(),
             Ls.s_idx[cur].as<int>(), Ls.s_off[1 - cur].as<int>(), Ls.s_idx[1 - cur].as<int>(),
             Ls.cap_strong, woff, Ls.weak_idx.as<int>(), Ls.weak_tgt.as<int>(), Ls.cap_weak, P0,
             P1, tb, te, Ls.cl_mask.as<unsigned>(), mplane, maxs_prev, Ls.cl_cnt.as<int2>(),
             dstat);
    } else {
      const unsigned ntiles = (unsigned)((P1 - P0 + CL_WARPS * CL_PPW - 1) / (CL_WARPS * CL_PPW));
      note_launch();
      launch(k_classify, ntiles, CL_WARPS * 32, 0, st,
          l, geo, theta, Ls.s_off[cur].as<int>(), Ls.s_idx[cur].as<int>(),
          Ls.s_off[1 - cur].as<int>(), Ls.s_idx[1 - cur].as<int>(), Ls.cap_strong, woff,
          Ls.weak_idx.as<int>(), Ls.weak_tgt.as<int>(), Ls.cap_weak, lbstate(), ntiles, P0, P1,
          tb, te, lvl_max + l, dstat);
    }
    cur = 1 - cur;
  }
  {
    const long long tb = part.lo(L), te = part.hi(L);
    const unsigned ntiles = (unsigned)((te - tb + CL_WARPS * CL_TPW - 1) / (CL_WARPS * CL_TPW));
    if (cl_split() && te - tb >= 4 * CL_SPLIT_MIN) {
      const unsigned stiles = (unsigned)((te - tb + SCAN_TILE - 1) / SCAN_TILE);
      const int* maxs_fin = cl_chunked() ? lvl_max + L : lvl_max + (L + 1);
      note_launch();
      launch(k_reclassify_pred, CL_GRID_CAP, 256, 0, st, L, geo, theta, Ls.s_off[cur].as<int>(),
             Ls.s_idx[cur].as<int>(), tb, te, Ls.cl_cnt.as<int4>(), Ls.cl_mask.as<unsigned>(),
             rplane, maxs_fin, dstat);
      const ScanOut so{{Ls.p2p_off.as<int>() + tb, Ls.p2l_off.as<int>() + tb,
                        Ls.m2p_off.as<int>() + tb},
                       nullptr, nullptr};
      note_launch();
      launch(k_scan_counts<3, 4>, stiles, SCAN_THREADS, 0, st,
             reinterpret_cast<const int*>(Ls.cl_cnt.as<int4>()), te - tb, so, lbstate(), stiles,
             nullptr, dstat);
      note_launch();
      launch(k_reclassify_fill, CL_GRID_CAP, 256, 0, st, Ls.s_off[cur].as<int>(),
             Ls.s_idx[cur].as<int>(), Ls.p2p_off.as<int>(), Ls.p2p_idx.as<int>(), Ls.cap_p2p,
             Ls.p2l_off.as<int>(), Ls.p2l_idx.as<int>(), Ls.cap_p2l, Ls.m2p_off.as<int>(),
             Ls.m2p_idx.as<int>(), Ls.cap_m2p, tb, te, Ls.cl_mask.as<unsigned>(), rplane,
             maxs_fin, Ls.cl_cnt.as<int4>(), dstat);
    } else {
      note_launch();
      launch(k_reclassify, ntiles, CL_WARPS * 32, 0, st,
          L, geo, theta, Ls.s_off[cur].as<int>(), Ls.s_idx[cur].as<int>(), Ls.p2p_off.as<int>(),
          Ls.p2p_idx.as<int>(), Ls.cap_p2p, Ls.p2l_off.as<int>(), Ls.p2l_idx.as<int>(),
          Ls.cap_p2l, Ls.m2p_off.as<int>(), Ls.m2p_idx.as<int>(), Ls.cap_m2p, lbstate(), ntiles,
          tb, te, dstat);
    }
  }
  if (part.G > 1) {
    // empty lists for boxes this rank does not own: monotone CSR offsets
    for (int l = 1; l <= L; ++l) {
      note_launch();
      launch(k_csr_pad, nblk((1ll << (2 * l)) + 1, 256), 256, 0, st, woff + level_base(l), 1ll << (2 * l),
                                                           part.lo(l), part.hi(l));
    }
    for (DBuf* o : {&Ls.p2p_off, &Ls.p2l_off, &Ls.m2p_off}) {
      note_launch();
      launch(k_csr_pad, nblk(nleaf + 1, 256), 256, 0, st, o->as<int>(), nleaf, part.lo(L), part.hi(L));
    }
  }
}

__global__ void k_list_totals(const int* w, const int* a, const int* b, const int* c,
                              DevStatus* st) {
  pdl_enter();
  if (threadIdx.x == 0) {
    st->list_total[0] = *w;
    st->list_total[1] = *a;
    st->list_total[2] = *b;
    st->list_total[3] = *c;
  }
}

void run_stats(const TreeState& T, ListState& Ls, DevStatus* dstat, cudaStream_t st,
               const Part& part) {
  const int L = T.L;
  const long long nbox = level_base(L + 1);
  const long long nleaf = 1ll << (2 * L);
  FMM_CUDA(cudaMemsetAsync(Ls.hist.p, 0, sizeof(int) * 4 * HIST_BINS, st));
  auto hist = [&](const int* off, long long n, int kind) {
    if (n <= 0) return;
    note_launch();
    launch(k_histogram, std::min(nblk(n, 256), 296u), 256, 0, st, off, n, kind, Ls.hist.as<int>(),
                                                              dstat);
  };
  if (part.G == 1) {
    hist(Ls.weak_off.as<int>(), nbox, 0);
  } else {
    // owned boxes per level; shared (top) levels are counted by rank 0 only
    for (int l = 0; l <= L; ++l) {
      if (part.shared(l) && part.rank != 0) continue;
      hist(Ls.weak_off.as<int>() + level_base(l) + part.lo(l), part.hi(l) - part.lo(l), 0);
    }
  }
  const long long f0 = part.lo(L), f1 = part.hi(L);
  hist(Ls.p2p_off.as<int>() + f0, f1 - f0, 1);
  hist(Ls.p2l_off.as<int>() + f0, f1 - f0, 2);
  hist(Ls.m2p_off.as<int>() + f0, f1 - f0, 3);
  // the totals travel with the status word (no extra host round trips)
  note_launch();
  launch(k_list_totals, 1, 32, 0, st, Ls.weak_off.as<int>() + nbox, Ls.p2p_off.as<int>() + nleaf,
         Ls.p2l_off.as<int>() + nleaf, Ls.m2p_off.as<int>() + nleaf, dstat);
}

}  // namespace fmm
