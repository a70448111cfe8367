// Connectivity ("connect" phase): θ-criterion interaction lists, bit-exact.
//
// Reference: connectivity.py:47-68 (classify_level), :71-96
// (reclassify_finest), :99-114 (build_connectivity); predicates
// geometry.py:27-54 restated bit-exactly in common.cuh.
//
// One warp per target box.  Candidates of box b are the children of the
// boxes strongly coupled to its parent, generated in ascending order, so the
// ballot/popc compaction below writes every list already sorted ascending
// (the property connectivity.py:10-12 promises).  Counts -> device scan ->
// fill; the weak lists of all levels form one global CSR (global box ids),
// which is also the pair list the single M2L launch consumes.  No host sync:
// list buffers are sized from capacities kept in the context, and a fill that
// would overflow only raises ST_OVERFLOW (the host then regrows and reruns).
#include "engine.h"

namespace fmm {

namespace {

constexpr int CONN_THREADS = 256;

struct LevelGeo {
  const double* cx;
  const double* cy;
  const double* r;
};

// candidate c (0-based) of target b at level l: child (c & 3) of the (c >> 2)-th
// strong box of b's parent
__global__ void __launch_bounds__(CONN_THREADS)
k_classify(int l, LevelGeo geo, double theta, const int* __restrict__ ps_off,
           const int* __restrict__ ps_idx, int* wcnt, int* scnt,
           // fill mode (woff != nullptr)
           const int* __restrict__ woff, int* widx, int* wtgt, long long wcap,
           const int* __restrict__ soff, int* sidx, long long scap, DevStatus* st) {
  const long long b = (blockIdx.x * (long long)blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  const long long nb = 1ll << (2 * l);
  if (b >= nb || lists_overflowed(st)) return;
  const long long gb = level_base(l) + b;
  const long long lb = level_base(l);
  const double rt = geo.r[gb], xt = geo.cx[gb], yt = geo.cy[gb];
  const int a0 = ps_off[b >> 2], a1 = ps_off[(b >> 2) + 1];
  const int ncand = 4 * (a1 - a0);
  const bool fill = woff != nullptr;
  long long wpos = 0, spos = 0;
  if (fill) {
    wpos = woff[gb];
    spos = soff[b];
    if (lane == 0) {
      const long long wend = woff[gb + 1], send = soff[b + 1];
      if (wend > wcap || send > scap) {
        atomicOr(&st->flags, ST_OVERFLOW);
        atomicOr(&st->overflow_where, 1);
      }
    }
    if (woff[gb + 1] > wcap || soff[b + 1] > scap) return;
  }
  int nw = 0, ns = 0;
  for (int c0 = 0; c0 < ncand; c0 += 32) {
    const int c = c0 + lane;
    bool valid = c < ncand, far = false;
    int cand = 0;
    if (valid) {
      cand = 4 * ps_idx[a0 + (c >> 2)] + (c & 3);
      const long long gc = lb + cand;
      // d = |c_target - c_source| (geometry.py:40), then the θ-test (:41)
      const double d = numpy_cabs(xt - geo.cx[gc], yt - geo.cy[gc]);
      far = well_separated(rt, geo.r[gc], d, theta);
    }
    const unsigned wm = __ballot_sync(0xffffffffu, valid && far);
    const unsigned sm = __ballot_sync(0xffffffffu, valid && !far);
    if (fill) {
      const unsigned below = (1u << lane) - 1u;
      if (valid && far) {
        const long long o = wpos + nw + __popc(wm & below);
        widx[o] = (int)(lb + cand);
        wtgt[o] = (int)gb;
      }
      if (valid && !far) sidx[spos + ns + __popc(sm & below)] = cand;
    }
    nw += __popc(wm);
    ns += __popc(sm);
  }
  if (!fill && lane == 0) {
    wcnt[b] = nw;
    scnt[b] = ns;
  }
}

// finest reclassification with the radii exchanging roles (connectivity.py:71-96)
__global__ void __launch_bounds__(CONN_THREADS)
k_reclassify(int L, LevelGeo geo, double theta, const int* __restrict__ s_off,
             const int* __restrict__ s_idx, int* c_p2p, int* c_p2l, int* c_m2p,
             const int* __restrict__ o_p2p, int* i_p2p, long long cap_p2p,
             const int* __restrict__ o_p2l, int* i_p2l, long long cap_p2l,
             const int* __restrict__ o_m2p, int* i_m2p, long long cap_m2p, DevStatus* st) {
  const long long b = (blockIdx.x * (long long)blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  const long long nb = 1ll << (2 * L);
  if (b >= nb || lists_overflowed(st)) return;
  const long long lb = level_base(L);
  const double rt = geo.r[lb + b], xt = geo.cx[lb + b], yt = geo.cy[lb + b];
  const int a0 = s_off[b], a1 = s_off[b + 1];
  const bool fill = o_p2p != nullptr;
  long long p0 = 0, l0 = 0, m0 = 0;
  if (fill) {
    if (o_p2p[b + 1] > cap_p2p || o_p2l[b + 1] > cap_p2l || o_m2p[b + 1] > cap_m2p) {
      if (lane == 0) {
        atomicOr(&st->flags, ST_OVERFLOW);
        atomicOr(&st->overflow_where, 2);
      }
      return;
    }
    p0 = o_p2p[b]; l0 = o_p2l[b]; m0 = o_m2p[b];
  }
  int np = 0, nl = 0, nm = 0;
  for (int c0 = a0; c0 < a1; c0 += 32) {
    const int c = c0 + lane;
    const bool valid = c < a1;
    int src = 0, kind = 0;   // 0 p2p, 1 p2l (larger source), 2 m2p (smaller source)
    if (valid) {
      src = s_idx[c];
      const double rs = geo.r[lb + src];
      const double d = numpy_cabs(xt - geo.cx[lb + src], yt - geo.cy[lb + src]);
      const bool sw = well_separated_swapped(rt, rs, d, theta);
      const bool moved = sw && src != b && rs != rt;
      kind = moved ? (rs > rt ? 1 : 2) : 0;
    }
    const unsigned mp = __ballot_sync(0xffffffffu, valid && kind == 0);
    const unsigned ml = __ballot_sync(0xffffffffu, valid && kind == 1);
    const unsigned mm = __ballot_sync(0xffffffffu, valid && kind == 2);
    if (fill && valid) {
      const unsigned below = (1u << lane) - 1u;
      if (kind == 0) i_p2p[p0 + np + __popc(mp & below)] = src;
      else if (kind == 1) i_p2l[l0 + nl + __popc(ml & below)] = src;
      else i_m2p[m0 + nm + __popc(mm & below)] = src;
    }
    np += __popc(mp); nl += __popc(ml); nm += __popc(mm);
  }
  if (!fill && lane == 0) {
    c_p2p[b] = np; c_p2l[b] = nl; c_m2p[b] = nm;
  }
}

__global__ void k_root_lists(int* weak_off, int* s_off, int* s_idx) {
  weak_off[0] = 0;
  weak_off[1] = 0;     // the root has no far field (connectivity.py:106)
  s_off[0] = 0;
  s_off[1] = 1;
  s_idx[0] = 0;        // strong[0] = [0] (connectivity.py:107)
}

__global__ void k_radius(const double* hw, const double* hh, double* r, long long n) {
  long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (i < n) r[i] = glibc_hypot(hw[i], hh[i]);
}

// list-length histograms and maxima for EngineReport (engine.py:185-204):
// warp-aggregated (match_any) into a block-private SMEM histogram, then one
// global add per non-empty bin
__global__ void __launch_bounds__(256)
k_histogram(const int* __restrict__ off, long long n, int kind, int* hist, DevStatus* st) {
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
  k_radius<<<nblk(nbox, 256), 256, 0, st>>>(T.box_hw.as<double>(), T.box_hh.as<double>(),
                                            T.box_r.as<double>(), nbox);
}

void run_connectivity(const TreeState& T, ListState& Ls, double theta, DevStatus* dstat,
                      cudaStream_t st) {
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
  for (DBuf* b : {&Ls.cnt_a, &Ls.cnt_b, &Ls.cnt_c}) b->reserve(sizeof(int) * nleaf);
  for (DBuf* b : {&Ls.p2p_off, &Ls.p2l_off, &Ls.m2p_off}) b->reserve(sizeof(int) * (nleaf + 1));
  Ls.p2p_idx.reserve(sizeof(int) * Ls.cap_p2p);
  Ls.p2l_idx.reserve(sizeof(int) * Ls.cap_p2l);
  Ls.m2p_idx.reserve(sizeof(int) * Ls.cap_m2p);
  Ls.hist.reserve(sizeof(int) * 4 * HIST_BINS);

  const LevelGeo geo{T.box_cx.as<double>(), T.box_cy.as<double>(), T.box_r.as<double>()};
  int* woff = Ls.weak_off.as<int>();
  note_launch();
  k_root_lists<<<1, 1, 0, st>>>(woff, Ls.s_off[0].as<int>(), Ls.s_idx[0].as<int>());
  int cur = 0;
  for (int l = 1; l <= L; ++l) {
    const long long nb = 1ll << (2 * l);
    const unsigned blocks = nblk(nb * 32, CONN_THREADS);
    const int* ps_off = Ls.s_off[cur].as<int>();
    const int* ps_idx = Ls.s_idx[cur].as<int>();
    int* wcnt = Ls.cnt_a.as<int>();
    int* scnt = Ls.cnt_b.as<int>();
    note_launch();
    k_classify<<<blocks, CONN_THREADS, 0, st>>>(l, geo, theta, ps_off, ps_idx, wcnt, scnt,
                                                nullptr, nullptr, nullptr, 0, nullptr, nullptr,
                                                0, dstat);
    // weak offsets continue the global CSR: base = end of the previous level
    int* wo = woff + level_base(l);
    scan_exclusive(wcnt, wo, nb, Ls.totals, st, wo);
    int* so = Ls.s_off[1 - cur].as<int>();
    scan_exclusive(scnt, so, nb, Ls.totals, st, nullptr);
    note_launch();
    k_classify<<<blocks, CONN_THREADS, 0, st>>>(l, geo, theta, ps_off, ps_idx, nullptr, nullptr,
                                                woff, Ls.weak_idx.as<int>(),
                                                Ls.weak_tgt.as<int>(), Ls.cap_weak, so,
                                                Ls.s_idx[1 - cur].as<int>(), Ls.cap_strong,
                                                dstat);
    cur = 1 - cur;
  }
  {
    const unsigned blocks = nblk(nleaf * 32, CONN_THREADS);
    const int* s_off = Ls.s_off[cur].as<int>();
    const int* s_idx = Ls.s_idx[cur].as<int>();
    note_launch();
    k_reclassify<<<blocks, CONN_THREADS, 0, st>>>(
        L, geo, theta, s_off, s_idx, Ls.cnt_a.as<int>(), Ls.cnt_b.as<int>(), Ls.cnt_c.as<int>(),
        nullptr, nullptr, 0, nullptr, nullptr, 0, nullptr, nullptr, 0, dstat);
    scan_exclusive(Ls.cnt_a.as<int>(), Ls.p2p_off.as<int>(), nleaf, Ls.totals, st);
    scan_exclusive(Ls.cnt_b.as<int>(), Ls.p2l_off.as<int>(), nleaf, Ls.totals, st);
    scan_exclusive(Ls.cnt_c.as<int>(), Ls.m2p_off.as<int>(), nleaf, Ls.totals, st);
    note_launch();
    k_reclassify<<<blocks, CONN_THREADS, 0, st>>>(
        L, geo, theta, s_off, s_idx, nullptr, nullptr, nullptr, Ls.p2p_off.as<int>(),
        Ls.p2p_idx.as<int>(), Ls.cap_p2p, Ls.p2l_off.as<int>(), Ls.p2l_idx.as<int>(),
        Ls.cap_p2l, Ls.m2p_off.as<int>(), Ls.m2p_idx.as<int>(), Ls.cap_m2p, dstat);
  }
}

void run_stats(const TreeState& T, ListState& Ls, DevStatus* dstat, cudaStream_t st) {
  const long long nbox = level_base(T.L + 1);
  const long long nleaf = 1ll << (2 * T.L);
  FMM_CUDA(cudaMemsetAsync(Ls.hist.p, 0, sizeof(int) * 4 * HIST_BINS, st));
  note_launch();
  k_histogram<<<std::min(nblk(nbox, 256), 296u), 256, 0, st>>>(Ls.weak_off.as<int>(), nbox, 0, Ls.hist.as<int>(),
                                               dstat);
  note_launch();
  k_histogram<<<std::min(nblk(nleaf, 256), 296u), 256, 0, st>>>(Ls.p2p_off.as<int>(), nleaf, 1,
                                                Ls.hist.as<int>(), dstat);
  note_launch();
  k_histogram<<<std::min(nblk(nleaf, 256), 296u), 256, 0, st>>>(Ls.p2l_off.as<int>(), nleaf, 2,
                                                Ls.hist.as<int>(), dstat);
  note_launch();
  k_histogram<<<std::min(nblk(nleaf, 256), 296u), 256, 0, st>>>(Ls.m2p_off.as<int>(), nleaf, 3,
                                                Ls.hist.as<int>(), dstat);
}

}  // namespace fmm
