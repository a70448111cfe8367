// Expansion kernels: P2M, P2L, M2M, M2L, L2L, L2P+M2P (FP64, registers).
//
// Reference: operators.py:194-386 (unit operators), engine.py:67-160 (phase
// drivers).  Conventions kept verbatim: p2m a_0 = 0, a_j = -sum g (z-z0)^(j-1);
// p2l b_k = sum g/(z-z0)^(k+1); every shift = source center - target center;
// scaled cascades with the unscaled fallback outside |r| in [1e-12, 1e12].
// a_0 is identically zero in the harmonic pipeline (p2m writes 0 and m2m
// preserves it), so the a_0 log corrections (operators.py:236-241, 345-350)
// are never live and are not evaluated.
//
// Every kernel is compiled for a fixed order PM >= p; coefficients above the
// runtime p are zero-padded.  All shift operators are triangular in the
// right direction (m2m lower, l2l upper, m2l's dense form has no p
// dependence), so the first p+1 outputs equal the order-p operator exactly in
// exact arithmetic.  B200 note (profiles/r01_fp64_peak.json): DMMA and DFMA
// share one FP64 pipe (36.8 vs 36.5 TFLOP/s, 36.4 mixed), so the M2L stays a
// register cascade on the vector pipe rather than an FP64 tensor-core GEMM.
#include "engine.h"

namespace fmm {

namespace {

constexpr double SCALED_LO = 1e-12, SCALED_HI = 1e12;   // operators.py:168-169

__device__ __forceinline__ cplx ld_coef(const double2* base, int j, int p) {
  if (j > p) return cplx{0.0, 0.0};
  double2 v = base[j];
  return cplx{v.x, v.y};
}

// --------------------------------------------------------------------------
// P2M (engine.py:67-82): one thread per leaf, sequential over its sources
template <int PM>
__global__ void __launch_bounds__(128)
k_p2m(int L, const int* __restrict__ offL, const double2* __restrict__ src_pos,
      const double* __restrict__ src_g, const double* __restrict__ cx,
      const double* __restrict__ cy, double2* mult, int p) {
  const long long b = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (b >= (1ll << (2 * L))) return;
  const long long gb = level_base(L) + b;
  const double x0 = cx[gb], y0 = cy[gb];
  cplx acc[PM + 1];
#pragma unroll
  for (int j = 0; j <= PM; ++j) acc[j] = cplx{0.0, 0.0};
  const int s0 = offL[b], s1 = offL[b + 1];
  for (int i = s0; i < s1; ++i) {
    const double2 z = src_pos[i];
    const cplx d{z.x - x0, z.y - y0};
    cplx w{src_g[i], 0.0};
#pragma unroll
    for (int j = 1; j <= PM; ++j) {
      acc[j] = csub(acc[j], w);
      w = cmul(w, d);
    }
  }
  double2* out = mult + gb * (p + 1);
#pragma unroll
  for (int j = 0; j <= PM; ++j)
    if (j <= p) out[j] = make_double2(acc[j].x, acc[j].y);
}

// P2L (engine.py:85-93, operators.py:209-224): target-owned, sources ascending
template <int PM>
__global__ void __launch_bounds__(128)
k_p2l(int L, const int* __restrict__ offL, const int* __restrict__ l_off,
      const int* __restrict__ l_idx, const double2* __restrict__ src_pos,
      const double* __restrict__ src_g, const double* __restrict__ cx,
      const double* __restrict__ cy, double2* local, int p, DevStatus* st) {
  const long long b = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (b >= (1ll << (2 * L)) || lists_overflowed(st)) return;
  const long long lb = level_base(L);
  const double x0 = cx[lb + b], y0 = cy[lb + b];
  cplx loc[PM + 1];
#pragma unroll
  for (int j = 0; j <= PM; ++j) loc[j] = cplx{0.0, 0.0};
  for (int q = l_off[b]; q < l_off[b + 1]; ++q) {
    const int a = l_idx[q];
    cplx box[PM + 1];
#pragma unroll
    for (int j = 0; j <= PM; ++j) box[j] = cplx{0.0, 0.0};
    for (int i = offL[a]; i < offL[a + 1]; ++i) {
      const double2 z = src_pos[i];
      const cplx d{z.x - x0, z.y - y0};
      if (d.x == 0.0 && d.y == 0.0) {
        atomicOr(&st->flags, ST_P2L_SINGULAR);
        continue;
      }
      const cplx inv = crcp(d);
      cplx w = cscale(inv, src_g[i]);
#pragma unroll
      for (int k = 0; k <= PM; ++k) {
        box[k] = cadd(box[k], w);
        w = cmul(w, inv);
      }
    }
#pragma unroll
    for (int j = 0; j <= PM; ++j) loc[j] = cadd(loc[j], box[j]);
  }
  double2* out = local + (lb + b) * (p + 1);
#pragma unroll
  for (int j = 0; j <= PM; ++j)
    if (j <= p) out[j] = make_double2(loc[j].x, loc[j].y);
}

// --------------------------------------------------------------------------
// M2M (engine.py:96-100, operators.py:231-279): thread per parent, children 0..3
template <int PM>
__device__ __forceinline__ void m2m_shift(cplx (&a)[PM + 1], cplx r) {
  const double mag = numpy_cabs(r.x, r.y);
  if (mag >= SCALED_LO && mag <= SCALED_HI) {
    const cplx inv = crcp(r);
    cplx pw = inv;
#pragma unroll
    for (int j = 1; j <= PM; ++j) {
      a[j] = cmul(a[j], pw);
      pw = cmul(pw, inv);
    }
#pragma unroll
    for (int k = PM; k >= 2; --k)
#pragma unroll
      for (int j = k; j <= PM; ++j) a[j] = cadd(a[j], a[j - 1]);
    pw = r;
#pragma unroll
    for (int j = 1; j <= PM; ++j) {
      a[j] = cmul(a[j], pw);
      pw = cmul(pw, r);
    }
  } else {
#pragma unroll
    for (int k = PM; k >= 2; --k)
#pragma unroll
      for (int j = k; j <= PM; ++j) a[j] = cadd(a[j], cmul(r, a[j - 1]));
  }
}

template <int PM>
__global__ void __launch_bounds__(128)
k_m2m(int l, const double* __restrict__ cx, const double* __restrict__ cy, double2* mult, int p) {
  const long long k = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (k >= (1ll << (2 * l))) return;
  const long long gp = level_base(l) + k;
  const long long gc0 = level_base(l + 1) + 4 * k;
  cplx acc[PM + 1];
#pragma unroll
  for (int j = 0; j <= PM; ++j) acc[j] = cplx{0.0, 0.0};
  for (int c = 0; c < 4; ++c) {
    const long long gc = gc0 + c;
    const double2* src = mult + gc * (p + 1);
    cplx a[PM + 1];
#pragma unroll
    for (int j = 0; j <= PM; ++j) a[j] = ld_coef(src, j, p);
    m2m_shift<PM>(a, cplx{cx[gc] - cx[gp], cy[gc] - cy[gp]});   // child - parent
#pragma unroll
    for (int j = 0; j <= PM; ++j) acc[j] = cadd(acc[j], a[j]);
  }
  double2* out = mult + gp * (p + 1);
#pragma unroll
  for (int j = 0; j <= PM; ++j)
    if (j <= p) out[j] = make_double2(acc[j].x, acc[j].y);
}

// --------------------------------------------------------------------------
// L2L (engine.py:126-129, operators.py:282-317): thread per child
template <int PM>
__global__ void __launch_bounds__(128)
k_l2l(int l, const double* __restrict__ cx, const double* __restrict__ cy, double2* local,
      int p) {
  // parent level l, child level l+1
  const long long c = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (c >= (1ll << (2 * (l + 1)))) return;
  const long long gc = level_base(l + 1) + c;
  const long long gp = level_base(l) + (c >> 2);
  const double2* src = local + gp * (p + 1);
  cplx b[PM + 1];
#pragma unroll
  for (int j = 0; j <= PM; ++j) b[j] = ld_coef(src, j, p);
  const cplx r{cx[gp] - cx[gc], cy[gp] - cy[gc]};                 // parent - child
  const double mag = numpy_cabs(r.x, r.y);
  if (mag >= SCALED_LO && mag <= SCALED_HI) {
    cplx pw = r;
#pragma unroll
    for (int j = 1; j <= PM; ++j) {
      b[j] = cmul(b[j], pw);
      pw = cmul(pw, r);
    }
#pragma unroll
    for (int k = 0; k <= PM; ++k)
#pragma unroll
      for (int j = PM - k; j < PM; ++j) b[j] = csub(b[j], b[j + 1]);
    const cplx inv = crcp(r);
    pw = inv;
#pragma unroll
    for (int j = 1; j <= PM; ++j) {
      b[j] = cmul(b[j], pw);
      pw = cmul(pw, inv);
    }
  } else {
#pragma unroll
    for (int k = 0; k <= PM; ++k)
#pragma unroll
      for (int j = PM - k; j < PM; ++j) b[j] = csub(b[j], cmul(r, b[j + 1]));
  }
  double2* dst = local + gc * (p + 1);
#pragma unroll
  for (int j = 0; j <= PM; ++j)
    if (j <= p) {
      double2 v = dst[j];
      dst[j] = make_double2(v.x + b[j].x, v.y + b[j].y);
    }
}

// --------------------------------------------------------------------------
// M2L (engine.py:103-123, operators.py:320-351).  All levels in one launch:
// the weak lists form one global CSR sorted by (target, source), so the pair
// list is flat.  One thread per pair computes the full (p+1)-term cascade in
// registers; a warp takes 32 consecutive pairs and sums them per target with a
// segmented shuffle scan (deterministic tree order).  Targets whose pairs sit
// inside one warp are updated in place (exclusive ownership, no atomics);
// targets spanning warps leave ordered partials that k_m2l_fixup folds in.
template <int PM>
__global__ void __launch_bounds__(128)
k_m2l(const int* __restrict__ total_ptr, const int* __restrict__ w_src,
      const int* __restrict__ w_tgt, const double* __restrict__ cx,
      const double* __restrict__ cy, const double2* __restrict__ mult, double2* local,
      double2* partials, unsigned char* item_flags, int p, DevStatus* st) {
  if (lists_overflowed(st)) return;
  const long long npairs = *total_ptr;
  const long long nitems = (npairs + 31) >> 5;
  const int lane = threadIdx.x & 31;
  const long long warps_total = ((long long)gridDim.x * blockDim.x) >> 5;
  for (long long item = (blockIdx.x * (long long)blockDim.x + threadIdx.x) >> 5; item < nitems;
       item += warps_total) {
    const long long i = item * 32 + lane;
    const bool valid = i < npairs;
    const int t = valid ? w_tgt[i] : -1;
    cplx c[PM + 1];
    if (valid) {
      const int s = w_src[i];
      const cplx rho{cx[s] - cx[t], cy[s] - cy[t]};            // source - target
      const bool sing = rho.x == 0.0 && rho.y == 0.0;
      if (sing) atomicOr(&st->flags, ST_M2L_SINGULAR);
      const cplx inv = sing ? cplx{0.0, 0.0} : crcp(rho);
      const double2* a = mult + (long long)s * (p + 1);
      // prescale c_{j-1} = a_j (-1)^j / rho^j  (operators.py:334-338)
      cplx pw = inv;
#pragma unroll
      for (int k = 1; k <= PM; ++k) {
        const cplx v = cmul(ld_coef(a, k, p), pw);
        c[k - 1] = (k & 1) ? cplx{-v.x, -v.y} : v;
        pw = cmul(pw, inv);
      }
      c[PM] = cplx{0.0, 0.0};
      // pass 1, old-value slices (operators.py:339-341)
#pragma unroll
      for (int k = 2; k <= PM; ++k)
#pragma unroll
        for (int j = PM - k; j < PM; ++j) c[j] = cadd(c[j], c[j + 1]);
      // pass 2, new-value cascade (operators.py:342-344)
#pragma unroll
      for (int k = PM; k >= 1; --k)
#pragma unroll
        for (int j = k; j <= PM; ++j) c[j] = cadd(c[j], c[j - 1]);
      // postscale b_j = c_j / rho^j (operators.py:349-350)
      pw = inv;
#pragma unroll
      for (int j = 1; j <= PM; ++j) {
        c[j] = cmul(c[j], pw);
        pw = cmul(pw, inv);
      }
    } else {
#pragma unroll
      for (int j = 0; j <= PM; ++j) c[j] = cplx{0.0, 0.0};
    }
    // segmented inclusive scan over lanes keyed by target
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
      const int tu = __shfl_up_sync(0xffffffffu, t, d);
      const bool take = lane >= d && tu == t;
#pragma unroll
      for (int j = 0; j <= PM; ++j) {
        const double ux = __shfl_up_sync(0xffffffffu, c[j].x, d);
        const double uy = __shfl_up_sync(0xffffffffu, c[j].y, d);
        if (take) { c[j].x += ux; c[j].y += uy; }
      }
    }
    const int tn = __shfl_down_sync(0xffffffffu, t, 1);
    const int t0 = __shfl_sync(0xffffffffu, t, 0);
    bool seg_end;
    bool ends_after = false;
    if (lane == 31) {
      ends_after = valid && i + 1 < npairs && w_tgt[i + 1] == t;
      seg_end = valid;
    } else {
      seg_end = valid && tn != t;
    }
    if (seg_end) {
      const bool starts_before = (t == t0) && item > 0 && w_tgt[item * 32 - 1] == t;
      if (!starts_before && !ends_after) {
        double2* dst = local + (long long)t * (p + 1);
#pragma unroll
        for (int j = 0; j <= PM; ++j)
          if (j <= p) {
            double2 v = dst[j];
            dst[j] = make_double2(v.x + c[j].x, v.y + c[j].y);
          }
      } else {
        const int slot = starts_before ? 0 : 1;
        double2* dst = partials + (item * 2 + slot) * (p + 1);
#pragma unroll
        for (int j = 0; j <= PM; ++j)
          if (j <= p) dst[j] = make_double2(c[j].x, c[j].y);
        unsigned char f = starts_before ? (ends_after ? 5 : 1) : 2;
        // first and last segment of one item are written by different lanes
        atomicOr(reinterpret_cast<unsigned int*>(item_flags + (item & ~3ll)),
                 (unsigned int)f << (8 * (item & 3)));
      }
    }
  }
}

__global__ void k_m2l_fixup(const int* __restrict__ total_ptr, const int* __restrict__ w_tgt,
                            const double2* __restrict__ partials,
                            const unsigned char* __restrict__ item_flags, double2* local, int p,
                            const DevStatus* st) {
  if (lists_overflowed(st)) return;
  const long long npairs = *total_ptr;
  const long long nitems = (npairs + 31) >> 5;
  for (long long w = blockIdx.x * (long long)blockDim.x + threadIdx.x; w < nitems;
       w += (long long)gridDim.x * blockDim.x) {
    if (!(item_flags[w] & 2)) continue;          // chain head: tail segment continues
    const int t = w_tgt[w * 32 + 31];
    double2* dst = local + (long long)t * (p + 1);
    for (int j = 0; j <= p; ++j) {
      double sx = partials[(w * 2 + 1) * (p + 1) + j].x;
      double sy = partials[(w * 2 + 1) * (p + 1) + j].y;
      for (long long u = w + 1; u < nitems; ++u) {
        const double2 v = partials[(u * 2 + 0) * (p + 1) + j];
        sx += v.x;
        sy += v.y;
        if (!(item_flags[u] & 4)) break;
      }
      const double2 o = dst[j];
      dst[j] = make_double2(o.x + sx, o.y + sy);
    }
  }
}

// --------------------------------------------------------------------------
// L2P + M2P (engine.py:132-160): warp per finest box, lanes over its points.
// phi = L2P, then += each m2p source in ascending order (operators.py:358-386)
template <int PM>
__global__ void __launch_bounds__(128)
k_l2p_m2p(int L, const int* __restrict__ eoff, const double2* __restrict__ eval_pos,
          const int* __restrict__ m_off, const int* __restrict__ m_idx,
          const double* __restrict__ cx, const double* __restrict__ cy,
          const double2* __restrict__ mult, const double2* __restrict__ local, double2* phi,
          int p, DevStatus* st) {
  const long long b = (blockIdx.x * (long long)blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (b >= (1ll << (2 * L)) || lists_overflowed(st)) return;
  const int e0 = eoff[b], e1 = eoff[b + 1];
  if (e0 == e1) return;
  const long long lb = level_base(L);
  const double x0 = cx[lb + b], y0 = cy[lb + b];
  const double2* bl = local + (lb + b) * (p + 1);
  cplx loc[PM + 1];
#pragma unroll
  for (int j = 0; j <= PM; ++j) loc[j] = ld_coef(bl, j, p);
  for (int e = e0 + lane; e < e1; e += 32) {
    const double2 y = eval_pos[e];
    cplx acc;
    if (L > 0) {
      const cplx w{y.x - x0, y.y - y0};
      acc = loc[PM];
#pragma unroll
      for (int j = PM - 1; j >= 0; --j) acc = cadd(cmul(acc, w), loc[j]);
    } else {
      acc = cplx{0.0, 0.0};
    }
    for (int q = m_off[b]; q < m_off[b + 1]; ++q) {
      const long long ga = lb + m_idx[q];
      const cplx u{y.x - cx[ga], y.y - cy[ga]};
      if (u.x == 0.0 && u.y == 0.0) {
        atomicOr(&st->flags, ST_M2P_SINGULAR);
        continue;
      }
      const cplx inv = crcp(u);
      const double2* a = mult + ga * (p + 1);
      cplx h = ld_coef(a, PM, p);
#pragma unroll
      for (int j = PM - 1; j >= 1; --j) h = cadd(cmul(h, inv), ld_coef(a, j, p));
      acc = cadd(acc, cmul(h, inv));
    }
    phi[e] = make_double2(acc.x, acc.y);
  }
}

inline unsigned nblk(long long n, int t) { return (unsigned)((n + t - 1) / t); }

// --------------------------------------------------------------------------
template <int PM>
struct Launch {
  static void upward(const TreeState& T, const ListState& Ls, ExpState& E, const int* offL,
                     DevStatus* dstat, cudaStream_t st) {
    const int L = T.L, p = E.p;
    if (L == 0) return;
    const long long nleaf = 1ll << (2 * L);
    k_p2m<PM><<<nblk(nleaf, 128), 128, 0, st>>>(L, offL, T.src_pos.as<double2>(),
                                                T.src_g.as<double>(), T.box_cx.as<double>(),
                                                T.box_cy.as<double>(), E.mult.as<double2>(), p);
    k_p2l<PM><<<nblk(nleaf, 128), 128, 0, st>>>(
        L, offL, Ls.p2l_off.as<int>(), Ls.p2l_idx.as<int>(), T.src_pos.as<double2>(),
        T.src_g.as<double>(), T.box_cx.as<double>(), T.box_cy.as<double>(),
        E.local.as<double2>(), p, dstat);
  }
  static void m2m(const TreeState& T, ExpState& E, cudaStream_t st) {
    for (int l = T.L - 1; l >= 1; --l)
      k_m2m<PM><<<nblk(1ll << (2 * l), 128), 128, 0, st>>>(l, T.box_cx.as<double>(),
                                                           T.box_cy.as<double>(),
                                                           E.mult.as<double2>(), E.p);
  }
  static void m2l(const TreeState& T, const ListState& Ls, ExpState& E, DevStatus* dstat,
                  cudaStream_t st) {
    const int L = T.L;
    if (L == 0) return;
    const int* total = Ls.weak_off.as<int>() + level_base(L + 1);
    const long long items = (Ls.cap_weak + 31) / 32;
    E.partials.reserve(sizeof(double2) * 2 * items * (E.p + 1));
    E.item_flags.reserve(((items + 4) & ~3ll) + 8);
    FMM_CUDA(cudaMemsetAsync(E.item_flags.p, 0, ((items + 4) & ~3ll) + 8, st));
    int dev = 0, sms = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    const unsigned grid = (unsigned)std::min<long long>(nblk(items * 32, 128), 16ll * sms);
    k_m2l<PM><<<grid, 128, 0, st>>>(total, Ls.weak_idx.as<int>(), Ls.weak_tgt.as<int>(),
                                    T.box_cx.as<double>(), T.box_cy.as<double>(),
                                    E.mult.as<double2>(), E.local.as<double2>(),
                                    E.partials.as<double2>(), E.item_flags.as<unsigned char>(),
                                    E.p, dstat);
    k_m2l_fixup<<<std::max(1u, std::min(1024u, nblk(items, 128))), 128, 0, st>>>(
        total, Ls.weak_tgt.as<int>(), E.partials.as<double2>(),
        E.item_flags.as<unsigned char>(), E.local.as<double2>(), E.p, dstat);
  }
  static void l2l(const TreeState& T, ExpState& E, cudaStream_t st) {
    for (int l = 1; l < T.L; ++l)
      k_l2l<PM><<<nblk(1ll << (2 * (l + 1)), 128), 128, 0, st>>>(
          l, T.box_cx.as<double>(), T.box_cy.as<double>(), E.local.as<double2>(), E.p);
  }
  static void l2p_m2p(const TreeState& T, const ListState& Ls, ExpState& E, DevStatus* dstat,
                      cudaStream_t st) {
    const int L = T.L;
    const long long nleaf = 1ll << (2 * L);
    k_l2p_m2p<PM><<<nblk(nleaf * 32, 128), 128, 0, st>>>(
        L, T.eval_leaf_off.as<int>(), T.eval_pos.as<double2>(), Ls.m2p_off.as<int>(),
        Ls.m2p_idx.as<int>(), T.box_cx.as<double>(), T.box_cy.as<double>(),
        E.mult.as<double2>(), E.local.as<double2>(), E.phi.as<double2>(), E.p, dstat);
  }
};

template <class F>
void dispatch_p(int p, F&& f) {
  if (p <= 4) f(std::integral_constant<int, 4>{});
  else if (p <= 8) f(std::integral_constant<int, 8>{});
  else if (p <= 12) f(std::integral_constant<int, 12>{});
  else if (p <= 16) f(std::integral_constant<int, 16>{});
  else if (p <= 17) f(std::integral_constant<int, 17>{});
  else if (p <= 20) f(std::integral_constant<int, 20>{});
  else if (p <= 24) f(std::integral_constant<int, 24>{});
  else if (p <= 30) f(std::integral_constant<int, 30>{});
  else if (p <= 32) f(std::integral_constant<int, 32>{});
  else if (p <= 40) f(std::integral_constant<int, 40>{});
  else if (p <= 48) f(std::integral_constant<int, 48>{});
  else f(std::integral_constant<int, 64>{});
}

}  // namespace

bool p_supported(int p) { return p >= 1 && p <= 64; }

void run_upward(const TreeState& T, const ListState& Ls, ExpState& E, const int* offL,
                DevStatus* dstat, cudaStream_t st) {
  dispatch_p(E.p, [&](auto pm) { Launch<decltype(pm)::value>::upward(T, Ls, E, offL, dstat, st); });
}
void run_m2m(const TreeState& T, ExpState& E, cudaStream_t st) {
  dispatch_p(E.p, [&](auto pm) { Launch<decltype(pm)::value>::m2m(T, E, st); });
}
void run_m2l(const TreeState& T, const ListState& Ls, ExpState& E, DevStatus* dstat,
             cudaStream_t st) {
  dispatch_p(E.p, [&](auto pm) { Launch<decltype(pm)::value>::m2l(T, Ls, E, dstat, st); });
}
void run_l2l(const TreeState& T, ExpState& E, DevStatus* dstat, cudaStream_t st) {
  (void)dstat;
  dispatch_p(E.p, [&](auto pm) { Launch<decltype(pm)::value>::l2l(T, E, st); });
}
void run_l2p_m2p(const TreeState& T, const ListState& Ls, ExpState& E, DevStatus* dstat,
                 cudaStream_t st) {
  dispatch_p(E.p, [&](auto pm) { Launch<decltype(pm)::value>::l2p_m2p(T, Ls, E, dstat, st); });
}

}  // namespace fmm
