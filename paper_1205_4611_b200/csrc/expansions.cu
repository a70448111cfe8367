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
#include <cstdlib>
#include <string>

#include "engine.h"

namespace fmm {

namespace {

constexpr double SCALED_LO = 1e-12, SCALED_HI = 1e12;   // operators.py:168-169
// M2L variant: 0 = thread per pair, 1 = lane pair per pair over a flat pair
// list, 2 = lane pair per pair, one warp per target (default);
// FMM2D_M2L=pair|split|target overrides for A/B measurements
int m2l_variant() {
  static int v = [] {
    const char* e = getenv("FMM2D_M2L");
    if (e && std::string(e) == "pair") return 0;
    if (e && std::string(e) == "split") return 1;
    return 2;
  }();
  return v;
}

#ifndef M2L_MIN_BLOCKS
#define M2L_MIN_BLOCKS 4
#endif

// branch-free lane-dependent selection: m all ones -> a, zero -> b
__device__ __forceinline__ double dsel(double a, double b, unsigned long long m) {
  const unsigned long long x = __double_as_longlong(a), y = __double_as_longlong(b);
  return __longlong_as_double((x & m) | (y & ~m));
}
__device__ __forceinline__ double dxor(double a, unsigned long long s) {
  return __longlong_as_double(__double_as_longlong(a) ^ s);
}

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

// P2L (engine.py:85-93, operators.py:209-224): one warp per target leaf, lanes
// over the particles of its p2l source boxes (ascending), butterfly reduction
template <int PM>
__global__ void __launch_bounds__(128)
k_p2l(int L, const int* __restrict__ offL, const int* __restrict__ l_off,
      const int* __restrict__ l_idx, const double2* __restrict__ src_pos,
      const double* __restrict__ src_g, const double* __restrict__ cx,
      const double* __restrict__ cy, double2* local, int p, DevStatus* st) {
  const long long b = (blockIdx.x * (long long)blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (b >= (1ll << (2 * L)) || lists_overflowed(st)) return;
  const long long lb = level_base(L);
  double2* out = local + (lb + b) * (p + 1);
  const int q0 = l_off[b], q1 = l_off[b + 1];
  if (q0 == q1) {                    // no p2l sources: local starts at zero
    for (int j = lane; j <= p; j += 32) out[j] = make_double2(0.0, 0.0);
    return;
  }
  const double x0 = cx[lb + b], y0 = cy[lb + b];
  cplx acc[PM + 1];
#pragma unroll
  for (int j = 0; j <= PM; ++j) acc[j] = cplx{0.0, 0.0};
  for (int q = q0; q < q1; ++q) {
    const int a = l_idx[q];
    for (int i = offL[a] + lane; i < offL[a + 1]; i += 32) {
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
        acc[k] = cadd(acc[k], w);
        w = cmul(w, inv);
      }
    }
  }
#pragma unroll
  for (int j = 0; j <= PM; ++j) {
#pragma unroll
    for (int d = 16; d; d >>= 1) {
      acc[j].x += __shfl_xor_sync(0xffffffffu, acc[j].x, d);
      acc[j].y += __shfl_xor_sync(0xffffffffu, acc[j].y, d);
    }
    if (j <= p && (j & 31) == lane) out[j] = make_double2(acc[j].x, acc[j].y);
  }
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
__global__ void __launch_bounds__(128, M2L_MIN_BLOCKS)
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

// Same M2L with a lane PAIR per interaction: the cascades are real-linear, so
// lane 2i carries the real parts and lane 2i+1 the imaginary parts of pair i;
// only the pre/post scalings mix them (one shuffle per coefficient).  Half
// the registers of the thread-per-pair form, so twice the resident warps to
// hide FP64 and L2 latency.  16 pairs per warp item.
// Target-owned M2L (default).  One warp per target box walks the target's
// weak list in chunks of 16 pairs; lane pair (2i, 2i+1) carries the real /
// imaginary part of pair i (the cascades of operators.py:339-344 are
// real-linear).  Each lane accumulates its pairs in order, then a fixed xor
// butterfly over the 16 lane pairs folds them and the target row is updated
// once -- no partials, no fixup, no atomics.
template <int PM>
__global__ void __launch_bounds__(128)
k_m2l_target(long long nbox, const int* __restrict__ woff, const int* __restrict__ w_src,
             const double* __restrict__ cx, const double* __restrict__ cy,
             const double2* __restrict__ mult, double2* local, int p, DevStatus* st) {
  if (lists_overflowed(st)) return;
  const int lane = threadIdx.x & 31, h = lane & 1, pl = lane >> 1;
  const unsigned long long hm = h ? ~0ull : 0ull;
  const unsigned long long neg0 = h ? 0ull : 0x8000000000000000ull;
  const long long nwarps = ((long long)gridDim.x * blockDim.x) >> 5;
  for (long long t = (blockIdx.x * (long long)blockDim.x + threadIdx.x) >> 5; t < nbox;
       t += nwarps) {
    const int q0 = woff[t], q1 = woff[t + 1];
    if (q0 == q1) continue;
    const double tx = cx[t], ty = cy[t];
    double acc[PM + 1];
#pragma unroll
    for (int j = 0; j <= PM; ++j) acc[j] = 0.0;
    bool sing_any = false;
    for (int base = q0; base < q1; base += 16) {
      const int q = base + pl;
      const bool valid = q < q1;
      const int s = valid ? w_src[q] : (int)t;
      const cplx rho{cx[s] - tx, cy[s] - ty};                    // source - target
      const bool sing = valid && rho.x == 0.0 && rho.y == 0.0;
      sing_any |= sing;
      const cplx inv = (valid && !sing) ? crcp(rho) : cplx{0.0, 0.0};
      const double qx = -inv.x, qy = -inv.y;                     // q = -1/rho
      const double2* a = mult + (long long)s * (p + 1);
      double c[PM + 1];
      {   // c_{k-1} = (a_k q^k)_h ; the lane pair shares the power sequence
        double own = dsel(qy, qx, hm);
#pragma unroll
        for (int k = 1; k <= PM; ++k) {
          const double part = __shfl_xor_sync(0xffffffffu, own, 1);
          const double ps = dxor(part, neg0);
          const cplx ak = ld_coef(a, k, p);
          c[k - 1] = fma(ak.x, own, ak.y * ps);
          own = fma(ps, qy, own * qx);
        }
        c[PM] = 0.0;
      }
#pragma unroll
      for (int k = 2; k <= PM; ++k)               // pass 1, old values (operators.py:339-341)
#pragma unroll
        for (int j = PM - k; j < PM; ++j) c[j] += c[j + 1];
#pragma unroll
      for (int k = PM; k >= 1; --k)               // pass 2, new values (operators.py:342-344)
#pragma unroll
        for (int j = k; j <= PM; ++j) c[j] += c[j - 1];
      {   // b_j = c_j / rho^j = c_j (-q)^j (operators.py:349-350)
        acc[0] += c[0];
        double own = dsel(qy, qx, hm);
#pragma unroll
        for (int j = 1; j <= PM; ++j) {
          const double pp = __shfl_xor_sync(0xffffffffu, own, 1);
          const double cp = __shfl_xor_sync(0xffffffffu, c[j], 1);
          const double A = dsel(cp, c[j], hm);
          const double B = dsel(c[j], dxor(cp, 0x8000000000000000ull), hm);
          const double v = fma(A, own, B * pp);
          acc[j] += (j & 1) ? -v : v;
          own = fma(dxor(pp, neg0), qy, own * qx);
        }
      }
    }
    if (__any_sync(0xffffffffu, sing_any) && lane == 0) atomicOr(&st->flags, ST_M2L_SINGULAR);
    // fold the 16 lane pairs (same component), fixed butterfly order
#pragma unroll
    for (int j = 0; j <= PM; ++j) {
#pragma unroll
      for (int d = 2; d < 32; d <<= 1) acc[j] += __shfl_xor_sync(0xffffffffu, acc[j], d);
    }
    double* row = reinterpret_cast<double*>(local + t * (p + 1));
#pragma unroll
    for (int j = 0; j <= PM; ++j)
      if (j <= p && (j & 15) == pl) row[2 * j + h] += acc[j];
  }
}

// one coalesced row update of a target segment's sum (coefficient j, part comp)
__device__ __forceinline__ void m2l_emit(double2* local, double2* partials,
                                         unsigned char* item_flags, long long item, int p, int t,
                                         int j, int comp, double v, bool starts_before,
                                         bool ends_after) {
  if (!starts_before && !ends_after) {
    double* dst = reinterpret_cast<double*>(local + (long long)t * (p + 1)) + 2 * j + comp;
    *dst += v;
    return;
  }
  const int slot = starts_before ? 0 : 1;
  reinterpret_cast<double*>(partials + (item * 2 + slot) * (p + 1))[2 * j + comp] = v;
  if (j == 0 && comp == 0) {
    const unsigned f = starts_before ? (ends_after ? 5u : 1u) : 2u;
    atomicOr(reinterpret_cast<unsigned int*>(item_flags + (item & ~3ll)), f << (8 * (item & 3)));
  }
}

template <int PM>
__global__ void __launch_bounds__(128)
k_m2l_split(const int* __restrict__ total_ptr, const int* __restrict__ w_src,
            const int* __restrict__ w_tgt, const double* __restrict__ cx,
            const double* __restrict__ cy, const double2* __restrict__ mult, double2* local,
            double2* partials, unsigned char* item_flags, int p, DevStatus* st) {
  if (lists_overflowed(st)) return;
  extern __shared__ double red[];          // 4 warps x 32 lanes x RS doubles
  __shared__ int s_tgt[4][16];
  constexpr int RS = (PM + 1) | 1;         // odd row stride: conflict-free 8-byte banks
  const long long npairs = *total_ptr;
  const long long nitems = (npairs + 15) >> 4;
  const int lane = threadIdx.x & 31, h = lane & 1, pl = lane >> 1;
  const long long warps_total = ((long long)gridDim.x * blockDim.x) >> 5;
  for (long long item = (blockIdx.x * (long long)blockDim.x + threadIdx.x) >> 5; item < nitems;
       item += warps_total) {
    const long long i = item * 16 + pl;
    const bool valid = i < npairs;
    // padding lanes run the same code on box 0 with a zero reciprocal
    const int t = valid ? w_tgt[i] : -1;
    const int s = valid ? w_src[i] : 0;
    const int tt = valid ? t : 0;
    const cplx rho{cx[s] - cx[tt], cy[s] - cy[tt]};               // source - target
    const bool sing = valid && rho.x == 0.0 && rho.y == 0.0;
    if (__any_sync(0xffffffffu, sing) && lane == 0) atomicOr(&st->flags, ST_M2L_SINGULAR);
    const cplx inv = (valid && !sing) ? crcp(rho) : cplx{0.0, 0.0};
    // q = -1/rho: q^k = (-1)^k / rho^k.  The lane pair shares the power
    // sequence: each lane advances its own component, the partner's comes by
    // shuffle, so a complex power costs 2 FP64 ops per lane instead of 4.
    const double qx = -inv.x, qy = -inv.y;
    const double2* a = mult + (long long)s * (p + 1);
    double c[PM + 1];
    // lane-dependent choices as bit masks (a select on h would make the
    // compiler unswitch the unrolled loops and serialise both lane halves)
    const unsigned long long hm = h ? ~0ull : 0ull;            // all ones on the imag lane
    const unsigned long long neg0 = h ? 0ull : 0x8000000000000000ull;
    {
      double own = dsel(qy, qx, hm);                               // component h of q^1
#pragma unroll
      for (int k = 1; k <= PM; ++k) {
        const double part = __shfl_xor_sync(0xffffffffu, own, 1);
        const double ps = dxor(part, neg0);                        // partner, signed
        const cplx ak = ld_coef(a, k, p);
        c[k - 1] = fma(ak.x, own, ak.y * ps);                      // (a_k q^k)_h
        own = fma(ps, qy, own * qx);                               // (q^{k+1})_h
      }
      c[PM] = 0.0;
    }
#pragma unroll
    for (int k = 2; k <= PM; ++k)                 // pass 1, old values (operators.py:339-341)
#pragma unroll
      for (int j = PM - k; j < PM; ++j) c[j] += c[j + 1];
#pragma unroll
    for (int k = PM; k >= 1; --k)                 // pass 2, new values (operators.py:342-344)
#pragma unroll
      for (int j = k; j <= PM; ++j) c[j] += c[j - 1];
    {   // postscale b_j = c_j / rho^j = c_j (-q)^j (operators.py:349-350)
      double own = dsel(qy, qx, hm);
#pragma unroll
      for (int j = 1; j <= PM; ++j) {
        const double pp = __shfl_xor_sync(0xffffffffu, own, 1);    // partner of q^j
        const double cp = __shfl_xor_sync(0xffffffffu, c[j], 1);   // partner of c_j
        // (c q^j)_h  h=0: c_o w_o - c_p w_p ;  h=1: c_p w_o + c_o w_p
        const double A = dsel(cp, c[j], hm);
        const double B = dsel(c[j], dxor(cp, 0x8000000000000000ull), hm);
        const double v = fma(A, own, B * pp);
        c[j] = (j & 1) ? -v : v;
        own = fma(dxor(pp, neg0), qy, own * qx);
      }
    }
    // per-target sums through SMEM: every lane parks its row, then lane r
    // owns coefficient r>>1 (component r&1) and walks the 16 pairs in order,
    // emitting one coalesced row update per target segment
    double* row = red + ((threadIdx.x >> 5) * 32 + lane) * RS;
#pragma unroll
    for (int j = 0; j <= PM; ++j) row[j] = c[j];
    int* wt = s_tgt[threadIdx.x >> 5];
    if (h == 0) wt[pl] = t;
    const int t0 = __shfl_sync(0xffffffffu, t, 0);
    const bool first_cont = item > 0 && t0 >= 0 && w_tgt[item * 16 - 1] == t0;
    const long long last = min(item * 16 + 15, npairs - 1);
    const int t_last = w_tgt[last];
    const bool last_cont = last + 1 < npairs && w_tgt[last + 1] == t_last;
    __syncwarp();
    const double* wred = red + (threadIdx.x >> 5) * 32 * RS;
    for (int r = lane; r < 2 * (p + 1); r += 32) {
      const int j = r >> 1, comp = r & 1;
      double acc = 0.0;
      int seg_t = wt[0], seg_first = 1;
      for (int q = 0; q < 16; ++q) {
        const int tq = wt[q];
        if (tq < 0) break;
        if (tq != seg_t) {     // segment ends before pair q
          m2l_emit(local, partials, item_flags, item, p, seg_t, j, comp, acc,
                   seg_first && first_cont, false);
          seg_t = tq;
          seg_first = 0;
          acc = 0.0;
        }
        acc += wred[(2 * q + comp) * RS + j];
      }
      if (seg_t >= 0)
        m2l_emit(local, partials, item_flags, item, p, seg_t, j, comp, acc,
                 seg_first && first_cont, last_cont);
    }
    __syncwarp();
  }
}

// ordered fold of the partial sums of targets whose pairs span several warp
// items: one warp per item, lanes over coefficients (coalesced rows)
__global__ void k_m2l_fixup(const int* __restrict__ total_ptr, const int* __restrict__ w_tgt,
                            const double2* __restrict__ partials,
                            const unsigned char* __restrict__ item_flags, double2* local, int p,
                            int item_pairs, const DevStatus* st) {
  if (lists_overflowed(st)) return;
  const long long npairs = *total_ptr;
  const long long nitems = (npairs + item_pairs - 1) / item_pairs;
  const int lane = threadIdx.x & 31;
  const long long nwarps = ((long long)gridDim.x * blockDim.x) >> 5;
  for (long long w = (blockIdx.x * (long long)blockDim.x + threadIdx.x) >> 5; w < nitems;
       w += nwarps) {
    if (!(item_flags[w] & 2)) continue;          // chain head: its tail segment continues
    const int t = w_tgt[w * item_pairs + item_pairs - 1];
    double2* dst = local + (long long)t * (p + 1);
    for (int j = lane; j <= p; j += 32) {
      double2 s = partials[(w * 2 + 1) * (p + 1) + j];
      for (long long u = w + 1; u < nitems; ++u) {
        const double2 v = partials[(u * 2 + 0) * (p + 1) + j];
        s.x += v.x;
        s.y += v.y;
        if (!(item_flags[u] & 4)) break;
      }
      const double2 o = dst[j];
      dst[j] = make_double2(o.x + s.x, o.y + s.y);
    }
  }
}

// --------------------------------------------------------------------------
// L2P + M2P (engine.py:132-160): one thread per evaluation point (tree order),
// its leaf from the tree build.  phi = L2P (Horner in y - z0), then += each
// m2p source in ascending order (operators.py:358-386).  Coefficients stream
// from L1/L2 (the points of one leaf share them), so no register arrays.
template <int PM>
__global__ void __launch_bounds__(128)
k_l2p_m2p(long long m, int L, const unsigned* __restrict__ leaf,
          const double2* __restrict__ eval_pos, const int* __restrict__ m_off,
          const int* __restrict__ m_idx, const double* __restrict__ cx,
          const double* __restrict__ cy, const double2* __restrict__ mult,
          const double2* __restrict__ local, double2* phi, int p, DevStatus* st) {
  const long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (e >= m || lists_overflowed(st)) return;
  const long long lb = level_base(L);
  const long long b = leaf[e];
  const double2 y = eval_pos[e];
  const cplx w{y.x - cx[lb + b], y.y - cy[lb + b]};
  const double2* bl = local + (lb + b) * (p + 1);
  cplx c[PM + 1];
#pragma unroll
  for (int j = 0; j <= PM; ++j) c[j] = ld_coef(bl, j, p);   // all loads in flight at once
  cplx acc = c[PM];
#pragma unroll
  for (int j = PM - 1; j >= 0; --j) acc = cadd(cmul(acc, w), c[j]);
  for (int q = m_off[b]; q < m_off[b + 1]; ++q) {
    const long long ga = lb + m_idx[q];
    const cplx u{y.x - cx[ga], y.y - cy[ga]};
    if (u.x == 0.0 && u.y == 0.0) {
      atomicOr(&st->flags, ST_M2P_SINGULAR);
      continue;
    }
    const cplx inv = crcp(u);
    const double2* a = mult + ga * (p + 1);
#pragma unroll
    for (int j = 1; j <= PM; ++j) c[j] = ld_coef(a, j, p);
    cplx h = c[PM];
#pragma unroll
    for (int j = PM - 1; j >= 1; --j) h = cadd(cmul(h, inv), c[j]);
    acc = cadd(acc, cmul(h, inv));
  }
  phi[e] = make_double2(acc.x, acc.y);
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
    note_launch();
    k_p2m<PM><<<nblk(nleaf, 128), 128, 0, st>>>(L, offL, T.src_pos.as<double2>(),
                                                T.src_g.as<double>(), T.box_cx.as<double>(),
                                                T.box_cy.as<double>(), E.mult.as<double2>(), p);
    note_launch();
    k_p2l<PM><<<nblk(nleaf * 32, 128), 128, 0, st>>>(
        L, offL, Ls.p2l_off.as<int>(), Ls.p2l_idx.as<int>(), T.src_pos.as<double2>(),
        T.src_g.as<double>(), T.box_cx.as<double>(), T.box_cy.as<double>(),
        E.local.as<double2>(), p, dstat);
  }
  static void m2m(const TreeState& T, ExpState& E, cudaStream_t st) {
    for (int l = T.L - 1; l >= 1; --l) {
      note_launch();
      k_m2m<PM><<<nblk(1ll << (2 * l), 128), 128, 0, st>>>(l, T.box_cx.as<double>(),
                                                           T.box_cy.as<double>(),
                                                           E.mult.as<double2>(), E.p);
    }
  }
  static void m2l(const TreeState& T, const ListState& Ls, ExpState& E, DevStatus* dstat,
                  cudaStream_t st) {
    const int L = T.L;
    if (L == 0) return;
    const int* total = Ls.weak_off.as<int>() + level_base(L + 1);
    if (m2l_variant() == 2) {
      int dev = 0, sms = 148;
      cudaGetDevice(&dev);
      cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
      const long long nbox = level_base(L + 1);
      const unsigned grid = (unsigned)std::min<long long>(nblk(nbox * 32, 128), 64ll * sms);
      note_launch();
      k_m2l_target<PM><<<grid, 128, 0, st>>>(nbox, Ls.weak_off.as<int>(), Ls.weak_idx.as<int>(),
                                             T.box_cx.as<double>(), T.box_cy.as<double>(),
                                             E.mult.as<double2>(), E.local.as<double2>(), E.p,
                                             dstat);
      return;
    }
    const bool split = m2l_variant() == 1;
    const int item_pairs = split ? 16 : 32;
    const long long items = (Ls.cap_weak + item_pairs - 1) / item_pairs;
    E.partials.reserve(sizeof(double2) * 2 * items * (E.p + 1));
    E.item_flags.reserve(((items + 4) & ~3ll) + 8);
    FMM_CUDA(cudaMemsetAsync(E.item_flags.p, 0, ((items + 4) & ~3ll) + 8, st));
    int dev = 0, sms = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    const unsigned grid = (unsigned)std::min<long long>(nblk(items * 32, 128), 32ll * sms);
    note_launch();
    if (split) {
      constexpr int RS = (PM + 1) | 1;
      const int smem = 128 * RS * (int)sizeof(double);
      if (smem > 48 * 1024)
        FMM_CUDA(cudaFuncSetAttribute(k_m2l_split<PM>,
                                      cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
      k_m2l_split<PM><<<grid, 128, smem, st>>>(total, Ls.weak_idx.as<int>(), Ls.weak_tgt.as<int>(),
                                            T.box_cx.as<double>(), T.box_cy.as<double>(),
                                            E.mult.as<double2>(), E.local.as<double2>(),
                                            E.partials.as<double2>(),
                                            E.item_flags.as<unsigned char>(), E.p, dstat);
    } else {
      k_m2l<PM><<<grid, 128, 0, st>>>(total, Ls.weak_idx.as<int>(), Ls.weak_tgt.as<int>(),
                                      T.box_cx.as<double>(), T.box_cy.as<double>(),
                                      E.mult.as<double2>(), E.local.as<double2>(),
                                      E.partials.as<double2>(), E.item_flags.as<unsigned char>(),
                                      E.p, dstat);
    }
    note_launch();
    k_m2l_fixup<<<std::max(1u, std::min(4096u, nblk(items * 32, 128))), 128, 0, st>>>(
        total, Ls.weak_tgt.as<int>(), E.partials.as<double2>(),
        E.item_flags.as<unsigned char>(), E.local.as<double2>(), E.p, item_pairs, dstat);
  }
  static void l2l(const TreeState& T, ExpState& E, cudaStream_t st) {
    for (int l = 1; l < T.L; ++l) {
      note_launch();
      k_l2l<PM><<<nblk(1ll << (2 * (l + 1)), 128), 128, 0, st>>>(
          l, T.box_cx.as<double>(), T.box_cy.as<double>(), E.local.as<double2>(), E.p);
    }
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
  if (T.L == 0) {   // a single box: no expansions (engine.py:257)
    FMM_CUDA(cudaMemsetAsync(E.phi.p, 0, sizeof(double2) * T.m, st));
    return;
  }
  dispatch_p(E.p, [&](auto pm) {
    note_launch();
    k_l2p_m2p<decltype(pm)::value><<<nblk(T.m, 128), 128, 0, st>>>(
        T.m, T.L, T.eval_leaf, T.eval_pos.as<double2>(), Ls.m2p_off.as<int>(),
        Ls.m2p_idx.as<int>(), T.box_cx.as<double>(), T.box_cy.as<double>(),
        E.mult.as<double2>(), E.local.as<double2>(), E.phi.as<double2>(), E.p, dstat);
  });
}

}  // namespace fmm
