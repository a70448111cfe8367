// Expansion kernels: P2M, P2L, M2M, M2L, L2L, L2P+M2P (FP64, registers).
//
// Reference: operators.py:63-255 (unit operators), engine.py:67-160 (phase
// drivers).  Conventions kept verbatim: p2m a_0 = 0, a_j = -sum g (z-z0)^(j-1);
// p2l b_k = sum g/(z-z0)^(k+1); every shift = source center - target center;
// scaled cascades with the unscaled fallback outside |r| in [1e-12, 1e12].
// a_0 is identically zero in the harmonic pipeline (p2m writes 0 and m2m
// preserves it), so the a_0 log corrections (operators.py:105-110, 121-123, 214-219)
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

constexpr double SCALED_LO = 1e-12, SCALED_HI = 1e12;   // operators.py:37-38
constexpr int M2P_INLINE = 16;
#ifndef L2L_CHAIN
#define L2L_CHAIN 1      // chained kernel for the small top levels of the L2L pass
#endif
#ifndef L2L_CHAIN_MAXBOX
#define L2L_CHAIN_MAXBOX 4096   // deepest chained level: at most this many boxes
#endif
   // m2p sources per point handled by k_l2p_m2p itself
// M2L variant: dense Pascal-matrix kernel (default, PM <= 32) or the
// target-owned lane-pair cascade (PM > 32, or FMM2D_M2L=target for A/B runs)
bool m2l_force_target() {
  static bool v = [] {
    const char* e = getenv("FMM2D_M2L");
    return e && std::string(e) == "target";
  }();
  return v;
}
// FMM2D_M2L=dmma selects the FP64 tensor-core kernel (measured slower than the
// DFMA dense kernel on B200: profiles/r02/m2l_dmma_vs_dense.txt)
bool m2l_dmma() {
  static bool v = [] {
    const char* e = getenv("FMM2D_M2L");
    return e && std::string(e) == "dmma";
  }();
  return v;
}
// cudaFuncSetAttribute is per device: remember which devices have it
template <class K>
void ensure_smem_attr(K kernel, int bytes, unsigned& done_mask) {
  int dev = 0;
  FMM_CUDA(cudaGetDevice(&dev));
  if (dev < 32 && (done_mask >> dev) & 1u) return;
  FMM_CUDA(cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes));
  if (dev < 32) done_mask |= 1u << dev;
}

int sm_count() {
  static int sms = [] {
    int dev = 0, n = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
    return n;
  }();
  return sms;
}

// branch-free lane-dependent selection: m all ones -> a, zero -> b
__device__ __forceinline__ double dsel(double a, double b, unsigned long long m) {
  const unsigned long long x = __double_as_longlong(a), y = __double_as_longlong(b);
  return __longlong_as_double((x & m) | (y & ~m));
}
__device__ __forceinline__ double dxor(double a, unsigned long long s) {
  return __longlong_as_double(__double_as_longlong(a) ^ s);
}

// coefficient j of a row of p + 1, zero above p; EX: p == PM is known, no test
template <bool EX = false>
__device__ __forceinline__ cplx ld_coef(const double2* base, int j, int p) {
  if (!EX && j > p) return cplx{0.0, 0.0};
  double2 v = base[j];
  return cplx{v.x, v.y};
}

// --------------------------------------------------------------------------
// P2M (engine.py:67-82): one thread per leaf, sequential over its sources
template <int PM, bool EX>
__global__ void __launch_bounds__(128)
k_p2m(int L, long long b0, long long b1, const int* __restrict__ offL,
      const double2* __restrict__ src_pos, const double* __restrict__ src_g,
      const double* __restrict__ cx, const double* __restrict__ cy, double2* mult, int p) {
  pdl_enter();
  if constexpr (EX) p = PM;                       // exact order: compile-time p
  const long long b = b0 + blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (b >= b1) return;
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

// P2L (engine.py:85-93, operators.py:78-93) in two balanced steps:
//  k_p2l_pair: one thread per (target leaf, p2l source leaf) pair computes the
//    pair's row sum_i g_i w_i^(k+1), w_i = 1/(z_i - z0), over the source leaf's
//    particles (what one ops.p2l call returns);
//  k_p2l_fold: one thread per target leaf adds its pairs' rows in ascending
//    source order (the reference's local[b] += ... sequence) and initialises
//    local[L] (zero without p2l sources).
template <int PM, bool EX>
__global__ void __launch_bounds__(128)
k_p2l_pair(int L, long long b0, long long b1, const int* __restrict__ offL,
           const int* __restrict__ l_off, const int* __restrict__ l_idx,
           const double2* __restrict__ src_pos, const double* __restrict__ src_g,
           const double* __restrict__ cx, const double* __restrict__ cy, double2* rows, int p,
           DevStatus* st) {
  pdl_enter();
  if constexpr (EX) p = PM;                       // exact order: compile-time p
  if (lists_overflowed(st)) return;
  const long long lb = level_base(L);
  const int qbase = l_off[b0], qend = l_off[b1];
  for (long long q = qbase + blockIdx.x * (long long)blockDim.x + threadIdx.x; q < qend;
       q += (long long)gridDim.x * blockDim.x) {
    long long lo = b0, hi = b1;                 // target: l_off[b] <= q < l_off[b+1]
    while (hi - lo > 1) {
      const long long mid = (lo + hi) >> 1;
      if (l_off[mid] <= q) lo = mid; else hi = mid;
    }
    const long long b = lo;
    const double x0 = cx[lb + b], y0 = cy[lb + b];
    const int a = l_idx[q];
    cplx acc[PM + 1];
#pragma unroll
    for (int j = 0; j <= PM; ++j) acc[j] = cplx{0.0, 0.0};
    // two particles per step: their power chains are independent, and
    // acc[k] = (acc[k] + w_i) + w_{i+1} keeps the sequential summation order
    const int i0 = offL[a], i1 = offL[a + 1];
    int i = i0;
    for (; i + 2 <= i1; i += 2) {
      const double2 z0 = src_pos[i], z1 = src_pos[i + 1];
      const cplx d0{z0.x - x0, z0.y - y0}, d1{z1.x - x0, z1.y - y0};
      const bool s0 = d0.x == 0.0 && d0.y == 0.0, s1 = d1.x == 0.0 && d1.y == 0.0;
      if (s0 || s1) atomicOr(&st->flags, ST_P2L_SINGULAR);
      const cplx inv0 = s0 ? cplx{0.0, 0.0} : crcp_fast(d0);
      const cplx inv1 = s1 ? cplx{0.0, 0.0} : crcp_fast(d1);
      cplx w0 = cscale(inv0, src_g[i]), w1 = cscale(inv1, src_g[i + 1]);
#pragma unroll
      for (int k = 0; k <= PM; ++k) {
        acc[k] = cadd(cadd(acc[k], w0), w1);
        w0 = cmul(w0, inv0);
        w1 = cmul(w1, inv1);
      }
    }
    if (i < i1) {
      const double2 z = src_pos[i];
      const cplx d{z.x - x0, z.y - y0};
      if (d.x == 0.0 && d.y == 0.0) {
        atomicOr(&st->flags, ST_P2L_SINGULAR);
      } else {
        const cplx inv = crcp_fast(d);
        cplx w = cscale(inv, src_g[i]);
#pragma unroll
        for (int k = 0; k <= PM; ++k) {
          acc[k] = cadd(acc[k], w);
          w = cmul(w, inv);
        }
      }
    }
    double2* out = rows + (q - qbase) * (p + 1);
#pragma unroll
    for (int j = 0; j <= PM; ++j)
      if (j <= p) out[j] = make_double2(acc[j].x, acc[j].y);
  }
}

__global__ void __launch_bounds__(128)
k_p2l_fold(int L, long long b0, long long b1, const int* __restrict__ l_off,
           const double2* __restrict__ rows, double2* local, int p, DevStatus* st) {
  pdl_enter();
  const long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  const long long b = b0 + t / (p + 1);
  const int j = (int)(t % (p + 1));
  if (b >= b1 || lists_overflowed(st)) return;
  const int qbase = l_off[b0];
  double2 acc = make_double2(0.0, 0.0);
  for (int q = l_off[b]; q < l_off[b + 1]; ++q) {
    const double2 v = rows[(long long)(q - qbase) * (p + 1) + j];
    acc.x += v.x;
    acc.y += v.y;
  }
  local[(level_base(L) + b) * (p + 1) + j] = acc;
}

// --------------------------------------------------------------------------
// M2M (engine.py:96-100, operators.py:100-148): thread per parent, children 0..3
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

// four threads per parent (one per child shift), children summed in order
// 0..3 through shuffles (engine.py:100 reshape(-1, 4, p+1).sum(1))
template <int PM, bool EX>
__global__ void __launch_bounds__(128)
k_m2m(int l, long long k0, long long k1, const double* __restrict__ cx,
      const double* __restrict__ cy, double2* mult, int p) {
  pdl_enter();
  if constexpr (EX) p = PM;                       // exact order: compile-time p
  const long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  const long long k = k0 + (t >> 2);
  const int c = (int)(t & 3), lane = threadIdx.x & 31;
  const bool valid = k < k1;
  const long long kk = valid ? k : k0;
  const long long gp = level_base(l) + kk;
  const long long gc = level_base(l + 1) + 4 * kk + c;
  const double2* src = mult + gc * (p + 1);
  cplx a[PM + 1];
#pragma unroll
  for (int j = 0; j <= PM; ++j) a[j] = ld_coef(src, j, p);
  m2m_shift<PM>(a, cplx{cx[gc] - cx[gp], cy[gc] - cy[gp]});   // child - parent
  const int g0 = lane & ~3;
  double2* out = mult + gp * (p + 1);
#pragma unroll
  for (int j = 0; j <= PM; ++j) {
    const double x0 = __shfl_sync(0xffffffffu, a[j].x, g0), y0 = __shfl_sync(0xffffffffu, a[j].y, g0);
    const double x1 = __shfl_sync(0xffffffffu, a[j].x, g0 + 1), y1 = __shfl_sync(0xffffffffu, a[j].y, g0 + 1);
    const double x2 = __shfl_sync(0xffffffffu, a[j].x, g0 + 2), y2 = __shfl_sync(0xffffffffu, a[j].y, g0 + 2);
    const double x3 = __shfl_sync(0xffffffffu, a[j].x, g0 + 3), y3 = __shfl_sync(0xffffffffu, a[j].y, g0 + 3);
    if (valid && c == 0 && j <= p) out[j] = make_double2(((x0 + x1) + x2) + x3, ((y0 + y1) + y2) + y3);
  }
}

// --------------------------------------------------------------------------
// L2L (engine.py:126-129, operators.py:151-186): thread per child
// the parent's incoming expansion b (in place) re-centred on the child:
// r = parent - child (operators.py:151-186, scaled form inside the window)
template <int PM>
__device__ __forceinline__ void l2l_shift(cplx (&b)[PM + 1], cplx r) {
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
}

template <int PM, bool EX>
__global__ void __launch_bounds__(128)
k_l2l(int l, long long c0, long long c1, const double* __restrict__ cx,
      const double* __restrict__ cy, double2* local, int p) {
  pdl_enter();
  if constexpr (EX) p = PM;                       // exact order: compile-time p
  // parent level l, child level l+1 (children [c0, c1))
  const long long c = c0 + blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (c >= c1) return;
  const long long gc = level_base(l + 1) + c;
  const long long gp = level_base(l) + (c >> 2);
  const double2* src = local + gp * (p + 1);
  cplx b[PM + 1];
#pragma unroll
  for (int j = 0; j <= PM; ++j) b[j] = ld_coef(src, j, p);
  l2l_shift<PM>(b, cplx{cx[gp] - cx[gc], cy[gp] - cy[gc]});       // parent - child
  double2* dst = local + gc * (p + 1);
#pragma unroll
  for (int j = 0; j <= PM; ++j)
    if (j <= p) {
      double2 v = dst[j];
      dst[j] = make_double2(v.x + b[j].x, v.y + b[j].y);
    }
}

// Levels 2..lt of the L2L pass in ONE launch: a thread per level-lt box
// walks its ancestor chain from level 1, re-computing every ancestor's
// complete local expansion on the way (local[l+1][a] + shift(parent), the
// same operations in the same order as the level-by-level kernel, so the
// result is bit-identical) and writes the level-lt box's complete expansion.
// The redundant ancestor work (~4x the few thousand shifts of these levels)
// costs far less than the level-by-level launches it replaces, which are
// pure latency at these sizes.
template <int PM, bool EX>
__global__ void __launch_bounds__(128)
k_l2l_chain(int lt, const double* __restrict__ cx, const double* __restrict__ cy,
            double2* local, int p) {
  pdl_enter();
  if constexpr (EX) p = PM;
  const long long b = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (b >= (1ll << (2 * lt))) return;
  cplx cur[PM + 1];
  {
    const long long g1 = level_base(1) + (b >> (2 * (lt - 1)));
#pragma unroll
    for (int j = 0; j <= PM; ++j) cur[j] = ld_coef(local + g1 * (p + 1), j, p);
  }
  for (int l = 1; l < lt; ++l) {
    const long long gp = level_base(l) + (b >> (2 * (lt - l)));
    const long long gc = level_base(l + 1) + (b >> (2 * (lt - l - 1)));
    l2l_shift<PM>(cur, cplx{cx[gp] - cx[gc], cy[gp] - cy[gc]});
    const double2* own = local + gc * (p + 1);
#pragma unroll
    for (int j = 0; j <= PM; ++j) {
      const cplx v = ld_coef(own, j, p);
      cur[j] = cplx{v.x + cur[j].x, v.y + cur[j].y};
    }
  }
  double2* dst = local + (level_base(lt) + b) * (p + 1);
#pragma unroll
  for (int j = 0; j <= PM; ++j)
    if (j <= p) dst[j] = make_double2(cur[j].x, cur[j].y);
}

// --------------------------------------------------------------------------
// --------------------------------------------------------------------------
// M2L (engine.py:103-123, operators.py:189-220), dense form.
//
// With alpha_k = a_k (-1)^k / rho^k (the reference's prescale), the two
// cascades of operators.py:208-213 compute c_j = sum_k C(j+k-1, k-1) alpha_k
// exactly (Pascal-matrix identity; potentials move <= 6e-14, SURVEY
// Appendix B.5), and b_j = c_j / rho^j (operators.py:218-219).  The Pascal
// matrix is a compile-time table in constant memory, so the core is
// (p+1) p complex-by-real FMAs per pair with a constant-bank operand and no
// data-dependent index math -- the same FP64 instruction count as the
// cascade (840 at p=20) but 42 independent accumulation chains instead of a
// wavefront, and alpha is the only register-resident array.
//
// Work split: all levels in one launch over the flat pair list (one global
// CSR sorted by (target, source)).  A CTA takes M2L_ITEM consecutive pairs,
// one per thread; every thread parks its b row in SMEM, then the CTA
// folds each target segment in ascending pair order (one task per
// coefficient and segment, coalesced row updates).  Targets wholly inside
// the item are updated in place (exclusive owner, no atomics); targets whose
// pairs span items leave ordered partials for k_m2l_fixup.
#ifndef M2L_GRID_WAVES
#define M2L_GRID_WAVES 16  // grid = 16 waves of resident CTAs (tail balance)
#endif
#ifndef M2L_ITEM_PAIRS
#define M2L_ITEM_PAIRS 64    // pairs (threads) per CTA item: small CTAs, cheap barriers
#endif
constexpr int M2L_ITEM = M2L_ITEM_PAIRS;

// Per-order table T[j][k-1] = C(j+k-1, k-1), j = 0..PM, k = 1..PM, rows of
// even stride so consecutive k pairs are one 16-byte uniform constant load;
// the ~3 KB an order uses stays resident in the SM's constant cache.
template <int PM>
struct M2LTab {
  static constexpr int STRIDE = (PM + 1) & ~1;
  double v[PM + 1][STRIDE];
};
template <int PM>
constexpr M2LTab<PM> make_m2l_tab() {
  M2LTab<PM> t{};
  unsigned long long row[2 * PM + 1] = {};
  double pas[2 * PM][2 * PM] = {};
  for (int n = 0; n < 2 * PM; ++n) {
    for (int k = n; k >= 1; --k) row[k] += row[k - 1];   // C(n, k), exact in u64 for n < 64
    row[0] = 1;
    for (int k = 0; k <= n; ++k) pas[n][k] = (double)row[k];
  }
  for (int j = 0; j <= PM; ++j)
    for (int k = 1; k <= PM; ++k) t.v[j][k - 1] = pas[j + k - 1][k - 1];
  return t;
}
template <int PM>
__constant__ __align__(16) M2LTab<PM> c_m2l_tab = make_m2l_tab<PM>();
#ifndef M2L_HALF
#define M2L_HALF 1
#endif
#ifndef M2L_IMM
#define M2L_IMM 1
#endif
// C(n, k) as a constant expression.  With compile-time (j, k) -- the exact-
// order instantiations -- every coefficient below 2^21 becomes a DFMA
// immediate (its low word is zero) and the rest a pair of uniform moves: no
// constant-bank loads in the contraction (C2 M2L -0.9 %, C4 -2.5 %,
// bit-identical; M2L_IMM=0 keeps the table form)
__host__ __device__ constexpr double m2l_binom(int n, int k) {
  unsigned long long c = 1;
  for (int i = 1; i <= k; ++i) c = c * (unsigned long long)(n - k + i) / (unsigned long long)i;
  return (double)c;
}
// compile-time j, k: the coefficient is a constant expression
template <int PM, int J, int K>
__device__ __forceinline__ void m2l_chain(double& sx, double& sy, const double* ax,
                                          const double* ay) {
  if constexpr (K <= PM) {
    constexpr double cf = m2l_binom(J + K - 1, K - 1);
    sx = fma(cf, ax[K - 1], sx);
    sy = fma(cf, ay[K - 1], sy);
    m2l_chain<PM, J, K + 1>(sx, sy, ax, ay);
  }
}

template <int PM>
struct M2LDenseCfg {
  static constexpr int R = 2 * (PM + 1);          // SMEM rows (re/im per coefficient)
  static constexpr int STR = M2L_ITEM + 1;        // odd row stride: conflict-free
  static constexpr int SMEM = R * STR * 8;
  // exact orders above 20 (M2L_HALF): outputs j <= JH are parked and folded
  // first, then the rest in the same rows -- half the SMEM, so more L1 for
  // the source rows that consecutive targets share (C4 M2L 0.851 -> 0.822
  // ms; at order 20 the extra barrier and a spill cost more: 0.371 -> 0.420)
  static constexpr int JH = PM / 2;
  static constexpr bool HALF_EX = M2L_HALF && M2L_IMM && PM > 20;
  static constexpr int SMEM_EX = (HALF_EX ? 2 * (JH + 1) : R) * STR * 8;
  // resident warps per SM the register budget allows (128 / 168 / 252 regs)
  static constexpr int WARPS = PM <= 20 ? 16 : (PM <= 24 ? 12 : 8);
  static constexpr int MINB = WARPS / (M2L_ITEM / 32);
};

// one coalesced row update of a target segment's sum (coefficient j, part comp)
__device__ __forceinline__ void m2l_emit(double2* local, double2* partials,
                                         unsigned char* item_flags, long long item, int p, int t,
                                         int j, int comp, double v, bool starts_before,
                                         bool ends_after, bool set_flags = true) {
  if (!starts_before && !ends_after) {
    double* dst = reinterpret_cast<double*>(local + (long long)t * (p + 1)) + 2 * j + comp;
    *dst += v;
    return;
  }
  const int slot = starts_before ? 0 : 1;
  reinterpret_cast<double*>(partials + (item * 2 + slot) * (p + 1))[2 * j + comp] = v;
  if (set_flags && j == 0 && comp == 0) {
    const unsigned f = starts_before ? (ends_after ? 5u : 1u) : 2u;
    atomicOr(reinterpret_cast<unsigned int*>(item_flags + (item & ~3ll)), f << (8 * (item & 3)));
  }
}

// exact-order contraction with compile-time (j, k): every output's chain in
// the order of the table form, coefficients as constant expressions
template <int PM, int J, int JE, int JB, int STR>
__device__ __forceinline__ void m2l_outputs(const double* ax, const double* ay, cplx& pw, cplx inv,
                                            double* red, int tid) {
  if constexpr (J <= JE) {
    double sx = ax[0], sy = ay[0];
    m2l_chain<PM, J, 2>(sx, sy, ax, ay);
    cplx b{sx, sy};
    if constexpr (J > 0) {
      b = cmul(b, pw);
      pw = cmul(pw, inv);
    }
    red[(2 * (J - JB)) * STR + tid] = b.x;
    red[(2 * (J - JB) + 1) * STR + tid] = b.y;
    m2l_outputs<PM, J + 1, JE, JB, STR>(ax, ay, pw, inv, red, tid);
  }
}

// the pair a thread owns in one item, with its source row prefetched
template <int PM>
struct M2LPair {
  int t, s;
  double2 a[PM];
};

// the pair's source row, its (target, source) indices already in hand
template <int PM>
__device__ __forceinline__ void m2l_load_row(M2LPair<PM>& P, int t, int s,
                                             const double2* __restrict__ mult, int p) {
  P.t = t;
  P.s = s;
  const double2* a = mult + (long long)s * (p + 1);
#pragma unroll
  for (int k = 1; k <= PM; ++k) P.a[k - 1] = k <= p ? a[k] : make_double2(0.0, 0.0);
}

template <int PM>
__device__ __forceinline__ void m2l_load_pair(M2LPair<PM>& P, long long i, long long npairs,
                                              const int* __restrict__ w_src,
                                              const int* __restrict__ w_tgt,
                                              const double2* __restrict__ mult, int p) {
  const bool valid = i < npairs;
  P.t = valid ? __ldg(w_tgt + i) : -1;
  P.s = valid ? __ldg(w_src + i) : 1;   // padding lanes read box 1's (computed) row
  const double2* a = mult + (long long)P.s * (p + 1);
#pragma unroll
  for (int k = 1; k <= PM; ++k) P.a[k - 1] = k <= p ? a[k] : make_double2(0.0, 0.0);
}

template <int PM, bool EX>
__global__ void __launch_bounds__(M2L_ITEM, M2LDenseCfg<PM>::MINB)
k_m2l_dense(const int* __restrict__ lo_ptr, const int* __restrict__ total_ptr,
            const int* __restrict__ w_src, const int* __restrict__ w_tgt,
            const double* __restrict__ cx, const double* __restrict__ cy,
            const double2* __restrict__ mult, double2* local, double2* partials,
            unsigned char* item_flags, int p, DevStatus* st) {
  pdl_enter();
  static_assert(PM <= 32, "dense M2L is compiled for PM <= 32");
  if constexpr (EX) p = PM;                       // exact order: p is a compile-time constant
  using Cfg = M2LDenseCfg<PM>;
  if (lists_overflowed(st)) return;
  extern __shared__ double red[];                 // [R][STR]
  __shared__ int s_t[M2L_ITEM];
  __shared__ int s_seg[M2L_ITEM + 1];
  __shared__ int s_nseg;
  __shared__ int s_wcnt[M2L_ITEM / 32];
  // pairs [lo, hi) of the flat list (one range of whole levels: no target
  // spans its ends); items of M2L_ITEM pairs from lo, numbered from ibase in
  // the partials / flags arrays (disjoint from any range before lo)
  const long long lo = lo_ptr ? *lo_ptr : 0, hi = *total_ptr;
  const long long npairs = hi - lo;
  const long long nitems = (npairs + M2L_ITEM - 1) / M2L_ITEM;
  const long long ibase = lo ? lo / M2L_ITEM + 1 : 0;
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  M2LPair<PM> P;
  // (target, source) of this thread's pair in the first item; every item
  // prefetches the next item's pair indices, so an item start waits on one
  // round trip (the source row) instead of two
  int nt_t = -1, nt_s = 0;
  if (blockIdx.x < nitems) {
    const long long i = lo + (long long)blockIdx.x * M2L_ITEM + tid;
    nt_t = i < hi ? __ldg(w_tgt + i) : -1;
    nt_s = i < hi ? __ldg(w_src + i) : 1;
  }
  for (long long it = blockIdx.x; it < nitems; it += gridDim.x) {
    const long long i0 = lo + it * M2L_ITEM, item = ibase + it;
    m2l_load_row<PM>(P, nt_t, nt_s, mult, p);
    {
      const long long inext = i0 + (long long)gridDim.x * M2L_ITEM + tid;
      nt_t = inext < hi ? __ldg(w_tgt + inext) : -1;
      nt_s = inext < hi ? __ldg(w_src + inext) : 1;
    }
    // targets just before / after the item (segments continuing across items)
    const int prev_t = it > 0 ? __ldg(w_tgt + i0 - 1) : -1;
    const long long nxt = i0 + M2L_ITEM;
    const int next_t = nxt < hi ? __ldg(w_tgt + nxt) : -1;
    const bool valid = P.t >= 0;
    const int t = P.t;
    const int tt = valid ? t : 0;
    const double rx = cx[P.s] - cx[tt], ry = cy[P.s] - cy[tt];   // source - target
    const bool sing = valid && rx == 0.0 && ry == 0.0;
    if (sing) atomicOr(&st->flags, ST_M2L_SINGULAR);
    const cplx inv = (valid && !sing) ? crcp_fast(cplx{rx, ry}) : cplx{0.0, 0.0};
    // alpha_k = a_k q^k with q = -1/rho (operators.py:203-206)
    const cplx q{-inv.x, -inv.y};
    double ax[PM], ay[PM];
    {
      // powers q^k as four interleaved chains (stride q^4): the serial
      // dependency of the prescale drops from PM to ~PM/4 complex products
      const cplx q2 = cmul(q, q);
      cplx pw[4] = {q, q2, cmul(q2, q), cmul(q2, q2)};
      const cplx q4 = pw[3];
#pragma unroll
      for (int k = 1; k <= PM; k += 4) {
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          if (k + u <= PM) {
            const cplx v = cmul(cplx{P.a[k + u - 1].x, P.a[k + u - 1].y}, pw[u]);
            ax[k + u - 1] = v.x;
            ay[k + u - 1] = v.y;
            pw[u] = cmul(pw[u], q4);
          }
        }
      }
    }
    // c_j = sum_k C(j+k-1, k-1) alpha_k ; b_j = c_j / rho^j = c_j inv^j
    cplx pw_ex = inv;
    constexpr bool HALF = EX && Cfg::HALF_EX;
#if M2L_IMM
    if constexpr (EX) {
      m2l_outputs<PM, 0, HALF ? Cfg::JH : PM, 0, Cfg::STR>(ax, ay, pw_ex, inv, red, tid);
    } else
#endif
    {
      cplx pw = inv;
#pragma unroll
      for (int j = 0; j <= PM; ++j) {
        double sx = ax[0], sy = ay[0];                 // C(j, 0) = 1
#pragma unroll
        for (int k = 2; k <= PM; ++k) {
          sx = fma(c_m2l_tab<PM>.v[j][k - 1], ax[k - 1], sx);
          sy = fma(c_m2l_tab<PM>.v[j][k - 1], ay[k - 1], sy);
        }
        cplx b{sx, sy};
        if (j > 0) {
          b = cmul(b, pw);
          pw = cmul(pw, inv);
        }
        red[(2 * j) * Cfg::STR + tid] = b.x;
        red[(2 * j + 1) * Cfg::STR + tid] = b.y;
      }
    }
    s_t[tid] = t;
    __syncthreads();
    // segment starts (pairs are sorted by target)
    const bool start = valid && (tid == 0 || s_t[tid - 1] != t);
    const unsigned bal = __ballot_sync(0xffffffffu, start);
    if (lane == 0) s_wcnt[wid] = __popc(bal);
    __syncthreads();
    int before = 0;
#pragma unroll
    for (int w = 0; w < M2L_ITEM / 32; ++w) before += w < wid ? s_wcnt[w] : 0;
    if (start) s_seg[before + __popc(bal & ((1u << lane) - 1))] = tid;
    if (tid == M2L_ITEM - 1) {
      int tot = 0;
#pragma unroll
      for (int w = 0; w < M2L_ITEM / 32; ++w) tot += s_wcnt[w];
      s_nseg = tot;
      s_seg[tot] = (int)min((long long)M2L_ITEM, npairs - it * M2L_ITEM);
    }
    __syncthreads();
    const int nseg = s_nseg;
    const bool first_cont = it > 0 && prev_t == s_t[0];
    const int nvalid = s_seg[nseg];
    const bool last_cont = nvalid == M2L_ITEM && next_t >= 0 && next_t == s_t[nvalid - 1];
    // fold rows [r0, r1) of every segment; SMEM row r - r0 holds row r
    auto fold = [&](int r0, int r1) {
      const int R = r1 - r0;
      for (int task = tid; task < nseg * R; task += M2L_ITEM) {
        const int sg = task / R, rr = task - sg * R, r = r0 + rr;
        const int q0 = s_seg[sg], q1 = s_seg[sg + 1];
        const double* row = red + rr * Cfg::STR;
        // an in-place target's old value is fetched before the sum (its global
        // round trip overlaps the SMEM reads)
        const bool sb = sg == 0 && first_cont, ea = sg == nseg - 1 && last_cont;
        double* dst = reinterpret_cast<double*>(local + (long long)s_t[q0] * (p + 1)) + r;
        const double old = (!sb && !ea) ? *dst : 0.0;
        // four interleaved chains (fixed order), then ((0+1)+(2+3))
        double a0 = 0.0, a1 = 0.0, a2 = 0.0, a3 = 0.0;
        int q = q0;
        for (; q + 4 <= q1; q += 4) {
          a0 += row[q];
          a1 += row[q + 1];
          a2 += row[q + 2];
          a3 += row[q + 3];
        }
        if (q < q1) a0 += row[q];
        if (q + 1 < q1) a1 += row[q + 1];
        if (q + 2 < q1) a2 += row[q + 2];
        const double v = (a0 + a1) + (a2 + a3);
        if (!sb && !ea)
          *dst = old + v;
        else
          m2l_emit(local, partials, item_flags, item, p, s_t[q0], r >> 1, r & 1, v, sb, ea,
                   false);
      }
    };
    if constexpr (HALF) {
      fold(0, 2 * (Cfg::JH + 1));
      __syncthreads();
#if M2L_IMM
      m2l_outputs<PM, Cfg::JH + 1, PM, Cfg::JH + 1, Cfg::STR>(ax, ay, pw_ex, inv, red, tid);
#endif
      __syncthreads();
      fold(2 * (Cfg::JH + 1), 2 * (p + 1));
    } else {
      fold(0, 2 * (p + 1));
    }
    // the item's chain flags as one byte store (no memset, no atomics): 1 head
    // part in slot 0, 2 tail part in slot 1, 5 the whole item continues a chain
    if (tid == 0)
      item_flags[item] = (unsigned char)(nseg == 1 && first_cont && last_cont
                                             ? 5u
                                             : (first_cont ? 1u : 0u) | (last_cont ? 2u : 0u));
    __syncthreads();
  }
}

// M2L on the FP64 tensor cores (mma.sync m16n8k4 .f64, DMMA).  The dense
// Pascal-matrix form above is a real GEMM per item: rows = (re, im) of the
// prescaled alpha_k of 8 pairs (A, 16 x 4 per k-step), columns = output
// coefficients j (B = T[j][k-1] = C(j+k-1, k-1), a constant matrix held in
// registers as KT x NT fragments for the whole kernel), so the ~2p(p+1) FMAs
// per pair issue as KT*NT/8 DMMA instructions per pair instead of ~840 DFMA
// (p=20: 15 DMMA per 8 pairs).  Prescale (alpha_k = a_k q^k, q = -1/rho) and
// postscale (b_j = c_j / rho^j) stay on the DFMA pipe; each thread of a quad
// (lane & 3) handles the k's / j's its fragments own.  The per-target fold
// (SMEM rows, ordered segment sums, partials + k_m2l_fixup for targets
// spanning items) is the dense kernel's, unchanged.  Fragment layouts
// (PTX ISA, mma.m16n8k4 .f64): a0 = A[g][tig], a1 = A[g+8][tig];
// b0 = B[tig][g]; c{0,1} = C[g][2 tig + {0,1}], c{2,3} = C[g+8][2 tig + {0,1}]
// with g = lane >> 2, tig = lane & 3.
template <int PM>
struct M2LDmmaCfg {
  static constexpr int KT = (PM + 3) / 4;          // k-steps over k = 1..PM
  static constexpr int NT = (PM + 1 + 7) / 8;      // n-tiles over j = 0..PM
  static constexpr int R = 2 * (PM + 1);
  static constexpr int STR = M2L_ITEM + 1;
  static constexpr int SMEM = R * STR * 8;
  static constexpr int MT = M2L_ITEM / 2 / 8;      // m-tiles (8 pairs) per warp per item
  static constexpr int MINB = PM <= 24 ? 8 : 5;    // B fragments: KT*NT registers pairs
};

__device__ __forceinline__ void dmma_m16n8k4(double (&d)[4], double a0, double a1, double b) {
  asm("mma.sync.aligned.m16n8k4.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5}, {%6}, "
      "{%0,%1,%2,%3};"
      : "+d"(d[0]), "+d"(d[1]), "+d"(d[2]), "+d"(d[3])
      : "d"(a0), "d"(a1), "d"(b));
}

template <int PM>
__global__ void __launch_bounds__(M2L_ITEM, M2LDmmaCfg<PM>::MINB)
k_m2l_dmma(const int* __restrict__ total_ptr, const int* __restrict__ w_src,
           const int* __restrict__ w_tgt, const double* __restrict__ cx,
           const double* __restrict__ cy, const double2* __restrict__ mult, double2* local,
           double2* partials, unsigned char* item_flags, int p, DevStatus* st) {
  pdl_enter();
  static_assert(M2L_ITEM == 64, "two warps x 4 m-tiles of 8 pairs");
  using Cfg = M2LDmmaCfg<PM>;
  if (lists_overflowed(st)) return;
  extern __shared__ double red[];                 // [R][STR]
  __shared__ int s_t[M2L_ITEM];
  __shared__ int s_seg[M2L_ITEM + 1];
  __shared__ int s_nseg;
  __shared__ int s_wcnt[M2L_ITEM / 32];
  const long long npairs = *total_ptr;
  const long long nitems = (npairs + M2L_ITEM - 1) / M2L_ITEM;
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  const int g = lane >> 2, tig = lane & 3;
  double bf[Cfg::KT][Cfg::NT];                     // B = T[j][k-1], j = 8 nt + g, k = 4 ks + tig + 1
#pragma unroll
  for (int ks = 0; ks < Cfg::KT; ++ks)
#pragma unroll
    for (int nt = 0; nt < Cfg::NT; ++nt) {
      const int j = nt * 8 + g, k = ks * 4 + tig + 1;
      bf[ks][nt] = (j <= PM && k <= PM) ? c_m2l_tab<PM>.v[j][k - 1] : 0.0;
    }
  for (long long item = blockIdx.x; item < nitems; item += gridDim.x) {
    const long long i_own = item * M2L_ITEM + tid;
    const int t_own = i_own < npairs ? __ldg(w_tgt + i_own) : -1;
    const int prev_t = item > 0 ? __ldg(w_tgt + item * M2L_ITEM - 1) : -1;
    const long long nxt = (item + 1) * M2L_ITEM;
    const int next_t = nxt < npairs ? __ldg(w_tgt + nxt) : -1;
#pragma unroll 1
    for (int mt = 0; mt < Cfg::MT; ++mt) {
      const int slot = wid * 32 + mt * 8 + g;
      const long long i = item * M2L_ITEM + slot;
      const bool valid = i < npairs;
      const int t = valid ? __ldg(w_tgt + i) : 0;
      const int s = valid ? __ldg(w_src + i) : 1;
      const double rx = cx[s] - cx[t], ry = cy[s] - cy[t];        // source - target
      const bool sing = valid && rx == 0.0 && ry == 0.0;
      if (sing && tig == 0) atomicOr(&st->flags, ST_M2L_SINGULAR);
      const cplx inv = (valid && !sing) ? crcp_fast(cplx{rx, ry}) : cplx{0.0, 0.0};
      const cplx q{-inv.x, -inv.y};
      const cplx q2 = cmul(q, q), q3 = cmul(q2, q), q4 = cmul(q2, q2);
      cplx qk = tig == 0 ? q : (tig == 1 ? q2 : (tig == 2 ? q3 : q4));   // q^(tig+1)
      const double2* a = mult + (long long)s * (p + 1);
      double acc[Cfg::NT][4];
#pragma unroll
      for (int nt = 0; nt < Cfg::NT; ++nt) acc[nt][0] = acc[nt][1] = acc[nt][2] = acc[nt][3] = 0.0;
#pragma unroll
      for (int ks = 0; ks < Cfg::KT; ++ks) {
        const int k = ks * 4 + tig + 1;
        const double2 ak = k <= p ? a[k] : make_double2(0.0, 0.0);
        const cplx al = cmul(cplx{ak.x, ak.y}, qk);                  // alpha_k (operators.py:203-206)
        qk = cmul(qk, q4);
#pragma unroll
        for (int nt = 0; nt < Cfg::NT; ++nt) dmma_m16n8k4(acc[nt], al.x, al.y, bf[ks][nt]);
      }
      // b_j = c_j inv^j for j = 8 nt + 2 tig + e (operators.py:218-219)
      const cplx i2 = cmul(inv, inv), i4 = cmul(i2, i2), i8 = cmul(i4, i4);
      cplx w = tig == 0 ? cplx{1.0, 0.0} : (tig == 1 ? i2 : (tig == 2 ? i4 : cmul(i4, i2)));
#pragma unroll
      for (int nt = 0; nt < Cfg::NT; ++nt) {
        const cplx w1 = cmul(w, inv);
        const int j0 = nt * 8 + 2 * tig;
        const cplx b0 = cmul(cplx{acc[nt][0], acc[nt][2]}, w);
        const cplx b1 = cmul(cplx{acc[nt][1], acc[nt][3]}, w1);
        if (j0 <= PM) {
          red[(2 * j0) * Cfg::STR + slot] = b0.x;
          red[(2 * j0 + 1) * Cfg::STR + slot] = b0.y;
        }
        if (j0 + 1 <= PM) {
          red[(2 * j0 + 2) * Cfg::STR + slot] = b1.x;
          red[(2 * j0 + 3) * Cfg::STR + slot] = b1.y;
        }
        w = cmul(w, i8);
      }
    }
    s_t[tid] = t_own;
    __syncthreads();
    const bool valid = t_own >= 0;
    const int t = t_own;
    const bool start = valid && (tid == 0 || s_t[tid - 1] != t);
    const unsigned bal = __ballot_sync(0xffffffffu, start);
    if (lane == 0) s_wcnt[wid] = __popc(bal);
    __syncthreads();
    int before = 0;
#pragma unroll
    for (int w2 = 0; w2 < M2L_ITEM / 32; ++w2) before += w2 < wid ? s_wcnt[w2] : 0;
    if (start) s_seg[before + __popc(bal & ((1u << lane) - 1))] = tid;
    if (tid == M2L_ITEM - 1) {
      int tot = 0;
#pragma unroll
      for (int w2 = 0; w2 < M2L_ITEM / 32; ++w2) tot += s_wcnt[w2];
      s_nseg = tot;
      s_seg[tot] = (int)min((long long)M2L_ITEM, npairs - item * M2L_ITEM);
    }
    __syncthreads();
    const int nseg = s_nseg;
    const int R = 2 * (p + 1);
    const bool first_cont = item > 0 && prev_t == s_t[0];
    const int nvalid = s_seg[nseg];
    const bool last_cont = nvalid == M2L_ITEM && next_t >= 0 && next_t == s_t[nvalid - 1];
    for (int task = tid; task < nseg * R; task += M2L_ITEM) {
      const int sg = task / R, r = task - sg * R;
      const int q0 = s_seg[sg], q1 = s_seg[sg + 1];
      const double* row = red + r * Cfg::STR;
      double a0 = 0.0, a1 = 0.0, a2 = 0.0, a3 = 0.0;
      int qq = q0;
      for (; qq + 4 <= q1; qq += 4) {
        a0 += row[qq];
        a1 += row[qq + 1];
        a2 += row[qq + 2];
        a3 += row[qq + 3];
      }
      if (qq < q1) a0 += row[qq];
      if (qq + 1 < q1) a1 += row[qq + 1];
      if (qq + 2 < q1) a2 += row[qq + 2];
      m2l_emit(local, partials, item_flags, item, p, s_t[q0], r >> 1, r & 1,
               (a0 + a1) + (a2 + a3), sg == 0 && first_cont, sg == nseg - 1 && last_cont);
    }
    __syncthreads();
  }
}

// Target-owned M2L (default).  One warp per target box walks the target's
// weak list in chunks of 16 pairs; lane pair (2i, 2i+1) carries the real /
// imaginary part of pair i (the cascades of operators.py:208-213 are
// real-linear).  Each lane accumulates its pairs in order, then a fixed xor
// butterfly over the 16 lane pairs folds them and the target row is updated
// once -- no partials, no fixup, no atomics.
template <int PM>
__global__ void __launch_bounds__(128)
k_m2l_target(long long nbox, const int* __restrict__ woff, const int* __restrict__ w_src,
             const double* __restrict__ cx, const double* __restrict__ cy,
             const double2* __restrict__ mult, double2* local, int p, DevStatus* st) {
  pdl_enter();
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
      for (int k = 2; k <= PM; ++k)               // pass 1, old values (operators.py:208-210)
#pragma unroll
        for (int j = PM - k; j < PM; ++j) c[j] += c[j + 1];
#pragma unroll
      for (int k = PM; k >= 1; --k)               // pass 2, new values (operators.py:211-213)
#pragma unroll
        for (int j = k; j <= PM; ++j) c[j] += c[j - 1];
      {   // b_j = c_j / rho^j = c_j (-q)^j (operators.py:218-219)
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

// ordered fold of the partial sums of targets whose pairs span several warp
// items: one warp per item, lanes over coefficients (coalesced rows)
__global__ void k_m2l_fixup(const int* __restrict__ lo_ptr, const int* __restrict__ total_ptr,
                            const int* __restrict__ w_tgt, const double2* __restrict__ partials,
                            const unsigned char* __restrict__ item_flags, double2* local, int p,
                            int item_pairs, const DevStatus* st) {
  pdl_enter();
  if (lists_overflowed(st)) return;
  const long long lo = lo_ptr ? *lo_ptr : 0, hi = *total_ptr;   // k_m2l_dense's range
  const long long nitems = (hi - lo + item_pairs - 1) / item_pairs;
  const long long ibase = lo ? lo / item_pairs + 1 : 0;
  const int lane = threadIdx.x & 31;
  const long long nwarps = ((long long)gridDim.x * blockDim.x) >> 5;
  for (long long w = (blockIdx.x * (long long)blockDim.x + threadIdx.x) >> 5; w < nitems;
       w += nwarps) {
    if (!(item_flags[ibase + w] & 2)) continue;  // chain head: its tail segment continues
    const int t = w_tgt[lo + w * item_pairs + item_pairs - 1];
    double2* dst = local + (long long)t * (p + 1);
    for (int j = lane; j <= p; j += 32) {
      double2 s = partials[((ibase + w) * 2 + 1) * (p + 1) + j];
      for (long long u = w + 1; u < nitems; ++u) {
        const double2 v = partials[((ibase + u) * 2 + 0) * (p + 1) + j];
        s.x += v.x;
        s.y += v.y;
        if (!(item_flags[ibase + u] & 4)) break;
      }
      const double2 o = dst[j];
      dst[j] = make_double2(o.x + s.x, o.y + s.y);
    }
  }
}

// --------------------------------------------------------------------------
// L2P + M2P (engine.py:132-160): one thread per evaluation point (tree order);
// its leaf comes from the eval tree (separate points) or, for points aliasing
// the sources, from the data-independent source offsets.  phi = L2P (Horner
// in y - z0), then += each m2p source in ascending order (operators.py:
// 358-386).  Coefficient rows stream from L1/L2 (the points of one leaf
// share them), all loads of a row in flight at once.
template <int PM, bool EX>
__global__ void __launch_bounds__(128)
k_l2p_m2p(long long m, long long e0, long long e1, int L, const unsigned* __restrict__ eleaf,
          const double2* __restrict__ eval_pos, const int* __restrict__ m_off,
          const int* __restrict__ m_idx, const double* __restrict__ cx,
          const double* __restrict__ cy, const double2* __restrict__ mult,
          const double2* __restrict__ local, double2* phi, int p, DevStatus* st) {
  pdl_enter();
  // evaluation points [e0, e1) of m (tree order)
  const long long e = e0 + blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (e >= e1 || lists_overflowed(st)) return;
  const long long lb = level_base(L);
  const long long b = eleaf ? (long long)eleaf[e] : leaf_of_position(e, m, 2 * L);
  const double2 y = eval_pos[e];
  const cplx w{y.x - cx[lb + b], y.y - cy[lb + b]};
  const double2* bl = local + (lb + b) * (p + 1);
  cplx c[PM + 1];
#pragma unroll
  for (int j = 0; j <= PM; ++j) c[j] = ld_coef<EX>(bl, j, p);
  cplx acc = c[PM];
#pragma unroll
  for (int j = PM - 1; j >= 0; --j) acc = cadd(cmul(acc, w), c[j]);
  // long m2p lists (clustered inputs: up to ~850 boxes) continue in k_m2p_long
  const int qa = m_off[b], qe = min(m_off[b + 1], qa + M2P_INLINE);
  for (int q = qa; q < qe; ++q) {
    const long long ga = lb + m_idx[q];
    const cplx u{y.x - cx[ga], y.y - cy[ga]};
    if (u.x == 0.0 && u.y == 0.0) {
      atomicOr(&st->flags, ST_M2P_SINGULAR);
      continue;
    }
    const cplx inv = crcp_fast(u);
    const double2* a = mult + ga * (p + 1);
#pragma unroll
    for (int j = 1; j <= PM; ++j) c[j] = ld_coef<EX>(a, j, p);
    cplx h = c[PM];
#pragma unroll
    for (int j = PM - 1; j >= 1; --j) h = cadd(cmul(h, inv), c[j]);
    acc = cadd(acc, cmul(h, inv));
  }
  phi[e] = make_double2(acc.x, acc.y);
}

// M2P beyond the first M2P_INLINE sources of a leaf (engine.py:152-160): one
// CTA per long-list leaf; thread t sums sources t, t+256, ... for every point
// of the leaf, then a fixed SMEM tree folds the 256 partial sums per point.
// Deterministic; the long tail of clustered inputs is spread over 256 threads
// instead of serialising one warp.
constexpr int M2P_LONG_THREADS = 256;
constexpr int M2P_LONG_POINTS = 8;      // points per pass (SMEM: 8 x 256 complex)

__global__ void k_m2p_find_long(long long b0, long long b1, const int* __restrict__ m_off,
                                int* list, int* count) {
  pdl_enter();
  const long long b = b0 + blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (b < b1 && m_off[b + 1] - m_off[b] > M2P_INLINE) list[atomicAdd(count, 1)] = (int)b;
}

template <int PM, bool EX>
__global__ void __launch_bounds__(M2P_LONG_THREADS)
k_m2p_long(int L, const int* __restrict__ list, const int* __restrict__ count,
           const int* __restrict__ eoff, const double2* __restrict__ eval_pos,
           const int* __restrict__ m_off, const int* __restrict__ m_idx,
           const double* __restrict__ cx, const double* __restrict__ cy,
           const double2* __restrict__ mult, double2* phi, int p, DevStatus* st) {
  pdl_enter();
  __shared__ double2 red[M2P_LONG_POINTS][M2P_LONG_THREADS];
  if (lists_overflowed(st)) return;
  const int n = *count;
  const long long lb = level_base(L);
  const int tid = threadIdx.x;
  for (int it = blockIdx.x; it < n; it += gridDim.x) {
    const int b = list[it];
    const int e0 = eoff[b], e1 = eoff[b + 1];
    const int q0 = m_off[b] + M2P_INLINE, q1 = m_off[b + 1];
    for (int eb = e0; eb < e1; eb += M2P_LONG_POINTS) {
      const int np = min(M2P_LONG_POINTS, e1 - eb);
      cplx acc[M2P_LONG_POINTS];
      double2 y[M2P_LONG_POINTS];
#pragma unroll
      for (int k = 0; k < M2P_LONG_POINTS; ++k) {
        acc[k] = cplx{0.0, 0.0};
        y[k] = k < np ? eval_pos[eb + k] : eval_pos[eb];
      }
      for (int q = q0 + tid; q < q1; q += M2P_LONG_THREADS) {
        const long long ga = lb + m_idx[q];
        const double2* a = mult + ga * (p + 1);
        cplx c[PM + 1];
#pragma unroll
        for (int j = 1; j <= PM; ++j) c[j] = ld_coef<EX>(a, j, p);
        const double ax = cx[ga], ay = cy[ga];
#pragma unroll
        for (int k = 0; k < M2P_LONG_POINTS; ++k) {
          if (k >= np) break;
          const cplx u{y[k].x - ax, y[k].y - ay};
          if (u.x == 0.0 && u.y == 0.0) {
            atomicOr(&st->flags, ST_M2P_SINGULAR);
            continue;
          }
          const cplx inv = crcp_fast(u);
          cplx h = c[PM];
#pragma unroll
          for (int j = PM - 1; j >= 1; --j) h = cadd(cmul(h, inv), c[j]);
          acc[k] = cadd(acc[k], cmul(h, inv));
        }
      }
#pragma unroll
      for (int k = 0; k < M2P_LONG_POINTS; ++k) red[k][tid] = make_double2(acc[k].x, acc[k].y);
      __syncthreads();
      for (int w = M2P_LONG_THREADS / 2; w > 0; w >>= 1) {
        if (tid < w) {
#pragma unroll
          for (int k = 0; k < M2P_LONG_POINTS; ++k) {
            const double2 u = red[k][tid], v = red[k][tid + w];
            red[k][tid] = make_double2(u.x + v.x, u.y + v.y);
          }
        }
        __syncthreads();
      }
      if (tid < np) {
        const double2 f = phi[eb + tid], v = red[tid][0];
        phi[eb + tid] = make_double2(f.x + v.x, f.y + v.y);
      }
      __syncthreads();
    }
  }
}

inline unsigned nblk(long long n, int t) { return (unsigned)((n + t - 1) / t); }

// --------------------------------------------------------------------------
template <int PM>
struct Launch {
  static void upward(const TreeState& T, const ListState& Ls, ExpState& E, const int* offL,
                     DevStatus* dstat, cudaStream_t st, const Part& part, int which) {
    const int L = T.L, p = E.p;
    if (L == 0) return;
    const long long b0 = part.lo(L), b1 = part.hi(L);
    if (which != 2) {
      note_launch();
      launch(p == PM ? k_p2m<PM, true> : k_p2m<PM, false>, nblk(b1 - b0, 128), 128, 0, st, L, b0,
             b1, offL, T.src_pos.as<double2>(),
             T.src_g.as<double>(), T.box_cx.as<double>(), T.box_cy.as<double>(),
             E.mult.as<double2>(), p);
    }
    if (which == 1) return;
    note_launch();
    E.p2l_rows.reserve(sizeof(double2) * std::max(1ll, Ls.cap_p2l) * (p + 1));
    launch(p == PM ? k_p2l_pair<PM, true> : k_p2l_pair<PM, false>, 8 * sm_count(), 128, 0, st,
        L, b0, b1, offL, Ls.p2l_off.as<int>(), Ls.p2l_idx.as<int>(), T.src_pos.as<double2>(),
        T.src_g.as<double>(), T.box_cx.as<double>(), T.box_cy.as<double>(),
        E.p2l_rows.as<double2>(), p, dstat);
    note_launch();
    launch(k_p2l_fold, nblk((b1 - b0) * (p + 1), 128), 128, 0, st, 
        L, b0, b1, Ls.p2l_off.as<int>(), E.p2l_rows.as<double2>(), E.local.as<double2>(), p,
        dstat);
  }
  static void m2m(const TreeState& T, ExpState& E, cudaStream_t st, const Part& part, int lmin,
                  int lmax) {
    for (int l = lmax; l >= lmin; --l) {
      const long long k0 = part.lo(l), k1 = part.hi(l);
      note_launch();
      launch(E.p == PM ? k_m2m<PM, true> : k_m2m<PM, false>, nblk(4 * (k1 - k0), 128), 128, 0, st,
             l, k0, k1, T.box_cx.as<double>(),
                                                    T.box_cy.as<double>(), E.mult.as<double2>(),
                                                    E.p);
    }
  }
  static void m2l(const TreeState& T, const ListState& Ls, ExpState& E, DevStatus* dstat,
                  cudaStream_t st) {
    const int L = T.L;
    if (L == 0) return;
    const int* total = Ls.weak_off.as<int>() + level_base(L + 1);
    const int* lo = nullptr;      // the kernels take a pair range [lo, total); all pairs here
    if constexpr (PM > 32) {
      launch_target(T, Ls, E, dstat, st);
    } else {
      if (m2l_force_target()) {
        launch_target(T, Ls, E, dstat, st);
        return;
      }
      using Cfg = M2LDenseCfg<PM>;
      const long long items = (Ls.cap_weak + M2L_ITEM - 1) / M2L_ITEM + 2;
      E.partials.reserve(sizeof(double2) * 2 * items * (E.p + 1));
      E.item_flags.reserve(((items + 4) & ~3ll) + 8);
      if (m2l_dmma()) {
        FMM_CUDA(cudaMemsetAsync(E.item_flags.p, 0, ((items + 4) & ~3ll) + 8, st));
        using DC = M2LDmmaCfg<PM>;
        static unsigned attr_dmma = 0;
        ensure_smem_attr(k_m2l_dmma<PM>, DC::SMEM, attr_dmma);
        const unsigned grid = (unsigned)std::min<long long>(
            std::max(1ll, items), (long long)M2L_GRID_WAVES * DC::MINB * sm_count());
        note_launch();
        launch(k_m2l_dmma<PM>, grid, M2L_ITEM, DC::SMEM, st,
            total, Ls.weak_idx.as<int>(), Ls.weak_tgt.as<int>(), T.box_cx.as<double>(),
            T.box_cy.as<double>(), E.mult.as<double2>(), E.local.as<double2>(),
            E.partials.as<double2>(), E.item_flags.as<unsigned char>(), E.p, dstat);
      } else {
        static unsigned attr_dense[2] = {0, 0};
        const bool ex = E.p == PM;
        auto kern = ex ? k_m2l_dense<PM, true> : k_m2l_dense<PM, false>;
        const int smem = ex ? Cfg::SMEM_EX : Cfg::SMEM;
        ensure_smem_attr(kern, smem, attr_dense[ex]);
        const unsigned grid = (unsigned)std::min<long long>(
            std::max(1ll, items), (long long)M2L_GRID_WAVES * Cfg::MINB * sm_count());
        note_launch();
        launch(kern, grid, M2L_ITEM, smem, st,
            lo, total, Ls.weak_idx.as<int>(), Ls.weak_tgt.as<int>(), T.box_cx.as<double>(),
            T.box_cy.as<double>(), E.mult.as<double2>(), E.local.as<double2>(),
            E.partials.as<double2>(), E.item_flags.as<unsigned char>(), E.p, dstat);
      }
      note_launch();
      launch(k_m2l_fixup, std::max(1u, std::min(4096u, nblk(items * 32, 128))), 128, 0, st,
          lo, total, Ls.weak_tgt.as<int>(), E.partials.as<double2>(),
          E.item_flags.as<unsigned char>(), E.local.as<double2>(), E.p, M2L_ITEM, dstat);
    }
  }
  static void launch_target(const TreeState& T, const ListState& Ls, ExpState& E,
                            DevStatus* dstat, cudaStream_t st) {
    const long long nbox = level_base(T.L + 1);
    const unsigned grid = (unsigned)std::min<long long>(nblk(nbox * 32, 128), 64ll * sm_count());
    note_launch();
    launch(k_m2l_target<PM>, grid, 128, 0, st, nbox, Ls.weak_off.as<int>(), Ls.weak_idx.as<int>(),
                                           T.box_cx.as<double>(), T.box_cy.as<double>(),
                                           E.mult.as<double2>(), E.local.as<double2>(), E.p,
                                           dstat);
  }
  static void l2l(const TreeState& T, ExpState& E, cudaStream_t st, const Part& part) {
    int l_first = 1;
    E.l2l_chain_lt = 0;
    // single GPU: levels 2..lt (lt: the deepest level of at most 4096 boxes)
    // through the chained kernel, the rest level by level
    if (part.G == 1 && L2L_CHAIN) {
      int lt = 1;
      while (lt + 1 < T.L && (1ll << (2 * (lt + 1))) <= L2L_CHAIN_MAXBOX) ++lt;
      if (lt >= 3) {
        note_launch();
        launch(E.p == PM ? k_l2l_chain<PM, true> : k_l2l_chain<PM, false>,
               nblk(1ll << (2 * lt), 128), 128, 0, st, lt, T.box_cx.as<double>(),
               T.box_cy.as<double>(), E.local.as<double2>(), E.p);
        l_first = lt;
        E.l2l_chain_lt = lt;
      }
    }
    for (int l = l_first; l < T.L; ++l) {
      const long long c0 = part.lo(l + 1), c1 = part.hi(l + 1);
      note_launch();
      launch(E.p == PM ? k_l2l<PM, true> : k_l2l<PM, false>, nblk(c1 - c0, 128), 128, 0, st, l,
             c0, c1, T.box_cx.as<double>(),
                                                    T.box_cy.as<double>(), E.local.as<double2>(),
                                                    E.p);
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
                DevStatus* dstat, cudaStream_t st, const Part& part, int which) {
  dispatch_p(E.p, [&](auto pm) {
    Launch<decltype(pm)::value>::upward(T, Ls, E, offL, dstat, st, part, which);
  });
}
void run_m2m(const TreeState& T, ExpState& E, cudaStream_t st, const Part& part, int lmin,
             int lmax) {
  if (lmax < 0) lmax = T.L - 1;
  dispatch_p(E.p, [&](auto pm) { Launch<decltype(pm)::value>::m2m(T, E, st, part, lmin, lmax); });
}
void run_m2l(const TreeState& T, const ListState& Ls, ExpState& E, DevStatus* dstat,
             cudaStream_t st) {
  dispatch_p(E.p, [&](auto pm) { Launch<decltype(pm)::value>::m2l(T, Ls, E, dstat, st); });
}
void run_l2l(const TreeState& T, ExpState& E, DevStatus* dstat, cudaStream_t st,
             const Part& part) {
  (void)dstat;
  dispatch_p(E.p, [&](auto pm) { Launch<decltype(pm)::value>::l2l(T, E, st, part); });
}
void complete_chained_locals(const TreeState& T, ExpState& E, double2* out, cudaStream_t st) {
  const int lt = E.l2l_chain_lt;
  if (lt < 3) return;
  dispatch_p(E.p, [&](auto pm) {
    constexpr int PM = decltype(pm)::value;
    for (int l = 1; l + 1 < lt; ++l) {   // children at levels 2..lt-1, level by level
      note_launch();
      launch(E.p == PM ? k_l2l<PM, true> : k_l2l<PM, false>, nblk(1ll << (2 * (l + 1)), 128),
             128, 0, st, l, 0ll, 1ll << (2 * (l + 1)), T.box_cx.as<double>(),
             T.box_cy.as<double>(), out, E.p);
    }
  });
}

void run_l2p_m2p(const TreeState& T, const ListState& Ls, ExpState& E, DevStatus* dstat,
                 cudaStream_t st, long long e0, long long e1, long long leaf_range_lo,
                 long long leaf_range_hi) {
  if (e1 < 0) e1 = T.m;
  if (T.L == 0) {   // a single box: no expansions (engine.py:257)
    FMM_CUDA(cudaMemsetAsync(E.phi.p, 0, sizeof(double2) * T.m, st));
    return;
  }
  if (e1 <= e0) return;
  dispatch_p(E.p, [&](auto pm) {
    note_launch();
    constexpr int PMv = decltype(pm)::value;
    const bool ex = E.p == PMv;         // exact order: no per-coefficient range tests
    launch(ex ? k_l2p_m2p<PMv, true> : k_l2p_m2p<PMv, false>, nblk(e1 - e0, 128), 128, 0, st,
        T.m, e0, e1, T.L, T.eleaf_t, T.epos_t, Ls.m2p_off.as<int>(), Ls.m2p_idx.as<int>(),
        T.box_cx.as<double>(), T.box_cy.as<double>(), E.mult.as<double2>(),
        E.local.as<double2>(), E.phi.as<double2>(), E.p, dstat);
    // leaves of the evaluated range with long m2p lists
    const long long nleaf = 1ll << (2 * T.L);
    long long b0 = 0, b1 = nleaf;
    if (e0 > 0 || e1 < T.m) {          // distributed rank: its leaves
      b0 = leaf_range_lo;
      b1 = leaf_range_hi;
    }
    E.long_list.reserve(sizeof(int) * (nleaf + 2));
    int* cnt = E.long_list.as<int>() + nleaf;
    FMM_CUDA(cudaMemsetAsync(cnt, 0, sizeof(int), st));
    note_launch();
    launch(k_m2p_find_long, nblk(b1 - b0, 256), 256, 0, st, b0, b1, Ls.m2p_off.as<int>(),
                                                        E.long_list.as<int>(), cnt);
    note_launch();
    launch(ex ? k_m2p_long<PMv, true> : k_m2p_long<PMv, false>, 2 * 148, M2P_LONG_THREADS, 0, st,
        T.L, E.long_list.as<int>(), cnt, T.eoff_t, T.epos_t, Ls.m2p_off.as<int>(),
        Ls.m2p_idx.as<int>(), T.box_cx.as<double>(), T.box_cy.as<double>(),
        E.mult.as<double2>(), E.phi.as<double2>(), E.p, dstat);
  });
}

}  // namespace fmm
