// Near field ("p2p" phase) with the un-permute fused into its epilogue, and
// the all-pairs direct sum.
//
// Reference: engine.py:163-182 (_p2p_phase), operators.py:258-292
// (reciprocal_parts / kernel_block), engine.py:266-267 (values[eval_perm] =
// phi), engine.py:282-300 (direct_evaluate).  Kernel G = g/(z_s - y) in real
// arithmetic: dx = x_s - x_y, dy = y_s - y_y, s = 1/(dx^2+dy^2),
// phi += g*dx*s - i*g*dy*s; exact coincidence (r2 == 0) contributes nothing
// and is counted.
//
// One warp per target leaf.  A leaf's points are spread over the lanes in
// groups: with n_e points in the current block of <= 32, G = 32 / n_e lanes
// share each point and stride the near sources; the G partial sums are then
// combined in fixed lane order, so results are deterministic.
#include "engine.h"

#include <algorithm>
#include <cstdlib>
#include <string>

namespace fmm {

namespace {

constexpr int P2P_WARPS = 4;
constexpr int P2P_THREADS = 32 * P2P_WARPS;
// near sources staged per warp per round: 256 for leaves of <= 32 points
// (C2: ~210 near sources per leaf, one round), 512 for the two-block kernel
// (C5: ~510 per leaf -- one staging round trip instead of two; 48 KB of SMEM
// per CTA; measured C5 P2P 4.12 -> 3.88 ms, C2 unchanged with 256).  The
// compute consumes every round in 256-source sub-chunks (same sums).
constexpr int P2P_CHUNK1 = 256, P2P_CHUNK2 = 512;
#ifndef P2P_SCAN
#define P2P_SCAN 1
#endif
#ifndef P2P_HI
#define P2P_HI 1
#endif
#ifndef P2P_EXACT
#define P2P_EXACT 0
#endif
#ifndef P2P_FAST
#define P2P_FAST 1
#endif


__device__ __forceinline__ void cp_async16(void* smem, const void* gmem) {
  const unsigned s = (unsigned)__cvta_generic_to_shared(smem);
  asm volatile("cp.async.ca.shared.global [%0], [%1], 16;\n" ::"r"(s), "l"(gmem));
}
__device__ __forceinline__ void cp_async8(void* smem, const void* gmem) {
  const unsigned s = (unsigned)__cvta_generic_to_shared(smem);
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(s), "l"(gmem));
}
__device__ __forceinline__ void cp_async_wait_all() {
  asm volatile("cp.async.wait_all;\n" ::: "memory");
}

// 1/x for x > 0 to ~1 ulp: MUFU.RCP64H seed (~23 bits), then one cubic
// Newton step y(1 + e + e^2), e = 1 - x y  (3 DFMA; error ~ e^3)
__device__ __forceinline__ double rcp_nr(double x) {
  double y;
  asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(x));
  const double e = fma(-x, y, 1.0);
  return fma(fma(e, e, e), y, y);
}

// One near-field interaction of source (z, g) with target y.  Exact
// coincidence (r2 == 0, hence dx == dy == 0) contributes nothing and is
// counted (operators.py:266-274); it is detected on the bit pattern of r2
// and handled by evaluating 1/1 instead of 1/0, so the loop has no branch
// and no FP64 compare: g * 1 * dx = 0 exactly.
__device__ __forceinline__ void p2p_term(double zx, double zy, double g, double yx, double yy,
                                         double& bx, double& by, int& skips) {
  const double dx = zx - yx, dy = zy - yy;
#if P2P_EXACT
  // the reference's rounding sequence (operators.py:265-272, 291): r2 = dx*dx;
  // r2 += dy*dy (two rounded products, one rounded add); s = 1/r2; the dot
  // product accumulates (dx*s)*g; only r2 == 0 is skipped
  const double r2 = __dadd_rn(__dmul_rn(dx, dx), __dmul_rn(dy, dy));
  const bool zero = r2 == 0.0;
  skips += zero;
#if P2P_EXACT > 1
  const double s = __drcp_rn(zero ? 1.0 : r2);
#else
  // MUFU seed (1/1 for a zero high word) + one cubic Newton step
  int hi = __double2hiint(r2);
  hi = hi == 0 ? 1072693248 : hi;
  double y;
  asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(__hiloint2double(hi, 0)));
  const double e = fma(-r2, y, 1.0);
  const double s = fma(fma(e, e, e), y, y);
#endif
  bx = fma(__dmul_rn(dx, s), g, bx);
  by = fma(__dmul_rn(dy, s), g, by);
#else
  double r2 = fma(dx, dx, dy * dy);
#if P2P_HI
  // r2 >= 0, so its high word is zero only for 0 or a denormal (which
  // rcp.approx.ftz cannot invert either): one 32-bit test selects the seed
  // of 1/1 instead; the Newton step then sees r2 = 0 and returns 3 y, a
  // finite factor on dx = dy = 0.  The skip count (operators.py:266-274) is
  // exactly r2 == 0: both words zero, one predicated add.
  int hi = __double2hiint(r2);
  const int lo = __double2loint(r2);
  asm("{\n\t.reg .pred z, c;\n\t.reg .b32 t;\n\tor.b32 t, %1, %2;\n\t"
      "setp.eq.s32 c, t, 0;\n\t@c add.s32 %0, %0, 1;\n\t"
      "setp.eq.s32 z, %1, 0;\n\tselp.b32 %1, 1072693248, %1, z;\n\t}"
      : "+r"(skips), "+r"(hi) : "r"(lo));
  double y;
  asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(__hiloint2double(hi, 0)));
  const double e = fma(-r2, y, 1.0);
  const double gs = g * fma(fma(e, e, e), y, y);
#else
  const long long bits = __double_as_longlong(r2);
  const bool zero = bits == 0;
  skips += zero;
  r2 = zero ? 1.0 : r2;
  const double gs = g * rcp_nr(r2);
#endif
  bx = fma(gs, dx, bx);
  by = fma(gs, dy, by);
#endif
}

// The same interaction without the coincidence test, for evaluations whose
// only coincident pairs are the points with themselves (aliased evaluation
// points, no two sources at one position: the tree's x tie pass checked,
// ST_DUPLICATES clear); the host counts those M skips.  The MUFU seed is taken
// from max(hi(r2), hi(2^-303)): unchanged for every r2 >= 2^-303, and for
// r2 == 0 (dx == dy == 0) a finite s ~ 5e91, so g s dx == 0 exactly.  The
// seed's low word is the (dead) seed input instead of zero: < 2^-20 relative
// on a ~2^-22 seed, which the cubic step takes below 2^-59.  14 instructions,
// 10 of them FP64, instead of 17.
__device__ __forceinline__ void p2p_term_fast(double zx, double zy, double g, double yx,
                                              double yy, double& bx, double& by) {
  const double dx = zx - yx, dy = zy - yy;
  const double r2 = fma(dx, dx, dy * dy);
  double y;
  asm("{\n\t.reg .b32 h, q, h2, q2;\n\t.reg .b64 s, t;\n\t"
      "mov.b64 {q, h}, %1;\n\t"
      "max.s32 h, h, 0x2d000000;\n\t"
      "mov.b64 s, {q, h};\n\t"
      "rcp.approx.ftz.f64 t, s;\n\t"
      "mov.b64 {q2, h2}, t;\n\t"
      "mov.b64 %0, {h, h2};\n\t}"
      : "=d"(y) : "d"(r2));
  const double e = fma(-r2, y, 1.0);
  const double gs = g * fma(fma(e, e, e), y, y);
  bx = fma(gs, dx, bx);
  by = fma(gs, dy, by);
}

// sum of the staged sources [j0, j1) on target y into (ax, ay): 4-way
// unrolled, two accumulator pairs, fixed order
template <bool FAST>
__device__ __forceinline__ void p2p_slice(const double2* sp, const double* sg, int j0, int j1,
                                          double2 y, double& ax, double& ay, int& skips) {
  const double2* zp = sp + j0;
  const double* gp = sg + j0;
  const int n = j1 - j0;
  double bx0 = 0.0, by0 = 0.0, bx1 = 0.0, by1 = 0.0;
  int j = 0;
  for (; j + 4 <= n; j += 4) {
    const double2 z0 = zp[j], z1 = zp[j + 1], z2 = zp[j + 2], z3 = zp[j + 3];
    const double g0 = gp[j], g1 = gp[j + 1], g2 = gp[j + 2], g3 = gp[j + 3];
    if (FAST) {
      p2p_term_fast(z0.x, z0.y, g0, y.x, y.y, bx0, by0);
      p2p_term_fast(z1.x, z1.y, g1, y.x, y.y, bx1, by1);
      p2p_term_fast(z2.x, z2.y, g2, y.x, y.y, bx0, by0);
      p2p_term_fast(z3.x, z3.y, g3, y.x, y.y, bx1, by1);
    } else {
      p2p_term(z0.x, z0.y, g0, y.x, y.y, bx0, by0, skips);
      p2p_term(z1.x, z1.y, g1, y.x, y.y, bx1, by1, skips);
      p2p_term(z2.x, z2.y, g2, y.x, y.y, bx0, by0, skips);
      p2p_term(z3.x, z3.y, g3, y.x, y.y, bx1, by1, skips);
    }
  }
  for (; j < n; ++j) {
    const double2 z = zp[j];
    if (FAST) p2p_term_fast(z.x, z.y, gp[j], y.x, y.y, bx0, by0);
    else p2p_term(z.x, z.y, gp[j], y.x, y.y, bx0, by0, skips);
  }
  ax += bx0 + bx1;
  ay += by0 + by1;
}

// One warp per target leaf.  The leaf's near sources (the concatenated source
// ranges of its p2p boxes, ascending) are staged into a per-warp SMEM buffer
// with cp.async; the box table (ids, ranges) is fetched once per 32 boxes
// with coalesced loads and a warp scan of the counts maps every staged slot
// to its box, so staging costs one copy per lane per 32 sources and no
// dependent global round trips per box.  With n_e points in the current
// block of <= 32, G = 32/n_e lane groups share each point; group k sums a
// CONTIGUOUS slice of the staged sources (immediate-offset SMEM reads,
// 4-way unrolled, two accumulator pairs), then the G partial sums are folded
// in fixed lane order -- deterministic, no atomics on values.
template <bool DUAL, bool FAST>
__global__ void __launch_bounds__(P2P_THREADS)
k_p2p(long long b0, long long b1, const int* __restrict__ soff, const int* __restrict__ eoff,
      const int* __restrict__ n_off, const int* __restrict__ n_idx,
      const double2* __restrict__ src_pos, const double* __restrict__ src_g,
      const double2* __restrict__ eval_pos, const int* __restrict__ eval_perm,
      const double2* __restrict__ phi_in, double2* values, long long out_base, DevStatus* st) {
  pdl_enter();
  constexpr int P2P_CHUNK = DUAL ? P2P_CHUNK2 : P2P_CHUNK1;
  __shared__ double2 s_pos[P2P_WARPS][P2P_CHUNK];
  __shared__ double s_g[P2P_WARPS][P2P_CHUNK];
  const long long b = b0 + ((blockIdx.x * (long long)blockDim.x + threadIdx.x) >> 5);
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  if (b >= b1) return;
  // one round trip for the status word and the leaf's point / near-box ranges
  const int flags = status_flags(st);
  const int e0 = eoff[b], e1 = eoff[b + 1];
  const int q0 = n_off[b], q1 = n_off[b + 1];
  if ((flags & ST_OVERFLOW) || e0 == e1) return;
  double2* sp = s_pos[w];
  double* sg = s_g[w];
  int skips = 0;
  // FAST: no per-pair coincidence test unless the tree found duplicate
  // sources; the leaf's points meet only themselves (e1 - e0 skips)
  const bool fast = FAST && !(flags & ST_DUPLICATES);
  if (fast && lane == 0) skips = e1 - e0;
  // DUAL: up to 64 points per pass -- block A (<= 32 points, G lane groups)
  // and, for leaves of 33..64 points, block B (the rest, GB groups) share
  // every staged chunk, so the near sources are staged once per 64 points
  for (int eb = e0; eb < e1; eb += DUAL ? 64 : 32) {
    const int neB = DUAL ? max(0, min(32, e1 - eb - 32)) : 0;
    const int GB = neB ? 32 / neB : 1;
    const bool activeB = neB && lane < GB * neB;
    const int eiB = neB ? lane % neB : 0, grpB = activeB ? lane / neB : 0;
    const double2 yB = activeB ? eval_pos[eb + 32 + eiB] : make_double2(0.0, 0.0);
    double axB = 0.0, ayB = 0.0;
    const int ne = min(32, e1 - eb);
    const int G = 32 / ne;
    const bool active = lane < G * ne;
    const int ei = lane % ne, grp = active ? lane / ne : 0;
    const double2 y = eval_pos[eb + ei];
    double ax = 0.0, ay = 0.0;
    // epilogue operands fetched now, landing while the pass computes
    const bool lead = active && grp == 0;
    const double2 fA = lead && phi_in ? phi_in[eb + ei] : make_double2(0.0, 0.0);
    const long long dA = !lead ? 0 : eval_perm ? (long long)eval_perm[eb + ei] : eb + ei - out_base;
    // walk the near boxes 32 at a time; (qb, ib) = next box and offset inside it
    int qb = q0, ib = 0;
    while (qb < q1) {
      int fill = 0;
#if P2P_SCAN
      // one group of <= 32 boxes per step: lane k holds box k's range, an
      // inclusive warp scan of the counts maps every staged slot to its box
      // (5-step shuffle search), so each lane issues one copy per 32 sources
      // instead of the warp walking the boxes one by one
      while (qb < q1 && fill < P2P_CHUNK) {
        const int nq = min(32, q1 - qb);
        int bs0 = 0, bcnt = 0;
        if (lane < nq) {
          const int a = n_idx[qb + lane];
          bs0 = soff[a];
          bcnt = soff[a + 1] - bs0;
          if (lane == 0) { bs0 += ib; bcnt -= ib; }
        }
        int incl = bcnt;
#pragma unroll
        for (int d = 1; d < 32; d <<= 1) {
          const int v = __shfl_up_sync(0xffffffffu, incl, d);
          if (lane >= d) incl += v;
        }
        const int total = __shfl_sync(0xffffffffu, incl, 31);
        const int take = min(total, P2P_CHUNK - fill);
        const int src_base = bs0 - (incl - bcnt);     // source of slot t in box k: src_base_k + t
        for (int t0 = 0; t0 < take; t0 += 32) {     // warp-uniform trip count
          const int t = t0 + lane;
          int k = 0;
#pragma unroll
          for (int st = 16; st; st >>= 1) {
            const int v = __shfl_sync(0xffffffffu, incl, k + st - 1);
            if (v <= t) k += st;
          }
          const int src = __shfl_sync(0xffffffffu, src_base, k & 31) + t;
          if (t < take) {
            cp_async16(sp + fill + t, src_pos + src);
            cp_async8(sg + fill + t, src_g + src);
          }
        }
        fill += take;
        if (take < total) {        // chunk full inside box k: resume there next round
          const unsigned over = __ballot_sync(0xffffffffu, incl > take);
          const int k = __ffs(over) - 1;
          const int excl_k = __shfl_sync(0xffffffffu, incl - bcnt, k);
          ib = (k == 0 ? ib : 0) + (take - excl_k);
          qb += k;
          break;
        }
        qb += nq;
        ib = 0;
      }
#else
      bool partial = false;
      while (qb < q1 && fill < P2P_CHUNK && !partial) {
        const int nq = min(32, q1 - qb);
        int bs0 = 0, bcnt = 0;
        if (lane < nq) {
          const int a = n_idx[qb + lane];
          bs0 = soff[a];
          bcnt = soff[a + 1] - bs0;
        }
        int k = 0;
        for (; k < nq && fill < P2P_CHUNK; ++k) {
          const int skip = k == 0 ? ib : 0;
          const int s0 = __shfl_sync(0xffffffffu, bs0, k) + skip;
          const int cnt = __shfl_sync(0xffffffffu, bcnt, k) - skip;
          const int take = min(cnt, P2P_CHUNK - fill);
          for (int t = lane; t < take; t += 32) {
            cp_async16(sp + fill + t, src_pos + s0 + t);
            cp_async8(sg + fill + t, src_g + s0 + t);
          }
          fill += take;
          if (take < cnt) {          // chunk full inside box k: resume there next round
            ib = skip + take;
            partial = true;
            break;
          }
        }
        qb += k;
        if (!partial) ib = 0;
      }
#endif
      cp_async_wait_all();
      __syncwarp();
      // the staged round is consumed in sub-chunks of P2P_CHUNK1 sources: the
      // slice boundaries, hence every point's summation order, are those of
      // 256-source rounds whatever the staging size (bit-identical results)
      for (int sub = 0; sub < fill; sub += P2P_CHUNK1) {
        const int f = min(P2P_CHUNK1, fill - sub);
        const double2* sps = sp + sub;
        const double* sgs = sg + sub;
        if (fast) {
          if (active) p2p_slice<true>(sps, sgs, f * grp / G, f * (grp + 1) / G, y, ax, ay, skips);
          // second block of points (leaves of 33..64 points): same staged chunk
          if (DUAL && activeB)
            p2p_slice<true>(sps, sgs, f * grpB / GB, f * (grpB + 1) / GB, yB, axB, ayB, skips);
        } else {
          if (active)
            p2p_slice<false>(sps, sgs, f * grp / G, f * (grp + 1) / G, y, ax, ay, skips);
          if (DUAL && activeB)
            p2p_slice<false>(sps, sgs, f * grpB / GB, f * (grpB + 1) / GB, yB, axB, ayB, skips);
        }
      }
      __syncwarp();
    }
    // fold the G lane groups of every point in fixed order
    for (int k = 1; k < G; ++k) {
      const double ox = __shfl_sync(0xffffffffu, ax, lane + k * ne);
      const double oy = __shfl_sync(0xffffffffu, ay, lane + k * ne);
      if (grp == 0) { ax += ox; ay += oy; }
    }
    // input order (engine.py:266-267), or tree order for distributed ranks
    if (lead) values[dA] = make_double2(fA.x + ax, fA.y - ay);
    if (DUAL && neB) {
      for (int k = 1; k < GB; ++k) {
        const double ox = __shfl_sync(0xffffffffu, axB, lane + k * neB);
        const double oy = __shfl_sync(0xffffffffu, ayB, lane + k * neB);
        if (grpB == 0) { axB += ox; ayB += oy; }
      }
      if (activeB && grpB == 0) {
        const int e = eb + 32 + eiB;
        const double2 f = phi_in ? phi_in[e] : make_double2(0.0, 0.0);
        values[eval_perm ? (long long)eval_perm[e] : e - out_base] =
            make_double2(f.x + axB, f.y - ayB);
      }
    }
  }
  for (int d = 16; d; d >>= 1) skips += __shfl_xor_sync(0xffffffffu, skips, d);
  if (lane == 0 && skips) atomicAdd(&st->p2p_skips, (unsigned long long)skips);
}

// all-pairs direct sum, asymmetric mode: thread per target, SMEM source tiles
constexpr int DIRECT_TILE = 256;

__global__ void __launch_bounds__(DIRECT_TILE)
k_direct(const double2* __restrict__ src, const double* __restrict__ g, long long n,
         const double2* __restrict__ tgt, long long m, double2* out) {
  pdl_enter();
  __shared__ double sx[DIRECT_TILE], sy[DIRECT_TILE], sg[DIRECT_TILE];
  const long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  const double2 y = t < m ? tgt[t] : make_double2(0.0, 0.0);
  double ax = 0.0, ay = 0.0;
  for (long long s0 = 0; s0 < n; s0 += DIRECT_TILE) {
    __syncthreads();
    const long long s = s0 + threadIdx.x;
    if (s < n) {
      const double2 z = src[s];
      sx[threadIdx.x] = z.x;
      sy[threadIdx.x] = z.y;
      sg[threadIdx.x] = g[s];
    }
    __syncthreads();
    const int cnt = (int)(n - s0 < DIRECT_TILE ? n - s0 : DIRECT_TILE);
    for (int j = 0; j < cnt; ++j) {
      const double dx = sx[j] - y.x, dy = sy[j] - y.y;
      const double r2 = fma(dx, dx, dy * dy);
      if (r2 != 0.0) {
        const double gs = sg[j] / r2;
        ax = fma(gs, dx, ax);
        ay = fma(gs, dy, ay);
      }
    }
  }
  if (t < m) out[t] = make_double2(ax, -ay);
}

// Symmetric direct sum (engine.py:302-323, evaluation points aliasing the
// sources): every unordered pair shares one reciprocal between its two
// directions, 13 FP64 instructions per pair instead of 2 x 10.  The point
// set is cut into nbs super-tiles of ST points; CTA (I, J), I < J, sums J
// into I's points and I into J's, CTA (I, I) sums its tile asymmetrically.
// Each CTA writes its partial potentials into its own slots of W[nbs][n]
// (W[J][i]: super-tile J's contribution to point i), and k_direct_fold adds
// a point's nbs slots in ascending J: deterministic, no atomics.
//
// Inside a CTA (8 warps, one i per thread): a 256-point j-chunk is staged in
// SMEM; in 8 sub-steps warp w takes j-block (w + s) & 7, so each j-block is
// owned by one warp at a time.  Lane l pairs its i with j = (l + k) & 31 at
// step k and holds that j's accumulator, handed one lane down after the
// step (lane l + 1's j is lane l's next): j's terms arrive in a fixed order.
// The reciprocal is the P2P's (rcp.approx seed, one cubic Newton step;
// r2 == 0 gives a finite seed and dx == dy == 0, so a coincident pair adds
// exact zeros, the reference's skip).
constexpr int DSYM_THREADS = 256;
#ifndef DSYM_NI
#define DSYM_NI 2           // i's per thread
#endif
#ifndef DSYM_MAX_TILES
#define DSYM_MAX_TILES 128
#endif

__device__ __forceinline__ double rcp_r2(double r2) {
  double y;
  asm("{\n\t.reg .b32 h, q, h2, q2;\n\t.reg .b64 s, t;\n\t"
      "mov.b64 {q, h}, %1;\n\t"
      "max.s32 h, h, 0x2d000000;\n\t"
      "mov.b64 s, {q, h};\n\t"
      "rcp.approx.ftz.f64 t, s;\n\t"
      "mov.b64 {q2, h2}, t;\n\t"
      "mov.b64 %0, {h, h2};\n\t}"
      : "=d"(y) : "d"(r2));
  const double e = fma(-r2, y, 1.0);
  return fma(fma(e, e, e), y, y);
}

__global__ void __launch_bounds__(DSYM_THREADS)
k_direct_sym(const double2* __restrict__ z, const double* __restrict__ g, long long n,
             long long ST, double2* __restrict__ W) {
  pdl_enter();
  const int I = blockIdx.y, J = blockIdx.x;
  if (J < I) return;
  __shared__ double2 s_z[DSYM_THREADS];
  __shared__ double s_g[DSYM_THREADS];
  __shared__ double2 s_acc[DSYM_THREADS];
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  const long long I0 = I * ST, I1 = min(n, I0 + ST), J0 = J * ST, J1 = min(n, J0 + ST);
  // DSYM_NI i's per thread (i-chunk DSYM_NI * 256): each staged j and each
  // accumulator hand-off serves DSYM_NI pairs
  for (long long ic = I0; ic < I1; ic += DSYM_NI * DSYM_THREADS) {
    double2 zi[DSYM_NI];
    double gi[DSYM_NI], ax[DSYM_NI], ay[DSYM_NI];
#pragma unroll
    for (int u = 0; u < DSYM_NI; ++u) {
      const long long i = ic + u * DSYM_THREADS + tid;
      zi[u] = i < I1 ? z[i] : make_double2(0.0, 0.0);
      gi[u] = i < I1 ? g[i] : 0.0;
      ax[u] = ay[u] = 0.0;
    }
    for (long long jc = J0; jc < J1; jc += DSYM_THREADS) {
      const long long j = jc + tid;
      const bool vj = j < J1;
      __syncthreads();
      s_z[tid] = vj ? z[j] : make_double2(0.0, 0.0);
      s_g[tid] = vj ? g[j] : 0.0;
      if (I != J) s_acc[tid] = (ic == I0 || !vj) ? make_double2(0.0, 0.0)
                                                 : W[(long long)I * n + j];
      __syncthreads();
      if (I == J) {
        // diagonal super-tile: asymmetric, each i over the whole chunk
#pragma unroll
        for (int u = 0; u < DSYM_NI; ++u) {
          double bx = 0.0, by = 0.0;
#pragma unroll 4
          for (int k = 0; k < DSYM_THREADS; ++k) {
            const double2 zj = s_z[k];
            const double dx = zj.x - zi[u].x, dy = zj.y - zi[u].y;
            const double y = rcp_r2(fma(dx, dx, dy * dy)) * s_g[k];
            bx = fma(y, dx, bx);
            by = fma(y, dy, by);
          }
          ax[u] += bx;
          ay[u] += by;
        }
        continue;
      }
      for (int sb = 0; sb < 8; ++sb) {
        const int base = ((wid + sb) & 7) * 32;
        double2 aj = s_acc[base + lane];
#pragma unroll 8
        for (int k = 0; k < 32; ++k) {
          const int jj = base + ((lane + k) & 31);
          const double2 zj = s_z[jj];
          const double gj = s_g[jj];
#pragma unroll
          for (int u = 0; u < DSYM_NI; ++u) {
            const double dx = zj.x - zi[u].x, dy = zj.y - zi[u].y;
            const double y = rcp_r2(fma(dx, dx, dy * dy));
            const double re = dx * y, im = dy * y;
            ax[u] = fma(gj, re, ax[u]);
            ay[u] = fma(gj, im, ay[u]);
            aj.x = fma(-gi[u], re, aj.x);
            aj.y = fma(-gi[u], im, aj.y);
          }
          aj.x = __shfl_sync(0xffffffffu, aj.x, lane + 1);
          aj.y = __shfl_sync(0xffffffffu, aj.y, lane + 1);
        }
        s_acc[base + lane] = aj;
        __syncthreads();
      }
      if (vj) W[(long long)I * n + j] = s_acc[tid];
    }
#pragma unroll
    for (int u = 0; u < DSYM_NI; ++u) {
      const long long i = ic + u * DSYM_THREADS + tid;
      if (i < I1) W[(long long)J * n + i] = make_double2(ax[u], ay[u]);
    }
  }
}

// phi_i = sum over super-tiles J (ascending) of W[J][i]; conjugate at the end
__global__ void k_direct_fold(const double2* __restrict__ W, long long n, int nbs,
                              double2* __restrict__ out) {
  pdl_enter();
  const long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (i >= n) return;
  double ax = 0.0, ay = 0.0;
  for (int J = 0; J < nbs; ++J) {
    const double2 v = W[(long long)J * n + i];
    ax += v.x;
    ay += v.y;
  }
  out[i] = make_double2(ax, -ay);
}

inline unsigned nblk(long long n, int t) { return (unsigned)((n + t - 1) / t); }

}  // namespace

void run_p2p(const TreeState& T, const ListState& Ls, ExpState& E, const int* offL,
             double2* values, DevStatus* dstat, cudaStream_t st, const Part& part,
             long long out_base) {
  const long long b0 = part.lo(T.L), b1 = part.hi(T.L);
  // leaves of more than 32 points (mean evaluation points per leaf): the
  // two-block kernel stages each leaf's near sources once per 64 points; the
  // one-block kernel keeps fewer registers for the common <= 32-point leaves
  const long long nleaf = 1ll << (2 * T.L);
  const bool dual = (T.m + nleaf - 1) / nleaf > 32;
  const int* eperm = out_base >= 0 ? nullptr : T.eperm_t;
  const double2* phi_in = E.phi.as<double2>();
  // fast interaction loop: aliased evaluation points on a single-GPU tree whose
  // x tie pass checked for duplicate sources (else the per-pair r2 == 0 test)
  const bool fast = P2P_FAST && T.aliased && T.dup_checked && part.G == 1;
  auto kern = dual ? (fast ? k_p2p<true, true> : k_p2p<true, false>)
                   : (fast ? k_p2p<false, true> : k_p2p<false, false>);
  note_launch();
  launch(kern, nblk((b1 - b0) * 32, P2P_THREADS), P2P_THREADS, 0,
         st, b0, b1, offL, T.eoff_t, Ls.p2p_off.as<int>(), Ls.p2p_idx.as<int>(),
         T.src_pos.as<double2>(), T.src_g.as<double>(), T.epos_t, eperm, phi_in,
         values, out_base, dstat);
}

void run_direct(const double2* src, const double* g, int64_t n, const double2* tgt, int64_t m,
                double2* out, cudaStream_t st) {
  note_launch();
  launch(k_direct, nblk(m, DIRECT_TILE), DIRECT_TILE, 0, st, src, g, n, tgt, m, out);
}

long long direct_sym_tiles(int64_t n, int64_t* st_out) {
  // super-tiles: a multiple of the i-chunk, >= 512 points, at most
  // DSYM_MAX_TILES of them (up to 8256 CTAs of equal work; W costs
  // n * nbs * 16 bytes)
  constexpr long long CH = DSYM_NI * DSYM_THREADS;
  const long long ST = std::max<long long>(
      512, ((n + DSYM_MAX_TILES - 1) / DSYM_MAX_TILES + CH - 1) / CH * CH);
  if (st_out) *st_out = ST;
  return (n + ST - 1) / ST;
}

void run_direct_symmetric(const double2* src, const double* g, int64_t n, double2* W,
                          double2* out, cudaStream_t st) {
  if (n <= 0) return;
  int64_t ST = 0;
  const long long nbs = direct_sym_tiles(n, &ST);
  note_launch();
  launch(k_direct_sym, dim3((unsigned)nbs, (unsigned)nbs), DSYM_THREADS, 0, st, src, g,
         (long long)n, (long long)ST, W);
  note_launch();
  launch(k_direct_fold, nblk(n, 256), 256, 0, st, W, (long long)n, (int)nbs, out);
}

}  // namespace fmm
