// Near field ("p2p" phase) with the un-permute fused into its epilogue, and
// the all-pairs direct sum.
//
// Reference: engine.py:163-182 (_p2p_phase), operators.py:389-423
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

namespace fmm {

namespace {

constexpr int P2P_WARPS = 4;
constexpr int P2P_THREADS = 32 * P2P_WARPS;
constexpr int P2P_CHUNK = 256;      // near sources staged per warp per round

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

// 1/r2 to ~1 ulp: MUFU reciprocal seed + two Newton steps on the FP64 pipe
__device__ __forceinline__ double rcp_nr(double x) {
  double y;
  asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(x));
  double e = fma(-x, y, 1.0);
  y = fma(y, e, y);
  e = fma(-x, y, 1.0);
  return fma(y, e, y);
}

// One warp per target leaf.  The leaf's near sources (the concatenated source
// ranges of its p2p boxes, ascending) are staged into a per-warp SMEM buffer
// with cp.async, then every lane streams them from SMEM (broadcast reads).
__global__ void __launch_bounds__(P2P_THREADS)
k_p2p(int L, const int* __restrict__ soff, const int* __restrict__ eoff,
      const int* __restrict__ n_off, const int* __restrict__ n_idx,
      const double2* __restrict__ src_pos, const double* __restrict__ src_g,
      const double2* __restrict__ eval_pos, const int* __restrict__ eval_perm,
      const double2* __restrict__ phi_in, double2* values, DevStatus* st) {
  __shared__ double2 s_pos[P2P_WARPS][P2P_CHUNK];
  __shared__ double s_g[P2P_WARPS][P2P_CHUNK];
  const long long b = (blockIdx.x * (long long)blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  if (b >= (1ll << (2 * L)) || lists_overflowed(st)) return;
  const int e0 = eoff[b], e1 = eoff[b + 1];
  if (e0 == e1) return;
  const int q0 = n_off[b], q1 = n_off[b + 1];
  double2* sp = s_pos[w];
  double* sg = s_g[w];
  unsigned long long skips = 0;
  for (int eb = e0; eb < e1; eb += 32) {
    const int ne = min(32, e1 - eb);
    const int G = 32 / ne;
    const bool active = lane < G * ne;
    const int ei = lane % ne, grp = lane / ne;
    double ax = 0.0, ay = 0.0;
    const double2 y = eval_pos[eb + ei];
    int q = q0, in_box = 0;
    while (q < q1) {
      // stage the next chunk of the concatenated near-source list
      int fill = 0;
      while (q < q1 && fill < P2P_CHUNK) {
        const int a = n_idx[q];
        const int s0 = soff[a] + in_box, s1 = soff[a + 1];
        const int take = min(s1 - s0, P2P_CHUNK - fill);
        for (int t = lane; t < take; t += 32) {
          cp_async16(sp + fill + t, src_pos + s0 + t);
          cp_async8(sg + fill + t, src_g + s0 + t);
        }
        fill += take;
        if (s0 + take == s1) { ++q; in_box = 0; } else { in_box += take; }
      }
      cp_async_wait_all();
      __syncwarp();
      if (active) {
        // four independent accumulator chains (fixed order, deterministic)
        double bx[4] = {0.0, 0.0, 0.0, 0.0}, by[4] = {0.0, 0.0, 0.0, 0.0};
        int j = grp;
        for (; j + 3 * G < fill; j += 4 * G) {
#pragma unroll
          for (int u = 0; u < 4; ++u) {
            const double2 z = sp[j + u * G];
            const double dx = z.x - y.x, dy = z.y - y.y;
            const double r2 = fma(dx, dx, dy * dy);
            const bool coincide = r2 == 0.0;
            skips += coincide;
            const double gs = coincide ? 0.0 : sg[j + u * G] * rcp_nr(r2);
            bx[u] = fma(gs, dx, bx[u]);
            by[u] = fma(gs, dy, by[u]);
          }
        }
        for (; j < fill; j += G) {
          const double2 z = sp[j];
          const double dx = z.x - y.x, dy = z.y - y.y;
          const double r2 = fma(dx, dx, dy * dy);
          const bool coincide = r2 == 0.0;
          skips += coincide;
          const double gs = coincide ? 0.0 : sg[j] * rcp_nr(r2);
          bx[0] = fma(gs, dx, bx[0]);
          by[0] = fma(gs, dy, by[0]);
        }
        ax += (bx[0] + bx[1]) + (bx[2] + bx[3]);
        ay += (by[0] + by[1]) + (by[2] + by[3]);
      }
      __syncwarp();
    }
    // fold the G lane groups of every point in fixed order
    for (int q = 1; q < G; ++q) {
      const double ox = __shfl_sync(0xffffffffu, ax, lane + q * ne);
      const double oy = __shfl_sync(0xffffffffu, ay, lane + q * ne);
      if (grp == 0) { ax += ox; ay += oy; }
    }
    if (active && grp == 0) {
      const int e = eb + ei;
      const double2 f = phi_in ? phi_in[e] : make_double2(0.0, 0.0);
      values[eval_perm[e]] = make_double2(f.x + ax, f.y - ay);
    }
  }
  for (int d = 16; d; d >>= 1) skips += __shfl_xor_sync(0xffffffffu, skips, d);
  if (lane == 0 && skips) atomicAdd(&st->p2p_skips, skips);
}

// all-pairs direct sum, asymmetric mode: thread per target, SMEM source tiles
constexpr int DIRECT_TILE = 256;

__global__ void __launch_bounds__(DIRECT_TILE)
k_direct(const double2* __restrict__ src, const double* __restrict__ g, long long n,
         const double2* __restrict__ tgt, long long m, double2* out) {
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

inline unsigned nblk(long long n, int t) { return (unsigned)((n + t - 1) / t); }

}  // namespace

void run_p2p(const TreeState& T, const ListState& Ls, ExpState& E, const int* offL,
             double2* values, DevStatus* dstat, cudaStream_t st) {
  const long long nleaf = 1ll << (2 * T.L);
  note_launch();
  k_p2p<<<nblk(nleaf * 32, P2P_THREADS), P2P_THREADS, 0, st>>>(
      T.L, offL, T.eval_leaf_off.as<int>(), Ls.p2p_off.as<int>(), Ls.p2p_idx.as<int>(),
      T.src_pos.as<double2>(), T.src_g.as<double>(), T.eval_pos.as<double2>(),
      T.eval_perm.as<int>(), E.phi.as<double2>(), values, dstat);
}

void run_direct(const double2* src, const double* g, int64_t n, const double2* tgt, int64_t m,
                double2* out, cudaStream_t st) {
  note_launch();
  k_direct<<<nblk(m, DIRECT_TILE), DIRECT_TILE, 0, st>>>(src, g, n, tgt, m, out);
}

}  // namespace fmm
