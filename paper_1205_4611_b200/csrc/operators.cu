// Unit-level expansion operators and per-level connectivity on the GPU: the
// reference's public building blocks (fmm2d.operators, operators.py:63-297;
// fmm2d.connectivity.classify_level / reclassify_finest, connectivity.py:47-96)
// as batched kernels behind the C ABI, for callers that drive the algorithm
// piecewise (the reference's own unit tests, experiments).  The fused engine
// (fmm2d.cu) does not use them.
//
// Arithmetic mirrors numpy's element semantics: complex multiply as
// (ac - bd, ad + bc) without contraction, complex division by Smith's
// algorithm (numpy's npymath), cascades in the reference's exact loop order,
// any order p >= 1 (coefficients live in global memory; one thread per batch
// row).  Summations over points run sequentially in point order (numpy's
// pairwise np.sum and BLAS dgemv associate differently: agreement is to
// rounding, which is what the reference's own tests assert).
#include "context.h"

namespace {

using fmm::cplx;

// numpy complex multiply / divide (npy_math_complex: no FMA contraction)
__device__ __forceinline__ cplx nmul(cplx a, cplx b) {
  return cplx{__dsub_rn(__dmul_rn(a.x, b.x), __dmul_rn(a.y, b.y)),
              __dadd_rn(__dmul_rn(a.x, b.y), __dmul_rn(a.y, b.x))};
}
__device__ __forceinline__ cplx nadd(cplx a, cplx b) {
  return cplx{__dadd_rn(a.x, b.x), __dadd_rn(a.y, b.y)};
}
__device__ __forceinline__ cplx nsub(cplx a, cplx b) {
  return cplx{__dsub_rn(a.x, b.x), __dsub_rn(a.y, b.y)};
}
// Smith's algorithm as numpy's complex128 true_divide loop
__device__ __forceinline__ cplx ndiv(cplx a, cplx b) {
  const double abr = fabs(b.x), abi = fabs(b.y);
  if (abr >= abi) {
    if (abr == 0.0 && abi == 0.0) return cplx{a.x / abr, a.y / abi};
    const double rat = __ddiv_rn(b.y, b.x);
    const double scl = __ddiv_rn(1.0, __dadd_rn(b.x, __dmul_rn(b.y, rat)));
    return cplx{__dmul_rn(__dadd_rn(a.x, __dmul_rn(a.y, rat)), scl),
                __dmul_rn(__dsub_rn(a.y, __dmul_rn(a.x, rat)), scl)};
  }
  const double rat = __ddiv_rn(b.x, b.y);
  const double scl = __ddiv_rn(1.0, __dadd_rn(b.y, __dmul_rn(b.x, rat)));
  return cplx{__dmul_rn(__dadd_rn(__dmul_rn(a.x, rat), a.y), scl),
              __dmul_rn(__dsub_rn(__dmul_rn(a.y, rat), a.x), scl)};
}
// principal-branch complex log (np.log)
__device__ __forceinline__ cplx nlog(cplx z) {
  return cplx{log(hypot(z.x, z.y)), atan2(z.y, z.x)};
}
__device__ __forceinline__ cplx ld(const double2* p, long long i) {
  const double2 v = p[i];
  return cplx{v.x, v.y};
}
__device__ __forceinline__ void st(double2* p, long long i, cplx v) { p[i] = make_double2(v.x, v.y); }

constexpr double SCALED_MIN = 1e-12, SCALED_MAX = 1e12;   // operators.py:37-38

// ---------------------------------------------------------------------------
// P2M (operators.py:63-75) over boxes given by point offsets; thread per
// (box, j): w_i = g_i * c_i^(j-1) by the reference's repeated multiplication,
// a_j = -sum_i w_i.
__global__ void k_op_p2m(long long nbox, int p, const long long* off, const double2* pos,
                         const double* g, const double2* center, double2* out) {
  const long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (t >= nbox * (p + 1)) return;
  const long long b = t / (p + 1);
  const int j = int(t % (p + 1));
  if (j == 0) {
    st(out, t, cplx{0.0, 0.0});
    return;
  }
  const cplx z0 = ld(center, b);
  cplx s{0.0, 0.0};
  for (long long i = off[b]; i < off[b + 1]; ++i) {
    const cplx c = nsub(ld(pos, i), z0);
    cplx w{g[i], 0.0};
    for (int k = 1; k < j; ++k) w = nmul(w, c);
    s = nadd(s, w);
  }
  st(out, t, cplx{-s.x, -s.y});
}

// P2L (operators.py:78-93): inv_i = 1/(z_i - z0), b_k = sum_i g_i inv_i^(k+1)
__global__ void k_op_p2l(long long nbox, int p, const long long* off, const double2* pos,
                         const double* g, const double2* center, double2* out, int* flag) {
  const long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (t >= nbox * (p + 1)) return;
  const long long b = t / (p + 1);
  const int k = int(t % (p + 1));
  const cplx z0 = ld(center, b);
  cplx s{0.0, 0.0};
  for (long long i = off[b]; i < off[b + 1]; ++i) {
    const cplx d = nsub(ld(pos, i), z0);
    if (d.x == 0.0 && d.y == 0.0) {
      atomicOr(flag, 1);
      return;
    }
    const cplx inv = ndiv(cplx{1.0, 0.0}, d);
    cplx w = nmul(cplx{g[i], 0.0}, inv);
    for (int q = 0; q < k; ++q) w = nmul(w, inv);
    s = nadd(s, w);
  }
  st(out, t, s);
}

// numpy's complex / int: the int promotes to complex (j + 0i), Smith division
__device__ __forceinline__ cplx div_int(cplx a, int j) { return ndiv(a, cplx{double(j), 0.0}); }

// M2M (operators.py:100-148): thread per row; a (in/out), pw scratch
__global__ void k_op_m2m(long long rows, int p, double2* a, const double2* shift, double2* pw,
                         int variant, int any_a0) {
  const long long r = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (r >= rows) return;
  double2* A = a + r * (p + 1);
  double2* P = pw + r * (p + 1);
  const cplx rr = ld(shift, r);
  const double mag = fmm::numpy_cabs(rr.x, rr.y);
  const bool scaled = variant == 0 && mag >= SCALED_MIN && mag <= SCALED_MAX;
  const cplx a0 = ld(A, 0);
  if (scaled) {                                                  // _m2m_scaled
    cplx q{1.0, 0.0};
    for (int j = 1; j <= p; ++j) {
      q = nmul(q, rr);
      st(P, j, q);
      st(A, j, ndiv(ld(A, j), q));
    }
    for (int k = p; k >= 2; --k)
      for (int j = k; j <= p; ++j) st(A, j, nadd(ld(A, j), ld(A, j - 1)));
    for (int j = 1; j <= p; ++j) st(A, j, nmul(nsub(ld(A, j), div_int(a0, j)), ld(P, j)));
  } else {                                                       // _m2m_unscaled
    for (int k = p; k >= 2; --k)
      for (int j = k; j <= p; ++j) st(A, j, nadd(ld(A, j), nmul(rr, ld(A, j - 1))));
    if (any_a0) {
      cplx rp = rr;
      for (int j = 1; j <= p; ++j) {
        st(A, j, nsub(ld(A, j), div_int(nmul(rp, a0), j)));
        rp = nmul(rp, rr);
      }
    }
  }
}

// L2L (operators.py:151-186)
__global__ void k_op_l2l(long long rows, int p, double2* b, const double2* shift, double2* pw) {
  const long long r = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (r >= rows) return;
  double2* B = b + r * (p + 1);
  double2* P = pw + r * (p + 1);
  const cplx rr = ld(shift, r);
  const double mag = fmm::numpy_cabs(rr.x, rr.y);
  if (mag >= SCALED_MIN && mag <= SCALED_MAX) {                  // _l2l_scaled
    cplx q{1.0, 0.0};
    for (int j = 1; j <= p; ++j) {
      q = nmul(q, rr);
      st(P, j, q);
      st(B, j, nmul(ld(B, j), q));
    }
    // slice update from old values == ascending sequential update
    for (int k = 0; k <= p; ++k)
      for (int j = p - k; j < p; ++j) st(B, j, nsub(ld(B, j), ld(B, j + 1)));
    for (int j = 1; j <= p; ++j) st(B, j, ndiv(ld(B, j), ld(P, j)));
  } else {                                                       // _l2l_unscaled
    for (int k = 0; k <= p; ++k)
      for (int j = p - k; j < p; ++j) st(B, j, nsub(ld(B, j), nmul(rr, ld(B, j + 1))));
  }
}

// M2L (operators.py:189-220): a read-only, c output, pw scratch
__global__ void k_op_m2l(long long rows, int p, const double2* a, const double2* shift,
                         double2* c, double2* pw, int any_a0, int* flag) {
  const long long r = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (r >= rows) return;
  const double2* A = a + r * (p + 1);
  double2* C = c + r * (p + 1);
  double2* P = pw + r * (p + 1);
  const cplx rho = ld(shift, r);
  if (rho.x == 0.0 && rho.y == 0.0) {
    atomicOr(flag, 1);
    return;
  }
  cplx q{1.0, 0.0};
  double sign = -1.0;
  for (int j = 1; j <= p; ++j) {
    q = nmul(q, rho);
    st(P, j, q);
    const cplx t = ndiv(ld(A, j), q);
    st(C, j - 1, cplx{__dmul_rn(t.x, sign), __dmul_rn(t.y, sign)});
    sign = -sign;
  }
  st(C, p, cplx{0.0, 0.0});
  for (int k = 2; k <= p; ++k)                                   // pass 1 (old values)
    for (int j = p - k; j < p; ++j) st(C, j, nadd(ld(C, j), ld(C, j + 1)));
  for (int k = p; k >= 1; --k)                                   // pass 2 (new values)
    for (int j = k; j <= p; ++j) st(C, j, nadd(ld(C, j), ld(C, j - 1)));
  const cplx a0 = ld(A, 0);
  if (any_a0) st(C, 0, nadd(ld(C, 0), nmul(a0, nlog(cplx{-rho.x, -rho.y}))));
  for (int j = 1; j <= p; ++j) st(C, j, ndiv(nsub(ld(C, j), div_int(a0, j)), ld(P, j)));
}

// L2P (operators.py:227-234) / M2P (237-255): thread per target
__global__ void k_op_l2p(long long nt, int p, const double2* b, cplx z0, const double2* tgt,
                         double2* out) {
  const long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (i >= nt) return;
  const cplx w = nsub(ld(tgt, i), z0);
  cplx acc = ld(b, p);
  for (int j = p - 1; j >= 0; --j) acc = nadd(nmul(acc, w), ld(b, j));
  st(out, i, acc);
}

__global__ void k_op_m2p(long long nt, int p, const double2* a, cplx z0, const double2* tgt,
                         double2* out, int* flag) {
  const long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (i >= nt) return;
  const cplx u = nsub(ld(tgt, i), z0);
  if (u.x == 0.0 && u.y == 0.0) {
    atomicOr(flag, 1);
    return;
  }
  const cplx inv = ndiv(cplx{1.0, 0.0}, u);
  cplx acc = ld(a, p);
  for (int j = p - 1; j >= 1; --j) acc = nadd(nmul(acc, inv), ld(a, j));
  acc = nmul(acc, inv);
  const cplx a0 = ld(a, 0);
  if (a0.x != 0.0 || a0.y != 0.0) acc = nadd(acc, nmul(a0, nlog(u)));
  st(out, i, acc);
}

// reciprocal_parts (operators.py:258-277): r2 = dx*dx; r2 += dy*dy; s = 1/r2
// (IEEE division); coincident pairs give 0 and are counted
__global__ void k_op_recip(long long nt, long long ns, const double2* src, const double2* tgt,
                           double* re, double* im, unsigned long long* skips) {
  const long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (t >= nt * ns) return;
  const long long i = t / ns, j = t % ns;
  const double2 s = src[j], y = tgt[i];
  const double dx = __dsub_rn(s.x, y.x), dy = __dsub_rn(s.y, y.y);
  const double r2 = __dadd_rn(__dmul_rn(dx, dx), __dmul_rn(dy, dy));
  double q = 0.0;
  if (r2 == 0.0)
    atomicAdd(skips, 1ull);
  else
    q = __ddiv_rn(1.0, r2);
  re[t] = __dmul_rn(dx, q);
  im[t] = __dmul_rn(dy, q);
}

// kernel_block (operators.py:280-292): thread per target, sources in order
__global__ void k_op_kernel_block(long long nt, long long ns, const double2* src,
                                  const double* g, const double2* tgt, double2* out,
                                  unsigned long long* skips) {
  const long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (i >= nt) return;
  const double2 y = tgt[i];
  double re = 0.0, im = 0.0;
  unsigned long long sk = 0;
  for (long long j = 0; j < ns; ++j) {
    const double2 s = src[j];
    const double dx = __dsub_rn(s.x, y.x), dy = __dsub_rn(s.y, y.y);
    const double r2 = __dadd_rn(__dmul_rn(dx, dx), __dmul_rn(dy, dy));
    if (r2 == 0.0) {
      ++sk;
      continue;
    }
    const double q = __ddiv_rn(1.0, r2);
    re = __dadd_rn(re, __dmul_rn(__dmul_rn(dx, q), g[j]));
    im = __dadd_rn(im, __dmul_rn(__dmul_rn(dy, q), g[j]));
  }
  out[i] = make_double2(re, -im);
  if (sk) atomicAdd(skips, sk);
}

// ---------------------------------------------------------------------------
// classify_level (connectivity.py:47-68): candidates of box b = children of
// its parent's strong list, ascending; weak = separated.  Pass 0 counts,
// pass 1 fills the CSR in candidate order.  Thread per target box.
__device__ __forceinline__ double box_radius(const double* hw, const double* hh, long long b) {
  return fmm::glibc_hypot(hw[b], hh[b]);
}

__global__ void k_op_classify(long long nbox, const double2* c, const double* hw,
                              const double* hh, const long long* poff, const long long* pidx,
                              double theta, int pass, long long* wcnt, long long* scnt,
                              const long long* woff, long long* widx, const long long* soff,
                              long long* sidx) {
  const long long b = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (b >= nbox) return;
  const long long par = b >> 2;
  const double rb = box_radius(hw, hh, b);
  const double2 cb = c[b];
  long long nw = 0, ns = 0;
  for (long long e = poff[par]; e < poff[par + 1]; ++e) {
    for (int q = 0; q < 4; ++q) {
      const long long a = pidx[e] * 4 + q;
      const double d = fmm::numpy_cabs(__dsub_rn(cb.x, c[a].x), __dsub_rn(cb.y, c[a].y));
      if (fmm::well_separated(rb, box_radius(hw, hh, a), d, theta)) {
        if (pass) widx[woff[b] + nw] = a;
        ++nw;
      } else {
        if (pass) sidx[soff[b] + ns] = a;
        ++ns;
      }
    }
  }
  if (!pass) {
    wcnt[b] = nw;
    scnt[b] = ns;
  }
}

// reclassify_finest (connectivity.py:71-96): moved = swapped & src != b &
// r_src != r_b; larger -> p2l, smaller -> m2p, rest -> p2p
__global__ void k_op_reclassify(long long nbox, const double2* c, const double* hw,
                                const double* hh, const long long* soff, const long long* sidx,
                                double theta, int pass, long long* cnt, const long long* ooff,
                                long long* o0, long long* o1, long long* o2) {
  const long long b = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (b >= nbox) return;
  const double rb = box_radius(hw, hh, b);
  const double2 cb = c[b];
  long long n[3] = {0, 0, 0};
  for (long long e = soff[b]; e < soff[b + 1]; ++e) {
    const long long a = sidx[e];
    const double ra = box_radius(hw, hh, a);
    const double d = fmm::numpy_cabs(__dsub_rn(cb.x, c[a].x), __dsub_rn(cb.y, c[a].y));
    const bool moved = fmm::well_separated_swapped(rb, ra, d, theta) && a != b && ra != rb;
    const int k = !moved ? 0 : (ra > rb ? 1 : 2);
    if (pass) (k == 0 ? o0 : k == 1 ? o1 : o2)[ooff[3 * b + k] + n[k]] = a;
    ++n[k];
  }
  if (!pass)
    for (int k = 0; k < 3; ++k) cnt[3 * b + k] = n[k];
}

inline unsigned blocks(long long n, int t = 256) { return unsigned((n + t - 1) / t); }

struct Scratch {
  fmm::DBuf bufs[16];
  int i = 0;
  template <class T> T* get(size_t count) {
    fmm::DBuf& b = bufs[i++];
    b.reserve(sizeof(T) * (count ? count : 1));
    return b.as<T>();
  }
};

template <class T> T* up(Scratch& s, const T* h, size_t n, cudaStream_t st) {
  T* d = s.get<T>(n);
  if (n) FMM_CUDA(cudaMemcpyAsync(d, h, sizeof(T) * n, cudaMemcpyHostToDevice, st));
  return d;
}
template <class T> void down(T* h, const T* d, size_t n, cudaStream_t st) {
  if (n) FMM_CUDA(cudaMemcpyAsync(h, d, sizeof(T) * n, cudaMemcpyDeviceToHost, st));
}

// exclusive prefix sum of n+1 counts (the last one zero) in ONE block: the
// block walks the array in 1024-element chunks carrying the running total
// (unit-level API sizes: one launch, no scratch)
__global__ void __launch_bounds__(1024) k_op_scan(const long long* in, long long* out, long long n) {
  __shared__ long long warp_tot[32];
  __shared__ long long carry;
  if (threadIdx.x == 0) carry = 0;
  __syncthreads();
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  for (long long base = 0; base <= n; base += 1024) {
    const long long i = base + threadIdx.x;
    const long long v = i <= n ? in[i] : 0;
    long long x = v;                                   // inclusive warp scan
    for (int d = 1; d < 32; d <<= 1) {
      const long long y = __shfl_up_sync(0xffffffffu, x, d);
      if (lane >= d) x += y;
    }
    if (lane == 31) warp_tot[w] = x;
    __syncthreads();
    if (w == 0) {
      long long t = warp_tot[lane];
      for (int d = 1; d < 32; d <<= 1) {
        const long long y = __shfl_up_sync(0xffffffffu, t, d);
        if (lane >= d) t += y;
      }
      warp_tot[lane] = t;
    }
    __syncthreads();
    const long long excl = carry + (w ? warp_tot[w - 1] : 0) + x - v;
    if (i <= n) out[i] = excl;
    __syncthreads();
    if (threadIdx.x == 1023) carry = excl + v;
    __syncthreads();
  }
}

void exclusive_scan(const long long* in, long long* out, long long n, cudaStream_t st) {
  k_op_scan<<<1, 1024, 0, st>>>(in, out, n);
}

template <class F> int op_call(fmm2d_ctx* c, F&& f) {
  if (!c) return FMM2D_EBADARG;
  return fmm::guarded(c, [&] {
    FMM_CUDA(cudaSetDevice(c->device));
    const int rc = f();
    FMM_CUDA(cudaStreamSynchronize(c->st));
    FMM_CUDA(cudaGetLastError());
    return rc;
  });
}

int read_flag(int* d_flag, cudaStream_t st) {
  int h = 0;
  FMM_CUDA(cudaMemcpyAsync(&h, d_flag, sizeof(int), cudaMemcpyDeviceToHost, st));
  FMM_CUDA(cudaStreamSynchronize(st));
  return h;
}

}  // namespace

extern "C" {

int fmm2d_op_p2m(fmm2d_ctx* c, int64_t nbox, const int64_t* off, const double* pos_xy,
                 const double* g, const double* center_xy, int p, double* out_xy) {
  return op_call(c, [&] {
    if (p < 1 || nbox < 0) return fmm::fail(c, FMM2D_EBADARG, "p must be >= 1");
    const long long n = off[nbox];
    Scratch s;
    auto* doff = up(s, (const long long*)off, nbox + 1, c->st);
    auto* dpos = up(s, (const double2*)pos_xy, n, c->st);
    auto* dg = up(s, g, n, c->st);
    auto* dc = up(s, (const double2*)center_xy, nbox, c->st);
    auto* dout = s.get<double2>(nbox * (p + 1));
    if (nbox) k_op_p2m<<<blocks(nbox * (p + 1)), 256, 0, c->st>>>(nbox, p, doff, dpos, dg, dc, dout);
    down((double2*)out_xy, dout, nbox * (p + 1), c->st);
    return FMM2D_OK;
  });
}

int fmm2d_op_p2l(fmm2d_ctx* c, int64_t nbox, const int64_t* off, const double* pos_xy,
                 const double* g, const double* center_xy, int p, double* out_xy) {
  return op_call(c, [&] {
    if (p < 0 || nbox < 0) return fmm::fail(c, FMM2D_EBADARG, "p must be >= 0");
    const long long n = off[nbox];
    Scratch s;
    auto* doff = up(s, (const long long*)off, nbox + 1, c->st);
    auto* dpos = up(s, (const double2*)pos_xy, n, c->st);
    auto* dg = up(s, g, n, c->st);
    auto* dc = up(s, (const double2*)center_xy, nbox, c->st);
    auto* dout = s.get<double2>(nbox * (p + 1));
    int* flag = s.get<int>(1);
    FMM_CUDA(cudaMemsetAsync(flag, 0, sizeof(int), c->st));
    if (nbox)
      k_op_p2l<<<blocks(nbox * (p + 1)), 256, 0, c->st>>>(nbox, p, doff, dpos, dg, dc, dout, flag);
    if (read_flag(flag, c->st))
      return fmm::fail(c, FMM2D_ESINGULAR, "p2l source coincides with the expansion center");
    down((double2*)out_xy, dout, nbox * (p + 1), c->st);
    return FMM2D_OK;
  });
}

// variant: 0 scaled (with the unscaled fallback outside [1e-12, 1e12]), 1 unscaled
int fmm2d_op_m2m(fmm2d_ctx* c, int64_t rows, int p, double* coeffs_xy, const double* shift_xy,
                 int variant) {
  return op_call(c, [&] {
    if (p < 1) return fmm::fail(c, FMM2D_EBADARG, "coefficient arrays need at least 2 terms (p >= 1)");
    Scratch s;
    auto* da = up(s, (const double2*)coeffs_xy, rows * (p + 1), c->st);
    auto* dr = up(s, (const double2*)shift_xy, rows, c->st);
    auto* pw = s.get<double2>(rows * (p + 1));
    int any_a0 = 0;
    for (long long r = 0; r < rows && !any_a0; ++r)
      any_a0 = coeffs_xy[2 * r * (p + 1)] != 0.0 || coeffs_xy[2 * r * (p + 1) + 1] != 0.0;
    if (rows) k_op_m2m<<<blocks(rows, 128), 128, 0, c->st>>>(rows, p, da, dr, pw, variant, any_a0);
    down((double2*)coeffs_xy, da, rows * (p + 1), c->st);
    return FMM2D_OK;
  });
}

int fmm2d_op_l2l(fmm2d_ctx* c, int64_t rows, int p, double* coeffs_xy, const double* shift_xy) {
  return op_call(c, [&] {
    if (p < 1) return fmm::fail(c, FMM2D_EBADARG, "coefficient arrays need at least 2 terms (p >= 1)");
    Scratch s;
    auto* db = up(s, (const double2*)coeffs_xy, rows * (p + 1), c->st);
    auto* dr = up(s, (const double2*)shift_xy, rows, c->st);
    auto* pw = s.get<double2>(rows * (p + 1));
    if (rows) k_op_l2l<<<blocks(rows, 128), 128, 0, c->st>>>(rows, p, db, dr, pw);
    down((double2*)coeffs_xy, db, rows * (p + 1), c->st);
    return FMM2D_OK;
  });
}

int fmm2d_op_m2l(fmm2d_ctx* c, int64_t rows, int p, const double* coeffs_xy,
                 const double* shift_xy, double* out_xy) {
  return op_call(c, [&] {
    if (p < 1) return fmm::fail(c, FMM2D_EBADARG, "coefficient arrays need at least 2 terms (p >= 1)");
    Scratch s;
    auto* da = up(s, (const double2*)coeffs_xy, rows * (p + 1), c->st);
    auto* dr = up(s, (const double2*)shift_xy, rows, c->st);
    auto* dc = s.get<double2>(rows * (p + 1));
    auto* pw = s.get<double2>(rows * (p + 1));
    int* flag = s.get<int>(1);
    FMM_CUDA(cudaMemsetAsync(flag, 0, sizeof(int), c->st));
    int any_a0 = 0;
    for (long long r = 0; r < rows && !any_a0; ++r)
      any_a0 = coeffs_xy[2 * r * (p + 1)] != 0.0 || coeffs_xy[2 * r * (p + 1) + 1] != 0.0;
    if (rows) k_op_m2l<<<blocks(rows, 128), 128, 0, c->st>>>(rows, p, da, dr, dc, pw, any_a0, flag);
    if (read_flag(flag, c->st))
      return fmm::fail(c, FMM2D_ESINGULAR, "m2l shift must be nonzero (boxes are separated)");
    down((double2*)out_xy, dc, rows * (p + 1), c->st);
    return FMM2D_OK;
  });
}

int fmm2d_op_l2p(fmm2d_ctx* c, int p, const double* coeffs_xy, const double* center_xy,
                 int64_t nt, const double* tgt_xy, double* out_xy) {
  return op_call(c, [&] {
    if (p < 0) return fmm::fail(c, FMM2D_EBADARG, "p must be >= 0");
    Scratch s;
    auto* db = up(s, (const double2*)coeffs_xy, p + 1, c->st);
    auto* dt = up(s, (const double2*)tgt_xy, nt, c->st);
    auto* dout = s.get<double2>(nt);
    if (nt)
      k_op_l2p<<<blocks(nt), 256, 0, c->st>>>(nt, p, db, cplx{center_xy[0], center_xy[1]}, dt, dout);
    down((double2*)out_xy, dout, nt, c->st);
    return FMM2D_OK;
  });
}

int fmm2d_op_m2p(fmm2d_ctx* c, int p, const double* coeffs_xy, const double* center_xy,
                 int64_t nt, const double* tgt_xy, double* out_xy) {
  return op_call(c, [&] {
    if (p < 1) return fmm::fail(c, FMM2D_EBADARG, "p must be >= 1");
    Scratch s;
    auto* da = up(s, (const double2*)coeffs_xy, p + 1, c->st);
    auto* dt = up(s, (const double2*)tgt_xy, nt, c->st);
    auto* dout = s.get<double2>(nt);
    int* flag = s.get<int>(1);
    FMM_CUDA(cudaMemsetAsync(flag, 0, sizeof(int), c->st));
    if (nt)
      k_op_m2p<<<blocks(nt), 256, 0, c->st>>>(nt, p, da, cplx{center_xy[0], center_xy[1]}, dt,
                                               dout, flag);
    if (read_flag(flag, c->st))
      return fmm::fail(c, FMM2D_ESINGULAR, "m2p target coincides with the expansion center");
    down((double2*)out_xy, dout, nt, c->st);
    return FMM2D_OK;
  });
}

int fmm2d_op_reciprocal_parts(fmm2d_ctx* c, int64_t ns, const double* src_xy, int64_t nt,
                              const double* tgt_xy, double* re, double* im, int64_t* n_skip) {
  return op_call(c, [&] {
    Scratch s;
    auto* ds = up(s, (const double2*)src_xy, ns, c->st);
    auto* dt = up(s, (const double2*)tgt_xy, nt, c->st);
    auto* dre = s.get<double>(ns * nt);
    auto* dim = s.get<double>(ns * nt);
    auto* sk = s.get<unsigned long long>(1);
    FMM_CUDA(cudaMemsetAsync(sk, 0, sizeof(unsigned long long), c->st));
    if (ns * nt) k_op_recip<<<blocks(ns * nt), 256, 0, c->st>>>(nt, ns, ds, dt, dre, dim, sk);
    down(re, dre, ns * nt, c->st);
    down(im, dim, ns * nt, c->st);
    down((unsigned long long*)n_skip, sk, 1, c->st);
    return FMM2D_OK;
  });
}

int fmm2d_op_kernel_block(fmm2d_ctx* c, int64_t ns, const double* src_xy, const double* g,
                          int64_t nt, const double* tgt_xy, double* out_xy, int64_t* n_skip) {
  return op_call(c, [&] {
    Scratch s;
    auto* ds = up(s, (const double2*)src_xy, ns, c->st);
    auto* dg = up(s, g, ns, c->st);
    auto* dt = up(s, (const double2*)tgt_xy, nt, c->st);
    auto* dout = s.get<double2>(nt);
    auto* sk = s.get<unsigned long long>(1);
    FMM_CUDA(cudaMemsetAsync(sk, 0, sizeof(unsigned long long), c->st));
    if (nt) k_op_kernel_block<<<blocks(nt, 128), 128, 0, c->st>>>(nt, ns, ds, dg, dt, dout, sk);
    down((double2*)out_xy, dout, nt, c->st);
    down((unsigned long long*)n_skip, sk, 1, c->st);
    return FMM2D_OK;
  });
}

// classify_level: geometry of level l (4^l boxes), parent strong CSR of level
// l-1 (local box ids).  Outputs: weak/strong CSR (offsets [nbox+1]); the index
// arrays need room for 16 * parent_off[4^(l-1)] entries in total.
int fmm2d_classify_level(fmm2d_ctx* c, int64_t nbox, const double* center_xy,
                         const double* half_width, const double* half_height,
                         const int64_t* parent_off, const int64_t* parent_idx, double theta,
                         int64_t* weak_off, int64_t* weak_idx, int64_t* strong_off,
                         int64_t* strong_idx) {
  return op_call(c, [&] {
    if (nbox < 4 || (nbox & 3)) return fmm::fail(c, FMM2D_EBADARG, "level must be >= 1");
    const long long npar = nbox / 4, ncand = 16 * parent_off[npar];  // 4 children x 4 candidates
    Scratch s;
    auto* dc = up(s, (const double2*)center_xy, nbox, c->st);
    auto* dhw = up(s, half_width, nbox, c->st);
    auto* dhh = up(s, half_height, nbox, c->st);
    auto* dpo = up(s, (const long long*)parent_off, npar + 1, c->st);
    auto* dpi = up(s, (const long long*)parent_idx, parent_off[npar], c->st);
    auto* cnt = s.get<long long>(2 * (nbox + 1));
    auto* off = s.get<long long>(2 * (nbox + 1));
    auto* idx = s.get<long long>(2 * ncand);
    FMM_CUDA(cudaMemsetAsync(cnt, 0, sizeof(long long) * 2 * (nbox + 1), c->st));
    long long *wc = cnt, *sc = cnt + nbox + 1, *wo = off, *so = off + nbox + 1;
    k_op_classify<<<blocks(nbox, 128), 128, 0, c->st>>>(nbox, dc, dhw, dhh, dpo, dpi, theta, 0, wc,
                                                        sc, nullptr, nullptr, nullptr, nullptr);
    exclusive_scan(wc, wo, nbox, c->st);
    exclusive_scan(sc, so, nbox, c->st);
    k_op_classify<<<blocks(nbox, 128), 128, 0, c->st>>>(nbox, dc, dhw, dhh, dpo, dpi, theta, 1,
                                                        nullptr, nullptr, wo, idx, so, idx + ncand);
    down((long long*)weak_off, wo, nbox + 1, c->st);
    down((long long*)strong_off, so, nbox + 1, c->st);
    FMM_CUDA(cudaStreamSynchronize(c->st));
    down((long long*)weak_idx, idx, weak_off[nbox], c->st);
    down((long long*)strong_idx, idx + ncand, strong_off[nbox], c->st);
    return FMM2D_OK;
  });
}

// reclassify_finest: finest geometry (4^L boxes) and strong CSR; outputs the
// p2p / p2l / m2p CSR (offsets [nbox+1]; each index array needs room for
// strong_off[nbox] entries).
int fmm2d_reclassify_finest(fmm2d_ctx* c, int64_t nbox, const double* center_xy,
                            const double* half_width, const double* half_height,
                            const int64_t* strong_off, const int64_t* strong_idx, double theta,
                            int64_t* p2p_off, int64_t* p2p_idx, int64_t* p2l_off,
                            int64_t* p2l_idx, int64_t* m2p_off, int64_t* m2p_idx) {
  return op_call(c, [&] {
    if (nbox < 1) return fmm::fail(c, FMM2D_EBADARG, "empty level");
    const long long ns = strong_off[nbox];
    Scratch s;
    auto* dc = up(s, (const double2*)center_xy, nbox, c->st);
    auto* dhw = up(s, half_width, nbox, c->st);
    auto* dhh = up(s, half_height, nbox, c->st);
    auto* dso = up(s, (const long long*)strong_off, nbox + 1, c->st);
    auto* dsi = up(s, (const long long*)strong_idx, ns, c->st);
    auto* cnt = s.get<long long>(3 * nbox + 1);
    auto* off = s.get<long long>(3 * nbox + 1);
    auto* idx = s.get<long long>(3 * ns);
    FMM_CUDA(cudaMemsetAsync(cnt, 0, sizeof(long long) * (3 * nbox + 1), c->st));
    k_op_reclassify<<<blocks(nbox, 128), 128, 0, c->st>>>(nbox, dc, dhw, dhh, dso, dsi, theta, 0,
                                                          cnt, nullptr, nullptr, nullptr, nullptr);
    // per-kind CSR offsets (the caller needs them on the host anyway)
    std::vector<long long> h(3 * nbox + 1);
    down(h.data(), cnt, 3 * nbox, c->st);
    FMM_CUDA(cudaStreamSynchronize(c->st));
    int64_t* offs[3] = {p2p_off, p2l_off, m2p_off};
    std::vector<long long> ooff(3 * nbox);
    for (int k = 0; k < 3; ++k) {
      long long acc = 0;
      for (long long b = 0; b < nbox; ++b) {
        offs[k][b] = acc;
        ooff[3 * b + k] = acc;
        acc += h[3 * b + k];
      }
      offs[k][nbox] = acc;
    }
    FMM_CUDA(cudaMemcpyAsync(off, ooff.data(), sizeof(long long) * 3 * nbox,
                             cudaMemcpyHostToDevice, c->st));
    k_op_reclassify<<<blocks(nbox, 128), 128, 0, c->st>>>(nbox, dc, dhw, dhh, dso, dsi, theta, 1,
                                                          nullptr, off, idx, idx + ns,
                                                          idx + 2 * ns);
    down((long long*)p2p_idx, idx, p2p_off[nbox], c->st);
    down((long long*)p2l_idx, idx + ns, p2l_off[nbox], c->st);
    down((long long*)m2p_idx, idx + 2 * ns, m2p_off[nbox], c->st);
    return FMM2D_OK;
  });
}

}  // extern "C"
