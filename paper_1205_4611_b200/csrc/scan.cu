// Device-wide exclusive scan of int32 counts: one kernel, decoupled look-back.
// Used for every CSR offset array (interaction lists) -- integer only, so the
// result is exact and independent of scheduling.
#include "engine.h"
#include "lookback.cuh"

namespace fmm {

namespace {

constexpr int SCAN_THREADS = 256;
constexpr int SCAN_ITEMS = 8;
constexpr int SCAN_TILE = SCAN_THREADS * SCAN_ITEMS;
constexpr unsigned long long FLAG_AGG = 1ull << 62;
constexpr unsigned long long FLAG_INC = 2ull << 62;
constexpr unsigned long long VAL_MASK = (1ull << 62) - 1;

__global__ void __launch_bounds__(SCAN_THREADS)
scan_tiles(const int* __restrict__ in, int* __restrict__ out, long long n,
           unsigned long long* status, unsigned int* counter, const int* base_ptr) {
  pdl_enter();
  __shared__ unsigned int s_tile;
  __shared__ long long s_warp[SCAN_THREADS / 32];
  __shared__ long long s_excl;
  if (threadIdx.x == 0) s_tile = atomicAdd(counter, 1u);
  // out[0] may alias *base_ptr; it is rewritten with the same value, so racing reads agree
  const long long obase = base_ptr ? *base_ptr : 0;
  __syncthreads();
  const long long tile = s_tile;
  const long long base = tile * SCAN_TILE + (long long)threadIdx.x * SCAN_ITEMS;
  int v[SCAN_ITEMS];
  long long tsum = 0;
#pragma unroll
  for (int q = 0; q < SCAN_ITEMS; ++q) {
    long long i = base + q;
    v[q] = i < n ? in[i] : 0;
    tsum += v[q];
  }
  // block exclusive scan of thread sums
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  long long incl = tsum;
#pragma unroll
  for (int d = 1; d < 32; d <<= 1) {
    long long o = __shfl_up_sync(0xffffffffu, incl, d);
    if (lane >= d) incl += o;
  }
  if (lane == 31) s_warp[wid] = incl;
  __syncthreads();
  if (wid == 0) {
    long long w = lane < SCAN_THREADS / 32 ? s_warp[lane] : 0;
    long long wi = w;
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
      long long o = __shfl_up_sync(0xffffffffu, wi, d);
      if (lane >= d) wi += o;
    }
    if (lane < SCAN_THREADS / 32) s_warp[lane] = wi - w;  // exclusive warp offsets
    if (lane == SCAN_THREADS / 32 - 1) {
      long long agg = wi;
      // publish + look back (single thread, predecessors are usually done)
      long long excl = 0;
      if (tile == 0) {
        atomicExch(&status[0], FLAG_INC | (unsigned long long)agg);
      } else {
        atomicExch(&status[tile], FLAG_AGG | (unsigned long long)agg);
        long long pidx = tile - 1;
        while (true) {
          unsigned long long s = atomicAdd(&status[pidx], 0ull);
          unsigned long long f = s & ~VAL_MASK;
          if (f == 0) continue;
          excl += (long long)(s & VAL_MASK);
          if (f == FLAG_INC) break;
          --pidx;
        }
        atomicExch(&status[tile], FLAG_INC | (unsigned long long)(excl + agg));
      }
      s_excl = excl;
      if ((tile + 1) * SCAN_TILE >= n) out[n] = (int)(obase + excl + agg);
    }
  }
  __syncthreads();
  long long run = s_excl + s_warp[wid] + (incl - tsum) + obase;
#pragma unroll
  for (int q = 0; q < SCAN_ITEMS; ++q) {
    long long i = base + q;
    if (i < n) out[i] = (int)run;
    run += v[q];
  }
}

__global__ void k_lb_advance(unsigned* base) {
  pdl_enter();
  if (threadIdx.x == 0 && blockIdx.x == 0) *base += LB_EPOCH_STRIDE;
}

__global__ void write_base_total(int* out, const int* base_ptr) {
  pdl_enter();
  out[0] = base_ptr ? *base_ptr : 0;
}

}  // namespace

unsigned* lb_base_prepare(DBuf& buf, bool& ready, cudaStream_t st) {
  if (!ready) {
    buf.reserve(64);
    FMM_CUDA(cudaMemsetAsync(buf.p, 0, 64, st));
    ready = true;
  }
  return buf.as<unsigned>();
}

void lb_advance(unsigned* base, cudaStream_t st) {
  note_launch();
  launch(k_lb_advance, 1, 32, 0, st, base);
}

void scan_exclusive(const int* in, int* out, int64_t n, DBuf& tmp, cudaStream_t st,
                    const int* base) {
  if (n <= 0) {
    note_launch();
    launch(write_base_total, 1, 1, 0, st, out, base);
    return;
  }
  const int64_t tiles = (n + SCAN_TILE - 1) / SCAN_TILE;
  const size_t bytes = sizeof(unsigned long long) * (tiles + 1);
  tmp.reserve(bytes);
  FMM_CUDA(cudaMemsetAsync(tmp.p, 0, bytes, st));
  auto* status = tmp.as<unsigned long long>();
  auto* counter = reinterpret_cast<unsigned int*>(status + tiles);
  note_launch();
  launch(scan_tiles, (unsigned)tiles, SCAN_THREADS, 0, st, in, out, n, status, counter, base);
}

}  // namespace fmm
