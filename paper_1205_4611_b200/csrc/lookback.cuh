// Single-pass multi-counter exclusive prefix across CTAs (decoupled
// look-back).  Tiles are taken in launch order through an atomic ticket, so
// every predecessor of a tile is already resident and the spin terminates.
//
// State per tile: an epoch-tagged flag word (0 none, 1 aggregate ready,
// 2 inclusive prefix ready) and NW 64-bit aggregates / inclusive prefixes.
// The epoch changes on every launch, so the flag array never needs clearing;
// the ticket counter is reset by the tile that draws the last ticket.
#pragma once
#include "common.cuh"

namespace fmm {

struct LookbackState {
  unsigned* flag;        // [ntiles]
  long long* aggv;       // [ntiles * NW]
  long long* incv;       // [ntiles * NW]
  unsigned* ticket;      // one counter, 0 between launches
  unsigned epoch;        // nonzero, distinct per launch
};

// draw this CTA's tile (thread 0 only); the last ticket resets the counter
__device__ __forceinline__ unsigned lb_ticket(const LookbackState& S, unsigned ntiles) {
  const unsigned t = atomicAdd(S.ticket, 1u);
  if (t == ntiles - 1) atomicExch(S.ticket, 0u);
  return t;
}

// publish agg[] for `tile` and return the exclusive prefix in excl[]; called
// by one full warp (all 32 lanes, same arguments).  The warp inspects a
// window of 32 predecessors per step (CUB-style), so a wave of tiles that
// publish together resolves in a few L2 round trips instead of one per tile.
// `head` starts a new chain (segmented scans: the first tile of a segment)
template <int NW>
__device__ __forceinline__ void lb_prefix(const LookbackState& S, unsigned tile,
                                          const long long (&agg)[NW], long long (&excl)[NW],
                                          bool head = false) {
  const unsigned tag = S.epoch << 2;
  const int lane = threadIdx.x & 31;
#pragma unroll
  for (int w = 0; w < NW; ++w) excl[w] = 0;
  if (tile == 0 || head) {
    if (lane == 0) {
#pragma unroll
      for (int w = 0; w < NW; ++w) S.incv[(long long)tile * NW + w] = agg[w];
      __threadfence();
      atomicExch(S.flag + tile, tag | 2u);
    }
    __syncwarp();
    return;
  }
  if (lane == 0) {
#pragma unroll
    for (int w = 0; w < NW; ++w) S.aggv[(long long)tile * NW + w] = agg[w];
    __threadfence();
    atomicExch(S.flag + tile, tag | 1u);
  }
  long long top = (long long)tile - 1;          // newest predecessor of the window
  while (true) {
    const long long p = top - lane;
    unsigned f = tag | 2u;                      // lanes past tile 0 act as a terminator
    if (p >= 0) {
      do {
        f = *(volatile unsigned*)(S.flag + p);
      } while ((f & ~3u) != tag || (f & 3u) == 0);
    }
    __syncwarp();
    __threadfence();
    const unsigned inc = __ballot_sync(0xffffffffu, (f & 3u) == 2u);
    const int stop = inc ? __ffs(inc) - 1 : 31;   // nearest inclusive prefix in the window
    long long v[NW];
#pragma unroll
    for (int w = 0; w < NW; ++w) {
      v[w] = 0;
      if (p >= 0 && lane <= stop)
        v[w] = (f & 3u) == 2u ? __ldcg(S.incv + p * NW + w) : __ldcg(S.aggv + p * NW + w);
#pragma unroll
      for (int d = 16; d; d >>= 1) v[w] += __shfl_xor_sync(0xffffffffu, v[w], d);
      excl[w] += v[w];
    }
    if (inc) break;
    top -= 32;
  }
  if (lane == 0) {
#pragma unroll
    for (int w = 0; w < NW; ++w) S.incv[(long long)tile * NW + w] = excl[w] + agg[w];
    __threadfence();
    atomicExch(S.flag + tile, tag | 2u);
  }
  __syncwarp();
}

}  // namespace fmm
