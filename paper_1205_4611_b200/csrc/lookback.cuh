// Single-pass multi-counter exclusive prefix across CTAs (decoupled
// look-back).  A tile is its CTA's linear launch index: CTAs are dispatched
// in increasing block index, so every predecessor of a tile is resident or
// done and the spin terminates (measured against an atomic ticket, which
// costs one more round trip per tile: C2 sort 0.340 -> 0.331 ms, C5 3.08 ->
// 3.00 ms; LB_TICKET=1 restores it).
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
  unsigned epoch;        // launch index within the evaluation (1 .. LB_EPOCH_STRIDE-1)
  const unsigned* base;  // device word advanced by LB_EPOCH_STRIDE per evaluation
};

// Epoch tags: a per-evaluation device-side base plus the launch's index
// within the evaluation.  Kernel arguments therefore repeat exactly from one
// evaluation to the next (a captured CUDA graph replays them unchanged) while
// the tags stay distinct across evaluations (flags are never cleared).
constexpr unsigned LB_EPOCH_STRIDE = 4096;
__device__ __forceinline__ unsigned lb_tag_epoch(unsigned local, const unsigned* base) {
  const unsigned e = (local + (base ? __ldcg(base) : 0u)) & 0x3fffffffu;
  return e ? e : 1u;
}
// one thread: advance the evaluation's epoch base (first kernel of a phase)
__device__ __forceinline__ void lb_advance_base(unsigned* base) {
  if (base) *base += LB_EPOCH_STRIDE;
}

// draw this CTA's tile (thread 0 only); the last ticket resets the counter
#ifndef LB_TICKET
#define LB_TICKET 0   // 1: tiles drawn through an atomic ticket (A/B)
#endif
__device__ __forceinline__ unsigned lb_ticket(const LookbackState& S, unsigned ntiles) {
#if !LB_TICKET
  // tile = launch index: CTAs are dispatched in increasing linear block
  // index (the assumption CUB's single-pass scans make), so predecessors are
  // resident or done; saves the ticket's atomic round trip
  (void)S; (void)ntiles;
  return blockIdx.x;
#endif
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
  const unsigned tag = lb_tag_epoch(S.epoch, S.base) << 2;
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

namespace fmm {

// Single-counter variant with the flag and the value packed in one 64-bit
// word (2-bit state | 30-bit epoch tag | 32-bit value): one load per window
// lane and no fence between value and flag, halving the latency of every
// look-back step.  Values (and prefixes) must fit in 32 bits.
struct LookbackPacked {
  unsigned long long* word;   // [ntiles]
  unsigned* ticket;
  unsigned epoch;             // launch index within the evaluation (see LookbackState)
  const unsigned* base;
};

__device__ __forceinline__ unsigned lb_ticket(const LookbackPacked& S, unsigned ntiles) {
#if !LB_TICKET
  (void)S; (void)ntiles;
  return blockIdx.x;
#endif
  const unsigned t = atomicAdd(S.ticket, 1u);
  if (t == ntiles - 1) atomicExch(S.ticket, 0u);
  return t;
}

__device__ __forceinline__ unsigned long long lb_pack(unsigned epoch, unsigned state,
                                                      unsigned value) {
  return ((unsigned long long)((epoch << 2) | state) << 32) | value;
}

// called by one full warp; returns the exclusive prefix of `agg` over the
// tiles of the current chain (a chain starts at tile 0 or a `head` tile)
__device__ __forceinline__ unsigned lb_prefix_packed(const LookbackPacked& S, unsigned tile,
                                                     unsigned agg, bool head) {
  const int lane = threadIdx.x & 31;
  const unsigned ep = lb_tag_epoch(S.epoch, S.base);
  if (tile == 0 || head) {
    if (lane == 0) atomicExch(S.word + tile, lb_pack(ep, 2u, agg));
    __syncwarp();
    return 0;
  }
  if (lane == 0) atomicExch(S.word + tile, lb_pack(ep, 1u, agg));
  unsigned excl = 0;
  long long top = (long long)tile - 1;
  while (true) {
    const long long p = top - lane;
    unsigned long long v = lb_pack(ep, 2u, 0u);   // lanes past tile 0: terminator
    if (p >= 0) {
      do {
        v = *(volatile unsigned long long*)(S.word + p);
      } while ((unsigned)(v >> 34) != ep || ((v >> 32) & 3u) == 0);
    }
    const unsigned st = (unsigned)(v >> 32) & 3u;
    const unsigned inc = __ballot_sync(0xffffffffu, st == 2u);
    const int stop = inc ? __ffs(inc) - 1 : 31;
    unsigned x = lane <= stop ? (unsigned)v : 0u;
#pragma unroll
    for (int d = 16; d; d >>= 1) x += __shfl_xor_sync(0xffffffffu, x, d);
    excl += x;
    if (inc) break;
    top -= 32;
  }
  if (lane == 0) atomicExch(S.word + tile, lb_pack(ep, 2u, excl + agg));
  __syncwarp();
  return excl;
}

}  // namespace fmm
