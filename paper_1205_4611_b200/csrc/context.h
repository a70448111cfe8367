// The library context (C ABI handle) and the host helpers shared by the
// single-GPU entry points (fmm2d.cu) and the distributed ones (dist.cu).
#pragma once
#include <cstring>
#include <new>
#include <string>
#include <vector>

#include "engine.h"
#include "../../include/fmm2d.h"

namespace fmm {

struct ApiError {
  int code;
  std::string msg;
};

// state of one rank of a distributed evaluation; see dist.cu
struct DistState {
  bool active = false;
  Part part;
  long long n_total = 0;
  int L = 0, p = 0, nd = 35;
  double theta = 0.5;
  std::vector<std::vector<long long>> off;     // data-independent offsets, steps 0..2L
  std::vector<std::vector<double>> rect;       // top split: 4 doubles per segment, steps 0..s0
  DBuf leaf_off;                               // int32 [4^L + 1] global leaf offsets
  long long off_key_n = -1;                   // (n_total, L) of off / leaf_off
  int off_key_L = -1;
  DBuf totals5;                                // list totals for the report
  DBuf rec_a, rec_b;                           // top-split records {x, y, g, idx}
  long long n_local = 0;                       // records held before the exchange
  std::vector<long long> seg_off;              // local record offsets per top segment
  DBuf d_seg_off, d_axis, sel, eqf, eqpre, skey, skey2, sval, sval2, cub_tmp, bbox;
  long long n_r = 0, g0 = 0;                   // owned subtree: size, tree-order start
  DBuf loc_pos, loc_g, loc_idx;
  DBuf flags, ids, keys, ids_sorted, keys_sorted, nsel;
  std::vector<long long> req_count[2];         // per owner: multipole boxes, particle leaves
  DBuf req_ids[2];                             // requests grouped by owner
  long long nmax_leaf = 0;                     // records per leaf in halo messages
  DBuf vals;                                   // owned values, tree order
  // separate evaluation points: sharded like the sources, routed to the rank
  // owning their top-split segment (coord <= cut), evaluated there
  bool separate = false;
  long long m_total = 0, m_local = 0, m_r = 0;
  DBuf erec_a, erec_b, loc_epos, loc_eidx, eoff_g, eleaf_g, ecount;
  std::vector<std::vector<double>> cuts;        // top split: cut per segment, steps 0..s0-1
  std::vector<std::vector<unsigned char>> axes; // ... and its axis
  cudaEvent_t ev[12] = {};
  long long launches0 = 0;
};

}  // namespace fmm

using namespace fmm;

// one instantiated CUDA graph of the evaluation pipeline (fmm2d.cu), valid for
// the exact configuration and device buffers it was captured with
struct GraphCache {
  bool valid = false;
  std::vector<long long> key;
  std::vector<cudaGraphExec_t> seg;  // segments, launched in order on ctx->st
  std::vector<int> act;              // host action after each segment (ACT_*)
  long long launches = 0;            // kernels inside (captured count)
  std::vector<std::vector<long long>> failed;   // keys whose capture failed: stay eager
  void clear() {
    for (auto e : seg) cudaGraphExecDestroy(e);
    seg.clear();
    act.clear();
    valid = false;
  }
};

struct fmm2d_ctx {
  int device = 0;
  cudaStream_t st = nullptr;
  cudaStream_t own_st = nullptr;     // the stream this context created (st may be external)
  cudaStream_t st_copy = nullptr;    // H2D of the inputs needed late (strengths, evaluation points)
  cudaEvent_t ev_inputs = nullptr;
  cudaEvent_t ev_pos = nullptr;      // positions uploaded (the late inputs queue behind)
  TreePlan plan;
  TreeState T;
  ListState Ls;
  ExpState E;
  DBuf d_status;
  DevStatus* h_status = nullptr;
  DevStatus* h_status_init = nullptr;  // constant reset image (graph-replay safe)
  GraphCache graph;
  cudaEvent_t ev_d2h = nullptr;
  cudaEvent_t ev_fork = nullptr, ev_join = nullptr;   // upward-pass side stream dependencies
  int* h_hist = nullptr;
  cudaEvent_t ev[10] = {};
  cudaEvent_t ev_side[5] = {};      // P2M / M2M on the side stream (overlapped)
  std::string err;
  bool have_tree = false, have_lists = false, have_eval = false;
  double theta = 0.5;
  long long deg_info[4] = {0, 0, 0, 0};
  double deg_xy[2] = {0, 0};
  DistState D;
};

namespace fmm {

inline int fail(fmm2d_ctx* c, int code, const std::string& msg) {
  if (c) c->err = msg;
  return code;
}

template <class F>
int guarded(fmm2d_ctx* c, F&& f) {
  try {
    c->err.clear();
    return f();
  } catch (const ApiError& e) {
    return fail(c, e.code, e.msg);
  } catch (const CudaError& e) {
    if (e.err == cudaErrorMemoryAllocation) return fail(c, FMM2D_EOOM, e.what);
    return fail(c, FMM2D_ECUDA, e.what);
  } catch (const std::bad_alloc&) {
    return fail(c, FMM2D_EOOM, "host allocation failed");
  }
}

inline void reset_status(fmm2d_ctx* c) {
  FMM_CUDA(cudaMemcpyAsync(c->d_status.p, c->h_status_init, sizeof(DevStatus),
                           cudaMemcpyHostToDevice, c->st));
}

inline void fetch_status(fmm2d_ctx* c) {
  FMM_CUDA(cudaMemcpyAsync(c->h_status, c->d_status.p, sizeof(DevStatus),
                           cudaMemcpyDeviceToHost, c->st));
}

inline float ev_ms(cudaEvent_t a, cudaEvent_t b) {
  float ms = 0.f;
  FMM_CUDA(cudaEventElapsedTime(&ms, a, b));
  return ms;
}

void validate(int64_t n, int64_t m, int nd, double theta, int p, bool need_p);
void leaf_stats(int64_t n, int L, fmm2d_report* rep);

}  // namespace fmm
