// C ABI and host orchestration of the B200 FMM engine (see include/fmm2d.h).
//
// One call = one CUDA stream of kernels with no host synchronisation between
// phases: tree -> connectivity -> P2M/P2L -> M2M -> M2L -> L2L -> L2P/M2P ->
// P2P(+un-permute), CUDA events between phases (the reference's phase timers,
// engine.py:217-270), then one small D2H of the status word.  List buffers
// are sized from capacities the context remembers; if a fill overflowed, the
// status says so and the call regrows and reruns (the context keeps the
// high-water mark, so steady-state calls never rerun).
#include <nvtx3/nvToolsExt.h>
#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <new>
#include <string>

#include "context.h"

#ifndef UPWARD_OVERLAP
#define UPWARD_OVERLAP 1   // P2M + M2M beside the connectivity phase
#endif

namespace fmm {

long long g_launches = 0;
unsigned long long g_dbuf_gen = 0;

CudaError::CudaError(cudaError_t e, const char* call, const char* file, int line) : err(e) {
  char buf[512];
  snprintf(buf, sizeof buf, "CUDA error %s (%s) in %s at %s:%d", cudaGetErrorName(e),
           cudaGetErrorString(e), call, file, line);
  what = buf;
}

void DBuf::reserve(size_t nbytes) {
  if (nbytes <= bytes) return;
  if (p) cudaFree(p);
  p = nullptr;
  bytes = 0;
  size_t want = std::max<size_t>(nbytes, 256);
  ++g_dbuf_gen;
  cudaError_t e = cudaMalloc(&p, want);
  if (e != cudaSuccess) {
    p = nullptr;
    cudaGetLastError();
    throw CudaError(e, "cudaMalloc", __FILE__, __LINE__);
  }
  bytes = want;
}

DBuf::~DBuf() {
  if (p) cudaFree(p);
}

}  // namespace fmm

namespace fmm {

void validate(int64_t n, int64_t m, int nd, double theta, int p, bool need_p) {
  if (n < 1) throw ApiError{FMM2D_EBADARG, "positions must be a non-empty 1-d complex array"};
  if (m < 1) throw ApiError{FMM2D_EBADARG, "eval_positions must be non-empty"};
  if (n >= (1ll << 31) - 2 || m >= (1ll << 31) - 2)
    throw ApiError{FMM2D_EBADARG, "at most 2^31-3 sources / evaluation points per call"};
  if (nd < 1) throw ApiError{FMM2D_EBADARG, "n_desired_per_box must be >= 1"};
  if (!(theta > 0.0 && theta < 1.0)) throw ApiError{FMM2D_EBADARG, "theta must lie in (0, 1)"};
  if (need_p && !p_supported(p))
    throw ApiError{FMM2D_EBADARG, "p_terms must lie in [1, 64] for the GPU engine"};
}

// leaf population statistics: sizes after S halvings are floor/ceil(n / 2^S)
void leaf_stats(int64_t n, int L, fmm2d_report* rep) {
  const int64_t nl = int64_t(1) << (2 * L);
  rep->finest_src_min = n / nl;
  rep->finest_src_max = (n + nl - 1) / nl;
  rep->finest_src_mean = (double)n / (double)nl;
}

void set_inputs(fmm2d_ctx* c, int64_t n, const double* pos, const double* g, int64_t m,
                const double* epos, bool device_io, int64_t* h2d) {
  TreeState& T = c->T;
  T.n = n;
  T.aliased = epos == nullptr;
  T.m = T.aliased ? n : m;
  T.inputs_ready = nullptr;
  if (device_io) {
    T.pos_p = reinterpret_cast<const double2*>(pos);
    T.g_p = g;
    T.epos_p = reinterpret_cast<const double2*>(epos);
    return;
  }
  // positions first on the compute stream (the tree starts with them); the
  // strengths and evaluation points travel on a copy stream, overlapping the
  // rank sorts, and run_tree waits for them just before their first use
  T.pos.reserve(sizeof(double2) * n);
  T.g.reserve(sizeof(double) * n);
  FMM_CUDA(cudaMemcpyAsync(T.pos.p, pos, sizeof(double2) * n, cudaMemcpyHostToDevice, c->st));
  // the late inputs queue behind the positions: the positions get the whole
  // host link (the tree waits on them), the rest lands during the rank sorts
  FMM_CUDA(cudaEventRecord(c->ev_pos, c->st));
  FMM_CUDA(cudaStreamWaitEvent(c->st_copy, c->ev_pos, 0));
  FMM_CUDA(cudaMemcpyAsync(T.g.p, g, sizeof(double) * n, cudaMemcpyHostToDevice, c->st_copy));
  *h2d += (sizeof(double2) + sizeof(double)) * n;
  T.pos_p = T.pos.as<double2>();
  T.g_p = T.g.as<double>();
  T.epos_p = nullptr;
  if (!T.aliased) {
    T.epos.reserve(sizeof(double2) * m);
    FMM_CUDA(cudaMemcpyAsync(T.epos.p, epos, sizeof(double2) * m, cudaMemcpyHostToDevice,
                             c->st_copy));
    *h2d += sizeof(double2) * m;
    T.epos_p = T.epos.as<double2>();
  }
  FMM_CUDA(cudaEventRecord(c->ev_inputs, c->st_copy));
  T.inputs_ready = c->ev_inputs;
}

// the degenerate box reported first by the reference: smallest level, then box
void raise_degenerate(fmm2d_ctx* c) {
  const unsigned long long key = c->h_status->degenerate_key;
  const int lev = (int)(key >> 40);
  const long long box = (long long)(key & ((1ull << 40) - 1));
  // box range from the data-independent offsets at step 2*lev
  std::vector<int> offs(2);
  const int* d_off = c->plan.d_off.as<int>() + off_base(2 * lev) + box;
  FMM_CUDA(cudaMemcpy(offs.data(), d_off, sizeof(int) * 2, cudaMemcpyDeviceToHost));
  double2 z;
  FMM_CUDA(cudaMemcpy(&z, c->T.src_pos.as<double2>() + offs[0], sizeof z,
                      cudaMemcpyDeviceToHost));
  c->deg_info[0] = offs[1] - offs[0];
  c->deg_info[1] = box;
  c->deg_info[2] = lev;
  c->deg_info[3] = c->T.L - lev;
  c->deg_xy[0] = z.x;
  c->deg_xy[1] = z.y;
  char buf[512];
  snprintf(buf, sizeof buf,
           "all %lld source points in box %lld at level %d coincide at (%.17g, %.17g) but %d "
           "more level(s) are required; reduce the level count or perturb the input",
           (long long)(offs[1] - offs[0]), box, lev, z.x, z.y, c->T.L - lev);
  throw ApiError{FMM2D_EDEGENERATE, buf};
}

void build_tree_impl(fmm2d_ctx* c, int nd) {
  TreeState& T = c->T;
  T.L = plan_levels(T.n, nd);
  plan_tree(c->plan, T.n, T.m, T.L, 0);
  run_tree(T, c->plan, c->d_status.as<DevStatus>(), c->st);
}


// --- CUDA graph of the device pipeline ---------------------------------------
// A steady-state evaluation (same configuration and device buffers as the
// previous call) replays one captured CUDA graph instead of ~70 individual
// launches: no per-kernel host launch cost and no launch gaps on the device.
// Capture happens once, right after an eager call of that configuration
// succeeded (so no buffer grows during capture).  The host actions the
// pipeline needs between kernels -- waiting for the late inputs' upload and
// starting the result download -- split the graph into segments.
// FMM2D_GRAPHS=0 disables graphs (A/B).
thread_local struct CaptureHook {
  cudaStream_t st = nullptr;
  GraphCache* g = nullptr;
} g_hook;

bool graphs_enabled() {
  static bool v = [] {
    const char* e = getenv("FMM2D_GRAPHS");
    return !(e && std::string(e) == "0");
  }();
  return v;
}

void end_segment(int action) {
  cudaGraph_t gr = nullptr;
  FMM_CUDA(cudaStreamEndCapture(g_hook.st, &gr));
  cudaGraphExec_t ex = nullptr;
  const cudaError_t e = cudaGraphInstantiate(&ex, gr, 0);
  cudaGraphDestroy(gr);
  FMM_CUDA(e);
  g_hook.g->seg.push_back(ex);
  g_hook.g->act.push_back(action);
}

// a timing event: recorded at replay time too when captured (an event
// record inside a capture is otherwise only an intra-graph dependency)
void rec_time(cudaEvent_t ev, cudaStream_t st) {
  if (g_hook.g) FMM_CUDA(cudaEventRecordWithFlags(ev, st, cudaEventRecordExternal));
  else FMM_CUDA(cudaEventRecord(ev, st));
}

bool capture_cut(int action) {
  if (!g_hook.g) return false;
  end_segment(action);
  FMM_CUDA(cudaStreamBeginCapture(g_hook.st, cudaStreamCaptureModeThreadLocal));
  return true;
}

// NVTX ranges around the host-side enqueue of each phase (header-only NVTX 3:
// no cost unless a profiler is attached); the device-side phase times are the
// CUDA events of the report
struct NvtxRange {
  explicit NvtxRange(const char* name) { nvtxRangePushA(name); }
  ~NvtxRange() { nvtxRangePop(); }
  NvtxRange(const NvtxRange&) = delete;
  NvtxRange& operator=(const NvtxRange&) = delete;
};

// everything from the status reset to the status download, on c->st
void enqueue_pipeline(fmm2d_ctx* c, int p, double theta, int nd, double2* values, double* out,
                      bool device_io) {
  TreeState& T = c->T;
  ExpState& E = c->E;
  ListState& Ls = c->Ls;
  const int L = T.L;
  DevStatus* dst = c->d_status.as<DevStatus>();
  g_launches = 0;
  reset_status(c);
  rec_time(c->ev[0], c->st);
  {
    NvtxRange r("fmm2d.sort");
    build_tree_impl(c, nd);
  }
  rec_time(c->ev[1], c->st);
  const int* offL = c->plan.d_off.as<int>() + off_base(2 * L);
  // P2M and M2M need only the tree: they run on the side stream while the
  // (latency-bound) connectivity kernels build the lists
  const bool overlap = UPWARD_OVERLAP && L > 0;
  if (overlap) {
    T.aux.ensure();
    FMM_CUDA(cudaEventRecord(c->ev_fork, c->st));
    FMM_CUDA(cudaStreamWaitEvent(T.aux.s, c->ev_fork, 0));
    rec_time(c->ev_side[0], T.aux.s);
    run_upward(T, Ls, E, offL, dst, T.aux.s, Part(), 1);
    rec_time(c->ev_side[1], T.aux.s);
    run_m2m(T, E, T.aux.s);
    rec_time(c->ev_side[2], T.aux.s);
    FMM_CUDA(cudaEventRecord(c->ev_join, T.aux.s));
  }
  // (M2L of the coarse levels beside the finest level's connectivity, on the
  // side stream, was measured: the two compete for the SMs and the step time
  // stays within +-1 % at C2-C5, so M2L runs once after the lists)
  {
    NvtxRange r("fmm2d.connect");
    run_connectivity(T, Ls, theta, dst, c->st);
  }
  rec_time(c->ev[2], c->st);
  if (L > 0)
    FMM_CUDA(cudaMemsetAsync(E.local.p, 0, sizeof(double2) * level_base(L) * (p + 1), c->st));
  run_upward(T, Ls, E, offL, dst, c->st, Part(), overlap ? 2 : 0);
  rec_time(c->ev[3], c->st);
  if (overlap) FMM_CUDA(cudaStreamWaitEvent(c->st, c->ev_join, 0));
  else run_m2m(T, E, c->st);
  rec_time(c->ev[4], c->st);
  {
    NvtxRange r("fmm2d.m2l");
    run_m2l(T, Ls, E, dst, c->st);
  }
  rec_time(c->ev[5], c->st);
  {
    NvtxRange r("fmm2d.l2l");
    run_l2l(T, E, dst, c->st);
  }
  rec_time(c->ev[6], c->st);
  {
    NvtxRange r("fmm2d.l2p_m2p");
    run_l2p_m2p(T, Ls, E, dst, c->st);
  }
  rec_time(c->ev[7], c->st);
  // P2P adds into phi and scatters to input order (engine.py:263-267)
  {
    NvtxRange r("fmm2d.p2p");
    run_p2p(T, Ls, E, offL, values, dst, c->st);
  }
  rec_time(c->ev[8], c->st);
  // the result download starts now, on the copy stream beside the report
  // kernels, instead of after the status round trip (a retry simply rewrites
  // the output; an error leaves it unspecified)
  // (a capture always cuts here for host-IO calls: the replay downloads into
  // the current call's output buffer)
  if (!device_io && (out || g_hook.g) && !capture_cut(ACT_D2H) && out) {
    FMM_CUDA(cudaStreamWaitEvent(c->st_copy, c->ev[8], 0));
    FMM_CUDA(cudaMemcpyAsync(out, values, sizeof(double2) * T.m, cudaMemcpyDeviceToHost,
                             c->st_copy));
  }
  run_stats(T, Ls, dst, c->st);
  fetch_status(c);
  FMM_CUDA(cudaMemcpyAsync(c->h_hist, Ls.hist.p, sizeof(int) * 4 * HIST_BINS,
                           cudaMemcpyDeviceToHost, c->st));
}

// the configuration a captured graph is valid for
std::vector<long long> graph_key(fmm2d_ctx* c, int p, double theta, int nd, const double2* values,
                                 bool device_io) {
  const TreeState& T = c->T;
  const ListState& Ls = c->Ls;
  long long th;
  std::memcpy(&th, &theta, sizeof th);
  return {T.n, T.m, T.aliased, T.L, p, nd, th, T.eval_full, T.exact_keys, device_io,
          (long long)T.pos_p, (long long)T.g_p, (long long)T.epos_p, (long long)values,
          Ls.cap_weak, Ls.cap_strong, Ls.cap_p2p, Ls.cap_p2l, Ls.cap_m2p,
          (long long)g_dbuf_gen};
}

void capture_graph(fmm2d_ctx* c, std::vector<long long> key, int p, double theta, int nd,
                   double2* values, bool device_io) {
  GraphCache& G = c->graph;
  G.clear();
  for (const auto& k : G.failed)
    if (k == key) return;
  const long long gen0 = g_dbuf_gen;
  g_hook.st = c->st;
  g_hook.g = &G;
  bool ok = true;
  try {
    FMM_CUDA(cudaStreamBeginCapture(c->st, cudaStreamCaptureModeThreadLocal));
    enqueue_pipeline(c, p, theta, nd, values, nullptr, device_io);
    const long long launches = g_launches;
    end_segment(ACT_NONE);
    G.launches = launches;
  } catch (const CudaError&) {
    ok = false;
    cudaGraph_t gr = nullptr;
    cudaStreamEndCapture(c->st, &gr);
    if (gr) cudaGraphDestroy(gr);
    cudaGetLastError();
  } catch (const ApiError&) {
    ok = false;
    cudaGraph_t gr = nullptr;
    cudaStreamEndCapture(c->st, &gr);
    if (gr) cudaGraphDestroy(gr);
    cudaGetLastError();
  }
  g_hook = CaptureHook{};
  if (ok && g_dbuf_gen == (unsigned long long)gen0) {
    G.key = std::move(key);
    G.valid = true;
  } else {
    G.clear();
    G.failed.push_back(key);
  }
}

void replay_graph(fmm2d_ctx* c, double2* values, double* out, bool device_io) {
  GraphCache& G = c->graph;
  for (size_t i = 0; i < G.seg.size(); ++i) {
    FMM_CUDA(cudaGraphLaunch(G.seg[i], c->st));
    if (G.act[i] == ACT_WAIT_INPUTS && c->T.inputs_ready) {
      FMM_CUDA(cudaStreamWaitEvent(c->st, c->T.inputs_ready, 0));
    } else if (G.act[i] == ACT_D2H && !device_io && out) {
      FMM_CUDA(cudaEventRecord(c->ev_d2h, c->st));
      FMM_CUDA(cudaStreamWaitEvent(c->st_copy, c->ev_d2h, 0));
      FMM_CUDA(cudaMemcpyAsync(out, values, sizeof(double2) * c->T.m, cudaMemcpyDeviceToHost,
                               c->st_copy));
    }
  }
  g_launches = G.launches;
}

int evaluate_impl(fmm2d_ctx* c, int64_t n, const double* pos, const double* g, int64_t m,
                  const double* epos, int p, double theta, int nd, double* out,
                  fmm2d_report* rep, bool device_io) {
  validate(n, epos ? m : n, nd, theta, p, true);
  const auto t_start = std::chrono::steady_clock::now();
  FMM_CUDA(cudaSetDevice(c->device));
  fmm2d_report r;
  std::memset(&r, 0, sizeof r);
  set_inputs(c, n, pos, g, m, epos, device_io, &r.h2d_bytes);
  TreeState& T = c->T;
  ExpState& E = c->E;
  ListState& Ls = c->Ls;
  const int L = plan_levels(n, nd);
  T.L = L;
  const long long nbox = level_base(L + 1);
  E.p = p;
  E.mult.reserve(sizeof(double2) * nbox * (p + 1));
  E.local.reserve(sizeof(double2) * nbox * (p + 1));
  E.phi.reserve(sizeof(double2) * T.m);
  if (!device_io) E.values.reserve(sizeof(double2) * T.m);
  double2* values = device_io ? reinterpret_cast<double2*>(out) : E.values.as<double2>();
  int attempt = 0;
  bool replayed = false;
  if (graphs_enabled()) {
    if (c->graph.valid && c->graph.key == graph_key(c, p, theta, nd, values, device_io)) {
      replay_graph(c, values, out, device_io);
      FMM_CUDA(cudaStreamSynchronize(c->st));
      if (!device_io && out) FMM_CUDA(cudaStreamSynchronize(c->st_copy));
      FMM_CUDA(cudaGetLastError());
      const int fl = c->h_status->flags;
      replayed = !(fl & (ST_RANK_RETRY | ST_EVAL_TIES | ST_OVERFLOW));
      if (!replayed) c->graph.clear();   // a retry path: rerun eagerly below
    }
  }
  for (; !replayed; ++attempt) {
    enqueue_pipeline(c, p, theta, nd, values, out, device_io);
    FMM_CUDA(cudaStreamSynchronize(c->st));
    if (!device_io && out) FMM_CUDA(cudaStreamSynchronize(c->st_copy));
    FMM_CUDA(cudaGetLastError());
    const DevStatus& s = *c->h_status;
    if (s.flags & ST_RANK_RETRY) {    // rare: clustered ties beyond the 32-bit keys
      if (T.exact_keys) throw ApiError{FMM2D_ECUDA, "rank key retry did not converge"};
      T.exact_keys = true;
      continue;
    }
    if ((s.flags & ST_EVAL_TIES) && T.aliased && !T.eval_full) {
      T.eval_full = true;             // a coordinate tie at a cut: evals need their own split
      continue;
    }
    if ((s.flags & ST_DEGENERATE)) raise_degenerate(c);
    if (s.flags & ST_OVERFLOW) {
      if (attempt >= 8) throw ApiError{FMM2D_ECUDA, "interaction-list capacity did not converge"};
      // regrow from the device-side totals
      int tw = 0, tp[3] = {0, 0, 0};
      const long long nleaf = 1ll << (2 * L);
      FMM_CUDA(cudaMemcpy(&tw, Ls.weak_off.as<int>() + nbox, sizeof(int), cudaMemcpyDeviceToHost));
      FMM_CUDA(cudaMemcpy(&tp[0], Ls.p2p_off.as<int>() + nleaf, sizeof(int), cudaMemcpyDeviceToHost));
      FMM_CUDA(cudaMemcpy(&tp[1], Ls.p2l_off.as<int>() + nleaf, sizeof(int), cudaMemcpyDeviceToHost));
      FMM_CUDA(cudaMemcpy(&tp[2], Ls.m2p_off.as<int>() + nleaf, sizeof(int), cudaMemcpyDeviceToHost));
      Ls.cap_weak = std::max<long long>(Ls.cap_weak * 2, (long long)tw + tw / 4 + 1024);
      Ls.cap_strong *= 4;
      Ls.cap_p2p = std::max<long long>(Ls.cap_p2p * 2, (long long)tp[0] + tp[0] / 4 + 1024);
      Ls.cap_p2l = std::max<long long>(Ls.cap_p2l * 2, (long long)tp[1] + tp[1] / 4 + 1024);
      Ls.cap_m2p = std::max<long long>(Ls.cap_m2p * 2, (long long)tp[2] + tp[2] / 4 + 1024);
      continue;
    }
    // a clean first attempt: capture this configuration for the next call
    if (graphs_enabled() && attempt == 0 && !(c->h_status->flags & ST_DEGENERATE)) {
      capture_graph(c, graph_key(c, p, theta, nd, values, device_io), p, theta, nd, values,
                    device_io);
    }
    break;
  }
  T.eval_full = false;                // next call starts on the aliased fast path again
  c->have_tree = c->have_lists = c->have_eval = true;
  c->theta = theta;
  const DevStatus& s = *c->h_status;
  if (s.flags & ST_P2L_SINGULAR)
    throw ApiError{FMM2D_ESINGULAR, "p2l source coincides with the expansion center"};
  if (s.flags & ST_M2L_SINGULAR)
    throw ApiError{FMM2D_ESINGULAR, "m2l shift must be nonzero (boxes are separated)"};
  if (s.flags & ST_M2P_SINGULAR)
    throw ApiError{FMM2D_ESINGULAR, "m2p target coincides with the expansion center"};
  if (!device_io && out) r.d2h_bytes = sizeof(double2) * T.m;   // downloaded above
  // report
  for (int q = 0; q < 8; ++q) r.phase_ms[q] = ev_ms(c->ev[q], c->ev[q + 1]);
  if (UPWARD_OVERLAP && L > 0) {
    // overlapped upward pass: P2M and M2M timed on their own stream (their
    // spans overlap the connectivity phase; the phases then sum to more than
    // device_ms, which stays the end-to-end device interval)
    r.phase_ms[2] = ev_ms(c->ev_side[0], c->ev_side[1]) + ev_ms(c->ev[2], c->ev[3]);
    r.phase_ms[3] = ev_ms(c->ev_side[1], c->ev_side[2]);
  }
  r.device_ms = ev_ms(c->ev[0], c->ev[8]);
  const auto t_end = std::chrono::steady_clock::now();
  r.total_ms = std::chrono::duration<double, std::milli>(t_end - t_start).count();
  r.phase_ms[8] = std::max(0.0, r.total_ms - r.device_ms);
  r.n_levels = L;
  r.retries = attempt;
  r.n_boxes = nbox;
  leaf_stats(n, L, &r);
  r.p2p_skips = (int64_t)s.p2p_skips;
  for (int q = 0; q < 4; ++q) r.list_totals[q] = s.list_total[q];
  for (int q = 0; q < 4; ++q) r.max_len[q] = s.max_len[q];
  r.kernel_launches = g_launches;
  if (rep) *rep = r;
  return FMM2D_OK;
}

}  // namespace

extern "C" {

int fmm2d_create(fmm2d_ctx** out, int device) {
  if (!out) return FMM2D_EBADARG;
  *out = nullptr;
  fmm2d_ctx* c = new (std::nothrow) fmm2d_ctx();
  if (!c) return FMM2D_EOOM;
  c->device = device;
  int rc = guarded(c, [&] {
    FMM_CUDA(cudaSetDevice(device));
    int least = 0, greatest = 0;
    FMM_CUDA(cudaDeviceGetStreamPriorityRange(&least, &greatest));
    FMM_CUDA(cudaStreamCreateWithPriority(&c->st, cudaStreamNonBlocking, greatest));
    c->own_st = c->st;
    FMM_CUDA(cudaStreamCreateWithFlags(&c->st_copy, cudaStreamNonBlocking));
    FMM_CUDA(cudaEventCreateWithFlags(&c->ev_inputs, cudaEventDisableTiming));
    FMM_CUDA(cudaEventCreateWithFlags(&c->ev_pos, cudaEventDisableTiming));
    for (auto& e : c->ev) FMM_CUDA(cudaEventCreate(&e));
    for (auto& e : c->ev_side) FMM_CUDA(cudaEventCreate(&e));
    c->d_status.reserve(sizeof(DevStatus));
    FMM_CUDA(cudaMallocHost(&c->h_status, sizeof(DevStatus)));
    FMM_CUDA(cudaMallocHost(&c->h_status_init, sizeof(DevStatus)));
    std::memset(c->h_status_init, 0, sizeof(DevStatus));
    c->h_status_init->degenerate_key = ~0ull;
    FMM_CUDA(cudaEventCreateWithFlags(&c->ev_d2h, cudaEventDisableTiming));
    FMM_CUDA(cudaEventCreateWithFlags(&c->ev_fork, cudaEventDisableTiming));
    FMM_CUDA(cudaEventCreateWithFlags(&c->ev_join, cudaEventDisableTiming));
    FMM_CUDA(cudaMallocHost(&c->h_hist, sizeof(int) * 4 * HIST_BINS));
    return FMM2D_OK;
  });
  if (rc != FMM2D_OK) {
    static thread_local std::string last;
    last = c->err;
    fmm2d_destroy(c);
    return rc;
  }
  *out = c;
  return FMM2D_OK;
}

void fmm2d_destroy(fmm2d_ctx* c) {
  if (!c) return;
  cudaSetDevice(c->device);
  if (c->st) cudaStreamSynchronize(c->st);
  for (auto& e : c->ev)
    if (e) cudaEventDestroy(e);
  for (auto& e : c->ev_side)
    if (e) cudaEventDestroy(e);
  for (auto& e : c->D.ev)
    if (e) cudaEventDestroy(e);
  c->graph.clear();
  if (c->ev_d2h) cudaEventDestroy(c->ev_d2h);
  if (c->ev_fork) cudaEventDestroy(c->ev_fork);
  if (c->ev_join) cudaEventDestroy(c->ev_join);
  if (c->h_status_init) cudaFreeHost(c->h_status_init);
  if (c->h_status) cudaFreeHost(c->h_status);
  if (c->h_hist) cudaFreeHost(c->h_hist);
  if (c->st_copy) cudaStreamSynchronize(c->st_copy);
  if (c->ev_inputs) cudaEventDestroy(c->ev_inputs);
  if (c->ev_pos) cudaEventDestroy(c->ev_pos);
  if (c->st_copy) cudaStreamDestroy(c->st_copy);
  if (c->own_st) cudaStreamDestroy(c->own_st);
  delete c;
}

const char* fmm2d_last_error(const fmm2d_ctx* c) { return c ? c->err.c_str() : "null context"; }

int fmm2d_num_levels(int64_t n, int nd) {
  if (n < 1 || nd < 1) return -1;
  return plan_levels(n, nd);
}

int fmm2d_num_levels_raw(int64_t n, int nd) {
  if (n < 1 || nd < 1) return -1;
  double raw = 0.5 * std::log2(0.625 * (double)n / (double)nd);
  return raw > 0 ? (int)std::ceil(raw) : 0;
}

int fmm2d_evaluate(fmm2d_ctx* c, int64_t n, const double* pos, const double* g, int64_t m,
                   const double* epos, int p, double theta, int nd, double* out,
                   fmm2d_report* rep) {
  if (!c) return FMM2D_EBADARG;
  return guarded(c, [&] { return evaluate_impl(c, n, pos, g, m, epos, p, theta, nd, out, rep, false); });
}

int fmm2d_evaluate_device(fmm2d_ctx* c, int64_t n, const double* pos, const double* g, int64_t m,
                          const double* epos, int p, double theta, int nd, double* out,
                          fmm2d_report* rep) {
  if (!c) return FMM2D_EBADARG;
  return guarded(c, [&] { return evaluate_impl(c, n, pos, g, m, epos, p, theta, nd, out, rep, true); });
}

int fmm2d_build_tree(fmm2d_ctx* c, int64_t n, const double* pos, const double* g, int64_t m,
                     const double* epos, int nd, int32_t* n_levels) {
  if (!c) return FMM2D_EBADARG;
  return guarded(c, [&] {
    validate(n, epos ? m : n, nd, 0.5, 1, false);
    FMM_CUDA(cudaSetDevice(c->device));
    int64_t h2d = 0;
    set_inputs(c, n, pos, g, m, epos, false, &h2d);
    for (int attempt = 0; attempt < 3; ++attempt) {
      reset_status(c);
      build_tree_impl(c, nd);
      fetch_status(c);
      FMM_CUDA(cudaStreamSynchronize(c->st));
      FMM_CUDA(cudaGetLastError());
      const int fl = c->h_status->flags;
      if (fl & ST_RANK_RETRY) {
        c->T.exact_keys = true;
      } else if ((fl & ST_EVAL_TIES) && c->T.aliased && !c->T.eval_full) {
        c->T.eval_full = true;
      } else {
        break;
      }
    }
    c->T.eval_full = false;
    c->have_tree = true;
    c->have_lists = c->have_eval = false;
    if (c->h_status->flags & ST_DEGENERATE) raise_degenerate(c);
    if (n_levels) *n_levels = c->T.L;
    return FMM2D_OK;
  });
}

int fmm2d_degenerate_info(fmm2d_ctx* c, int64_t info[4], double xy[2]) {
  if (!c) return FMM2D_EBADARG;
  for (int q = 0; q < 4; ++q) info[q] = c->deg_info[q];
  xy[0] = c->deg_xy[0];
  xy[1] = c->deg_xy[1];
  return FMM2D_OK;
}

int fmm2d_export_tree(fmm2d_ctx* c, double* center_xy, double* hw, double* hh,
                      int64_t* src_off, int64_t* eval_off, int64_t* src_perm, int64_t* eval_perm,
                      double* src_pos, double* src_g, double* eval_pos) {
  if (!c) return FMM2D_EBADARG;
  return guarded(c, [&] {
    if (!c->have_tree) throw ApiError{FMM2D_EBADARG, "no tree in this context"};
    FMM_CUDA(cudaSetDevice(c->device));
    const TreeState& T = c->T;
    const int L = T.L;
    const long long nbox = level_base(L + 1);
    std::vector<double> a(nbox), b(nbox);
    if (center_xy) {
      FMM_CUDA(cudaMemcpy(a.data(), T.box_cx.p, sizeof(double) * nbox, cudaMemcpyDeviceToHost));
      FMM_CUDA(cudaMemcpy(b.data(), T.box_cy.p, sizeof(double) * nbox, cudaMemcpyDeviceToHost));
      for (long long i = 0; i < nbox; ++i) {
        center_xy[2 * i] = a[i];
        center_xy[2 * i + 1] = b[i];
      }
    }
    if (hw) FMM_CUDA(cudaMemcpy(hw, T.box_hw.p, sizeof(double) * nbox, cudaMemcpyDeviceToHost));
    if (hh) FMM_CUDA(cudaMemcpy(hh, T.box_hh.p, sizeof(double) * nbox, cudaMemcpyDeviceToHost));
    const long long nleaf = 1ll << (2 * L);
    if (src_off || eval_off) {
      std::vector<int> so(off_base(2 * L + 1)), eo(nleaf + 1);
      FMM_CUDA(cudaMemcpy(so.data(), c->plan.d_off.p, sizeof(int) * so.size(),
                          cudaMemcpyDeviceToHost));
      FMM_CUDA(cudaMemcpy(eo.data(), T.eoff_t, sizeof(int) * (nleaf + 1),
                          cudaMemcpyDeviceToHost));
      long long w = 0;
      for (int l = 0; l <= L; ++l) {
        const long long nb = 1ll << (2 * l);
        const long long stride = 1ll << (2 * (L - l));
        for (long long k = 0; k <= nb; ++k, ++w) {
          if (src_off) src_off[w] = so[off_base(2 * l) + k];
          if (eval_off) eval_off[w] = eo[k * stride];
        }
      }
    }
    auto copy_idx = [&](int64_t* dst, const DBuf& src, long long cnt) {
      std::vector<int> t(cnt);
      FMM_CUDA(cudaMemcpy(t.data(), src.p, sizeof(int) * cnt, cudaMemcpyDeviceToHost));
      for (long long i = 0; i < cnt; ++i) dst[i] = t[i];
    };
    if (src_perm) copy_idx(src_perm, T.src_perm, T.n);
    if (eval_perm) {
      std::vector<int> t(T.m);
      FMM_CUDA(cudaMemcpy(t.data(), T.eperm_t, sizeof(int) * T.m, cudaMemcpyDeviceToHost));
      for (long long i = 0; i < T.m; ++i) eval_perm[i] = t[i];
    }
    if (src_pos)
      FMM_CUDA(cudaMemcpy(src_pos, T.src_pos.p, sizeof(double2) * T.n, cudaMemcpyDeviceToHost));
    if (src_g) FMM_CUDA(cudaMemcpy(src_g, T.src_g.p, sizeof(double) * T.n, cudaMemcpyDeviceToHost));
    if (eval_pos)
      FMM_CUDA(cudaMemcpy(eval_pos, T.epos_t, sizeof(double2) * T.m, cudaMemcpyDeviceToHost));
    return FMM2D_OK;
  });
}

int fmm2d_build_connectivity(fmm2d_ctx* c, int L, const double* center_xy, const double* hw,
                             const double* hh, double theta) {
  if (!c) return FMM2D_EBADARG;
  return guarded(c, [&] {
    if (L < 0 || L > 15) throw ApiError{FMM2D_EBADARG, "bad level count"};
    if (!(theta > 0.0 && theta < 1.0)) throw ApiError{FMM2D_EBADARG, "theta must lie in (0, 1)"};
    FMM_CUDA(cudaSetDevice(c->device));
    TreeState& T = c->T;
    T.L = L;
    const long long nbox = level_base(L + 1);
    for (DBuf* b : {&T.box_cx, &T.box_cy, &T.box_hw, &T.box_hh, &T.box_r})
      b->reserve(sizeof(double) * nbox);
    std::vector<double> a(nbox), b(nbox);
    for (long long i = 0; i < nbox; ++i) {
      a[i] = center_xy[2 * i];
      b[i] = center_xy[2 * i + 1];
    }
    FMM_CUDA(cudaMemcpy(T.box_cx.p, a.data(), sizeof(double) * nbox, cudaMemcpyHostToDevice));
    FMM_CUDA(cudaMemcpy(T.box_cy.p, b.data(), sizeof(double) * nbox, cudaMemcpyHostToDevice));
    FMM_CUDA(cudaMemcpy(T.box_hw.p, hw, sizeof(double) * nbox, cudaMemcpyHostToDevice));
    FMM_CUDA(cudaMemcpy(T.box_hh.p, hh, sizeof(double) * nbox, cudaMemcpyHostToDevice));
    compute_radius(T, c->st);
    for (int attempt = 0;; ++attempt) {
      reset_status(c);
      run_connectivity(T, c->Ls, theta, c->d_status.as<DevStatus>(), c->st);
      fetch_status(c);
      FMM_CUDA(cudaStreamSynchronize(c->st));
      FMM_CUDA(cudaGetLastError());
      if (!(c->h_status->flags & ST_OVERFLOW)) break;
      if (attempt >= 8) throw ApiError{FMM2D_ECUDA, "interaction-list capacity did not converge"};
      ListState& Ls = c->Ls;
      Ls.cap_weak *= 4; Ls.cap_strong *= 4; Ls.cap_p2p *= 4; Ls.cap_p2l *= 4; Ls.cap_m2p *= 4;
    }
    c->have_lists = true;
    c->have_tree = false;
    c->have_eval = false;
    return FMM2D_OK;
  });
}

int fmm2d_list_sizes(fmm2d_ctx* c, int64_t totals[4]) {
  if (!c) return FMM2D_EBADARG;
  return guarded(c, [&] {
    if (!c->have_lists) throw ApiError{FMM2D_EBADARG, "no interaction lists in this context"};
    const int L = c->T.L;
    const long long nbox = level_base(L + 1), nleaf = 1ll << (2 * L);
    int v[4];
    FMM_CUDA(cudaMemcpy(&v[0], c->Ls.weak_off.as<int>() + nbox, sizeof(int), cudaMemcpyDeviceToHost));
    FMM_CUDA(cudaMemcpy(&v[1], c->Ls.p2p_off.as<int>() + nleaf, sizeof(int), cudaMemcpyDeviceToHost));
    FMM_CUDA(cudaMemcpy(&v[2], c->Ls.p2l_off.as<int>() + nleaf, sizeof(int), cudaMemcpyDeviceToHost));
    FMM_CUDA(cudaMemcpy(&v[3], c->Ls.m2p_off.as<int>() + nleaf, sizeof(int), cudaMemcpyDeviceToHost));
    for (int q = 0; q < 4; ++q) totals[q] = v[q];
    return FMM2D_OK;
  });
}

int fmm2d_export_lists(fmm2d_ctx* c, int64_t* weak_off, int64_t* weak_idx, int64_t* p2p_off,
                       int64_t* p2p_idx, int64_t* p2l_off, int64_t* p2l_idx, int64_t* m2p_off,
                       int64_t* m2p_idx) {
  if (!c) return FMM2D_EBADARG;
  return guarded(c, [&] {
    if (!c->have_lists) throw ApiError{FMM2D_EBADARG, "no interaction lists in this context"};
    int64_t tot[4];
    int rc = fmm2d_list_sizes(c, tot);
    if (rc) return rc;
    const int L = c->T.L;
    const long long nbox = level_base(L + 1), nleaf = 1ll << (2 * L);
    auto cp = [&](int64_t* dst, const DBuf& src, long long cnt) {
      if (!dst || cnt == 0) return;
      std::vector<int> t(cnt);
      FMM_CUDA(cudaMemcpy(t.data(), src.p, sizeof(int) * cnt, cudaMemcpyDeviceToHost));
      for (long long i = 0; i < cnt; ++i) dst[i] = t[i];
    };
    cp(weak_off, c->Ls.weak_off, nbox + 1);
    cp(weak_idx, c->Ls.weak_idx, tot[0]);
    cp(p2p_off, c->Ls.p2p_off, nleaf + 1);
    cp(p2p_idx, c->Ls.p2p_idx, tot[1]);
    cp(p2l_off, c->Ls.p2l_off, nleaf + 1);
    cp(p2l_idx, c->Ls.p2l_idx, tot[2]);
    cp(m2p_off, c->Ls.m2p_off, nleaf + 1);
    cp(m2p_idx, c->Ls.m2p_idx, tot[3]);
    return FMM2D_OK;
  });
}

int fmm2d_histogram(fmm2d_ctx* c, int kind, int64_t* out, int nbins) {
  if (!c || kind < 0 || kind > 3 || nbins < 0) return FMM2D_EBADARG;
  return guarded(c, [&] {
    if (!c->have_eval) throw ApiError{FMM2D_EBADARG, "no evaluation in this context"};
    const int maxlen = c->h_status->max_len[kind];
    if (maxlen < HIST_BINS) {
      for (int i = 0; i < nbins; ++i) out[i] = i < HIST_BINS ? c->h_hist[kind * HIST_BINS + i] : 0;
      return FMM2D_OK;
    }
    // long lists: histogram from the offsets on the host
    const int L = c->T.L;
    const long long cnt = kind == 0 ? level_base(L + 1) : (1ll << (2 * L));
    const DBuf& src = kind == 0 ? c->Ls.weak_off : kind == 1 ? c->Ls.p2p_off
                    : kind == 2 ? c->Ls.p2l_off : c->Ls.m2p_off;
    std::vector<int> o(cnt + 1);
    FMM_CUDA(cudaMemcpy(o.data(), src.p, sizeof(int) * (cnt + 1), cudaMemcpyDeviceToHost));
    for (int i = 0; i < nbins; ++i) out[i] = 0;
    for (long long i = 0; i < cnt; ++i) {
      const int len = o[i + 1] - o[i];
      if (len < nbins) out[len]++;
    }
    return FMM2D_OK;
  });
}

int fmm2d_export_expansions(fmm2d_ctx* c, double* mult, double* local) {
  if (!c) return FMM2D_EBADARG;
  return guarded(c, [&] {
    if (!c->have_eval) throw ApiError{FMM2D_EBADARG, "no evaluation in this context"};
    const long long cnt = level_base(c->T.L + 1) * (c->E.p + 1);
    if (mult) FMM_CUDA(cudaMemcpy(mult, c->E.mult.p, sizeof(double2) * cnt, cudaMemcpyDeviceToHost));
    if (local) {
      // the chained L2L leaves the levels it passes through M2L-only: complete
      // them level by level on a copy (same arithmetic as the engine's chain)
      DBuf tmp;
      tmp.reserve(sizeof(double2) * cnt);
      FMM_CUDA(cudaMemcpyAsync(tmp.p, c->E.local.p, sizeof(double2) * cnt,
                               cudaMemcpyDeviceToDevice, c->st));
      complete_chained_locals(c->T, c->E, tmp.as<double2>(), c->st);
      FMM_CUDA(cudaMemcpyAsync(local, tmp.p, sizeof(double2) * cnt, cudaMemcpyDeviceToHost,
                               c->st));
      FMM_CUDA(cudaStreamSynchronize(c->st));
    }
    return FMM2D_OK;
  });
}

int fmm2d_export_phi(fmm2d_ctx* c, double* phi) {
  if (!c) return FMM2D_EBADARG;
  return guarded(c, [&] {
    if (!c->have_eval) throw ApiError{FMM2D_EBADARG, "no evaluation in this context"};
    FMM_CUDA(cudaMemcpy(phi, c->E.phi.p, sizeof(double2) * c->T.m, cudaMemcpyDeviceToHost));
    return FMM2D_OK;
  });
}

int fmm2d_direct(fmm2d_ctx* c, int64_t n, const double* pos, const double* g, int64_t m,
                 const double* epos, double* out) {
  if (!c) return FMM2D_EBADARG;
  return guarded(c, [&] {
    validate(n, epos ? m : n, 1, 0.5, 1, false);
    FMM_CUDA(cudaSetDevice(c->device));
    if (!epos) m = n;
    DBuf dp, dg, de, dout;
    dp.reserve(sizeof(double2) * n);
    dg.reserve(sizeof(double) * n);
    dout.reserve(sizeof(double2) * m);
    FMM_CUDA(cudaMemcpyAsync(dp.p, pos, sizeof(double2) * n, cudaMemcpyHostToDevice, c->st));
    FMM_CUDA(cudaMemcpyAsync(dg.p, g, sizeof(double) * n, cudaMemcpyHostToDevice, c->st));
    const double2* tgt = dp.as<double2>();
    if (epos) {
      de.reserve(sizeof(double2) * m);
      FMM_CUDA(cudaMemcpyAsync(de.p, epos, sizeof(double2) * m, cudaMemcpyHostToDevice, c->st));
      tgt = de.as<double2>();
    }
    run_direct(dp.as<double2>(), dg.as<double>(), n, tgt, m, dout.as<double2>(), c->st);
    FMM_CUDA(cudaMemcpyAsync(out, dout.p, sizeof(double2) * m, cudaMemcpyDeviceToHost, c->st));
    FMM_CUDA(cudaStreamSynchronize(c->st));
    FMM_CUDA(cudaGetLastError());
    return FMM2D_OK;
  });
}

int fmm2d_direct_symmetric(fmm2d_ctx* c, int64_t n, const double* pos, const double* g,
                           double* out) {
  if (!c) return FMM2D_EBADARG;
  return guarded(c, [&] {
    validate(n, n, 1, 0.5, 1, false);
    FMM_CUDA(cudaSetDevice(c->device));
    DBuf dp, dg, dw, dout;
    dp.reserve(sizeof(double2) * n);
    dg.reserve(sizeof(double) * n);
    dout.reserve(sizeof(double2) * n);
    dw.reserve(sizeof(double2) * n * direct_sym_tiles(n, nullptr));
    FMM_CUDA(cudaMemcpyAsync(dp.p, pos, sizeof(double2) * n, cudaMemcpyHostToDevice, c->st));
    FMM_CUDA(cudaMemcpyAsync(dg.p, g, sizeof(double) * n, cudaMemcpyHostToDevice, c->st));
    run_direct_symmetric(dp.as<double2>(), dg.as<double>(), n, dw.as<double2>(),
                         dout.as<double2>(), c->st);
    FMM_CUDA(cudaMemcpyAsync(out, dout.p, sizeof(double2) * n, cudaMemcpyDeviceToHost, c->st));
    FMM_CUDA(cudaStreamSynchronize(c->st));
    FMM_CUDA(cudaGetLastError());
    return FMM2D_OK;
  });
}

}  // extern "C"
