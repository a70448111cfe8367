// Host-side declarations shared by the engine translation units.
#pragma once
#include <cstddef>
#include <cstdint>
#include <string>
#include <utility>
#include <vector>
#include <cuda_runtime.h>

#include "common.cuh"

namespace fmm {

#define FMM_CUDA(call)                                                              \
  do {                                                                              \
    cudaError_t e_ = (call);                                                        \
    if (e_ != cudaSuccess) throw CudaError(e_, #call, __FILE__, __LINE__);          \
  } while (0)

struct CudaError {
  cudaError_t err;
  std::string what;
  CudaError(cudaError_t e, const char* call, const char* file, int line);
};

// grow-only device buffer (owning; not copyable)
struct DBuf {
  void* p = nullptr;
  size_t bytes = 0;
  DBuf() = default;
  DBuf(const DBuf&) = delete;
  DBuf& operator=(const DBuf&) = delete;
  void reserve(size_t nbytes);
  void swap(DBuf& o) {
    std::swap(p, o.p);
    std::swap(bytes, o.bytes);
  }
  template <class T> T* as() const { return static_cast<T*>(p); }
  ~DBuf();
};

// per (N, M, L, s0) plan: data-independent segment offsets and partition tiles
// (S = 2L - s0 split steps below the (sub)tree root)
struct TreePlan {
  int64_t n = -1, m = -1;
  int L = -1, s0 = -1, S = 0, sb = 0;
  int smem_bytes = 0;
  bool global_leaf_finalize = false;
  std::vector<int> tile_base;        // per global step s < sb: first tile index
  std::vector<int> tile_count;       // per global step
  DBuf d_off;                        // int32 offsets for steps 0..S (+1 per step)
  DBuf d_tile_seg, d_tile_start;     // concatenated tile tables of all global steps
  DBuf d_tile_desc;                  // per tile: {segment, tile start, segment start, end}
  std::vector<int> segt_base;        // per step: base of its first-tile-per-segment table
  DBuf d_seg_tile0;                  // per step and segment: first tile (+ sentinel)
  DBuf d_tile_flag;                  // per tile: parities + axis, written by the step before
};

__host__ __device__ inline int64_t step_base(int s) { return (int64_t(1) << s) - 1; }          // per-segment tables
__host__ __device__ inline int64_t off_base(int s) { return (int64_t(1) << s) - 1 + s; }        // offset tables (+1 each)
__host__ __device__ inline int64_t level_base(int l) { return ((int64_t(1) << (2 * l)) - 1) / 3; }  // boxes above level l

// Ownership in a distributed evaluation: rank `rank` of
// G = 2^s0 owns, at every level l with t = 2l - s0 >= 0, the contiguous boxes
// [rank << t, (rank + 1) << t) -- the subtree below top-split segment
// `rank`.  Levels above (2l < s0) are shared: every rank computes them
// redundantly.  G = 1 owns everything.
struct Part {
  int G = 1, rank = 0, s0 = 0;
  long long lo(int l) const {
    const int t = 2 * l - s0;
    return t < 0 ? 0 : (long long)rank << t;
  }
  long long hi(int l) const {
    const int t = 2 * l - s0;
    return t < 0 ? 1ll << (2 * l) : (long long)(rank + 1) << t;
  }
  bool shared(int l) const { return 2 * l < s0; }
  int ltop() const { return (s0 + 1) / 2; }          // first level with owned boxes
};

// Which part of the global pyramid a tree build covers.  Single GPU: the
// whole tree (s0 = 0).  Distributed: the subtree below segment `seg` of the
// top split (s0 = log2 G steps, done collectively), written into global-size
// output arrays at tree-order offset `out0`, with the original index of every
// local input point in `orig`.
struct TreeSpec {
  int s0 = 0;
  long long seg = 0;
  long long out0 = 0;
  const int* orig = nullptr;
  const int* eorig = nullptr;        // original index of every separate evaluation point
  bool root_given = false;
  double root[4] = {0, 0, 0, 0};     // x0, x1, y0, y1
};

// device state of one tree (kept between phases of an evaluation)
struct TreeState {
  TreeSpec spec;
  int64_t n = 0, m = 0;
  int L = 0;
  bool aliased = true;
  bool exact_keys = false;           // 64-bit rank keys (set after a tie-run overflow)
  bool dup_checked = false;          // this build's x tie pass raised ST_DUPLICATES if needed
  DBuf pos, g, epos;                 // owned input copies, original order
  const double2* pos_p = nullptr;    // inputs actually used (owned copies or caller's
  const double* g_p = nullptr;       //   device memory), original order
  const double2* epos_p = nullptr;
  cudaEvent_t inputs_ready = nullptr;  // strengths / evaluation points uploaded (host calls)
  DBuf keys_in, keys_out, vals_in, vals_out, cub_tmp, cub_tmp2;
  // second stream for the y-axis rank sort (runs beside the x-axis sort)
  struct Aux {
    cudaStream_t s = nullptr;
    cudaEvent_t fork = nullptr, join = nullptr;
    void ensure() {
      if (s) return;
      // lowest priority: side work (upward pass, coarse M2L) fills the SMs the
      // latency-bound main-stream kernels leave idle instead of delaying them
      int least = 0, greatest = 0;
      cudaDeviceGetStreamPriorityRange(&least, &greatest);
      cudaStreamCreateWithPriority(&s, cudaStreamNonBlocking, least);
      cudaEventCreateWithFlags(&fork, cudaEventDisableTiming);
      cudaEventCreateWithFlags(&join, cudaEventDisableTiming);
    }
    Aux() = default;
    Aux(const Aux&) = delete;
    Aux& operator=(const Aux&) = delete;
    ~Aux() {
      if (s) cudaStreamDestroy(s);
      if (fork) cudaEventDestroy(fork);
      if (join) cudaEventDestroy(join);
    }
  } aux;
  DBuf perm_x, perm_y, rank_x, rank_y;
  DBuf X0, X1, Y0, Y1;               // int2 (rank_x, rank_y) arrays
  DBuf xpar0, xpar1, ypar0, ypar1, cutrank;
  DBuf tile_cnt, tile_pre;
  DBuf lb_flags, lb_vals, lb_ticket;  // look-back state of the fused partition steps
  long long lb_tiles = 0;
  unsigned lb_epoch = 0;             // launch index within the evaluation
  DBuf lb_base;                      // device epoch base (lookback.cuh)
  bool lb_base_ready = false;
  DBuf rect_tab, cut_tab, axis_tab;
  DBuf leaf_of;                      // eval/source leaf ids (fallback + evals)
  // outputs (tree order)
  DBuf src_pos, src_g, src_perm;     // double2, double, int32
  DBuf eval_pos, eval_perm;          // double2, int32
  DBuf eval_leaf_off;                // int32[4^L + 1]
  bool eval_full = false;            // aliased evals take the full descend path (cut ties)
  // tree-ordered evaluation points as the consumers see them: the owned
  // buffers above, or -- aliased evaluation points with no coordinate tie at
  // any cut -- the source arrays themselves (identical partition)
  const double2* epos_t = nullptr;
  const int* eperm_t = nullptr;
  const int* eoff_t = nullptr;
  const unsigned* eleaf_t = nullptr; // leaf of every tree-ordered eval point (separate evals;
                                     // aliased ones derive it from the source offsets)
  DBuf box_cx, box_cy, box_hw, box_hh, box_r;  // all levels, global box id
  DBuf bbox;                         // double[4] + scratch
};

struct ListState {
  long long cap_weak = 0, cap_strong = 0, cap_p2p = 0, cap_p2l = 0, cap_m2p = 0;
  DBuf weak_off;                     // int32[nboxes_total + 1] global CSR
  DBuf weak_idx, weak_tgt;           // int32 (source global id, target global id)
  DBuf s_off[2], s_idx[2];           // strong lists ping-pong (level-local ids)
  DBuf lb_flags, lb_vals, lb_ticket;  // single-pass look-back state of the list kernels
  DBuf cl_cnt, cl_mask;              // split classify: per-target counts, far masks
  DBuf lvl_max;                      // int[L+2]: longest strong list per level (cl_heavy)
  long long cl_cnt_zeroed = 0;       // bytes of cl_cnt known to be zero
  long long lb_tiles = 0;
  unsigned lb_epoch = 0;             // launch index within the evaluation
  DBuf lb_base;                      // device epoch base (lookback.cuh)
  bool lb_base_ready = false;
  DBuf p2p_off, p2p_idx, p2l_off, p2l_idx, m2p_off, m2p_idx;  // finest, level-local ids
  DBuf totals;                       // int64 scratch for scans
  DBuf hist;                         // int32 histograms [4][HIST_BINS]
};

constexpr int HIST_BINS = 4096;

struct ExpState {
  int p = 0;
  DBuf mult, local;                  // double2[nboxes_total * (p+1)]
  DBuf phi;                          // double2[M] tree order
  DBuf values;                       // double2[M] input order
  DBuf partials, item_flags;         // M2L cross-warp partial sums
  DBuf long_list;                    // leaves with long m2p lists (+ count)
  DBuf p2l_rows;                     // one P2L row per p2l pair
  int l2l_chain_lt = 0;              // last L2L: levels 2..lt-1 left M2L-only (chained kernel)
};

// count of engine kernel launches (gpu_launches evidence in the report)
extern long long g_launches;
extern unsigned long long g_dbuf_gen;   // bumped on every device (re)allocation
// CUDA-graph capture of the evaluation (fmm2d.cu): a phase that needs a host
// action between two kernels calls capture_cut(); while capturing it closes
// the current graph segment (the replay performs the action between segment
// launches) and returns true; otherwise it returns false and the caller
// performs the action itself.
enum : int { ACT_NONE = 0, ACT_WAIT_INPUTS = 1, ACT_D2H = 2 };
bool capture_cut(int action);
// device epoch base of a look-back state: allocated + zeroed once, then
// advanced by one kernel per evaluation (graph-replay safe epoch tags)
unsigned* lb_base_prepare(DBuf& buf, bool& ready, cudaStream_t st);
void lb_advance(unsigned* base, cudaStream_t st);
inline void note_launch() { ++g_launches; }

// launch an engine kernel with programmatic dependent launch (see pdl_enter)
template <typename... KArgs, typename... Args>
inline void launch(void (*kern)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t st,
                   Args&&... args) {
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = 1;
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  FMM_CUDA(cudaLaunchKernelEx(&cfg, kern, static_cast<KArgs>(args)...));
}

// ---------------------------------------------------------------------------
// launchers (all enqueue on `st`, no host sync)
int plan_levels(int64_t n, int nd);
void plan_tree(TreePlan& plan, int64_t n, int64_t m, int L, int s0 = 0);
void run_tree(TreeState& T, TreePlan& plan, DevStatus* dstat, cudaStream_t st);

void run_connectivity(const TreeState& T, ListState& Ls, double theta, DevStatus* dstat,
                      cudaStream_t st, const Part& part = Part());

void compute_radius(TreeState& T, cudaStream_t st);
// which: 0 = P2M and P2L, 1 = P2M only (needs the tree only), 2 = P2L only (needs lists)
void run_upward(const TreeState& T, const ListState& Ls, ExpState& E, const int* offL,
                DevStatus* dstat, cudaStream_t st, const Part& part = Part(), int which = 0);
// M2M for parent levels lmax..lmin (descending); lmax < 0 means L-1
void run_m2m(const TreeState& T, ExpState& E, cudaStream_t st, const Part& part = Part(),
             int lmin = 1, int lmax = -1);
void run_m2l(const TreeState& T, const ListState& Ls, ExpState& E, DevStatus* dstat,
             cudaStream_t st);
void run_l2l(const TreeState& T, ExpState& E, DevStatus* dstat, cudaStream_t st,
             const Part& part = Part());
// debug seam: `out` (a copy of E.local) gets the complete local expansions of
// the levels the chained L2L kernel only passes through
void complete_chained_locals(const TreeState& T, ExpState& E, double2* out, cudaStream_t st);
// L2P + M2P for tree-ordered evaluation points [e0, e1) (e1 < 0: all)
void run_l2p_m2p(const TreeState& T, const ListState& Ls, ExpState& E, DevStatus* dstat,
                 cudaStream_t st, long long e0 = 0, long long e1 = -1,
                 long long leaf_range_lo = 0, long long leaf_range_hi = 0);
// values in input order, or (out_base >= 0) tree order starting at point out_base
void run_p2p(const TreeState& T, const ListState& Ls, ExpState& E, const int* offL,
             double2* values, DevStatus* dstat, cudaStream_t st, const Part& part = Part(),
             long long out_base = -1);
void run_stats(const TreeState& T, ListState& Ls, DevStatus* dstat, cudaStream_t st,
               const Part& part = Part());

void run_direct(const double2* src, const double* g, int64_t n, const double2* tgt, int64_t m,
                double2* out, cudaStream_t st);
// symmetric all-pairs direct sum (aliased points): W = double2[direct_sym_tiles(n) * n] scratch
long long direct_sym_tiles(int64_t n, int64_t* st_out);
void run_direct_symmetric(const double2* src, const double* g, int64_t n, double2* W,
                          double2* out, cudaStream_t st);

// device-wide exclusive scan of int32 counts: out[i] = *base + sum(in[0..i)),
// out[n] = *base + total (base = 0 when null).  `tmp` is grown as needed.
void scan_exclusive(const int* in, int* out, int64_t n, DBuf& tmp, cudaStream_t st,
                    const int* base = nullptr);

bool p_supported(int p);

}  // namespace fmm
