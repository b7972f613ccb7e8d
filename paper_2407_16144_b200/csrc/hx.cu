// hx: the B200 (sm_100a) CUDA layer of the rHPDHG solver.  See include/hx.h
// and DESIGN.md.
//
// Every rHPDHG iteration runs inside ONE persistent cooperative kernel
// (loop_kernel): two fused SpMV phases separated by software grid barriers.
// The reference's scalar control logic (src/solver.cpp:241-341) is
// REPLICATED in every CTA: after the end-of-iteration barrier each CTA
// reduces the same per-CTA partials in the same fixed order, so all CTAs hold
// bit-identical totals and take identical decisions with no broadcast step.
// No host round trip per iteration.
//
//   phase A (rows of the explicit A^T = columns j of A):
//     x_j   = T_prev.x_j, or (1-w) T_prev.x_j + w anchor_x_j      [solver.cpp:333-336]
//     aty_j = (A^T y)_j                                           [pdhg_core.cpp:80]
//     x+_j  = max(0, x_j - eta (aty_j + c_j))                     [pdhg_core.cpp:81-82]
//     partials ||[-(c + A^T y)]+||^2, c.x, ||x - x+||^2           [pdhg_core.cpp:60-63, 39]
//   phase B (rows i of A):
//     ax+_i = (A x+)_i                                            [pdhg_core.cpp:83]
//     y+_i  = y_i + eta ((2 ax+_i - ax_i) - b_i)                  [pdhg_core.cpp:84]
//     (1-w) y+ + w anchor_y and (1-w) ax+ + w ax_anchor, written
//     speculatively so a non-restart needs no extra pass        [solver.cpp:335-337]
//     partials ||Ax - b||^2, b.y, ||y - y+||^2, (y - y+).(Ax - Ax+)
//   controller (every CTA): KKT [pdhg_core.cpp:57-68], canonical residual
//     [:37-51], epochs, best iterate, termination [solver.cpp:292-295],
//     certificate-scan scheduling [:297-317], restart [:162-174, :319-332],
//     buffer roles for the next iteration.
//
// SpMV engine: nnz-chunked warp tasks with kLoadsPerLane independent index /
// value loads per lane in flight, products staged in shared memory, then
// lane-per-row sums in a fixed order: two interleaved partial sums over the
// row's ascending column order (even / odd positions) added at the end.  Rows
// of <= 2 nonzeros (bound rows, slack columns) get exactly the reference's
// order; longer rows differ from it only by rounding (~1e-16 relative), and
// halving the dependent-add chain is worth 3.9% on configs[1] (HX_RSUM).
//
// All reductions are fixed-order (static row->warp schedule, fixed trees, no
// floating-point atomics): results are bit-reproducible run to run.  Device
// arithmetic is compiled with -fmad=false so every scalar op rounds once,
// like the reference's SSE2 build.
#include <cub/device/device_radix_sort.cuh>
#include <cub/device/device_scan.cuh>

#include <algorithm>
#include <atomic>
#include <chrono>
#include <thread>
#include <cstdio>
#include <cstdlib>
#include <cmath>
#include <cstring>
#include <future>
#include <limits>
#include <memory>
#include <mutex>
#include <unordered_set>
#include <string>
#include <type_traits>

#include "hx_internal.cuh"

// HX_CHECKED builds (tools/variant.sh checked -DHX_CHECKED): device-side
// bounds checks on the SpMV engine's indices; a violation prints and traps.
// compute-sanitizer is unavailable on the GPU pool, so this is the
// out-of-bounds check the GPU test suite runs against.
#ifdef HX_CHECKED
#define HX_CHECK(cond, what, a, b)                                                                      \
  do {                                                                                                  \
    if (!(cond)) {                                                                                      \
      printf("HX_CHECK failed: %s (%lld, %lld) at %s:%d\n", what, (long long)(a), (long long)(b), __FILE__, \
             __LINE__);                                                                                 \
      __trap();                                                                                         \
    }                                                                                                   \
  } while (0)
#else
#define HX_CHECK(cond, what, a, b) \
  do {                             \
  } while (0)
#endif

namespace hx {

// kModePower: power iteration (src/sparse_matrix.cpp:138-179).  Teams only:
// kModeKkt (KKT of the current iterate with fresh products) and kModeScale
// (the diagonal preconditioning rounds), every rank on its own blocks with
// the cross-rank exchange through pushes and team barriers.
enum Mode : int { kModeLoop = 0, kModePower = 1, kModeKkt = 2, kModeScale = 3 };

// Buffer roles and per-iteration scalars every thread needs.
struct Roles {
  int x_src, x_anchor, x_mode, zx_out, xp_out;
  int y_cur, y_anchor, yp_out, yc_out;
  int ax_cur, ax_anchor, axp_out, axc_out;
  int stop;      // leave the kernel now
  int check;     // run the certificate-scan phases for this iteration
  int pw_mode;   // power: 0 gather x0, 1 gather z / zn
  int cand_on[4];
  int pad0;
  double w_x;        // Halpern weight that forms x in phase A
  double w_next;     // weight of the speculative combos in phase B
  double eta;
  double cand_scale; // 2/k for the normalized candidate
  double cn2[4];     // candidate l2 norms: 0 v_x diff, 1 v_y diff, 2 v_x norm, 3 v_y norm
  double pw_zn;
  // baseline schemes (solve_baseline, src/solver.cpp:344-509): z may live in
  // an average slot after a restart; the running average is updated from
  // slot avg_cur into slot avg_out (avg_mode 1: copy z, 2: w-weighted update)
  int x_src_avg, y_cur_avg, ax_cur_avg;
  int avg_mode, avg_cur, avg_out, avg_step;
  int y_unpushed;  // team: y_cur is a y+ whose owned rows the peers have not received yet (after a restart)
  int tr_slot;     // trace ring slot of this phase's iteration (-1: not traced / no ring)
  int pad_tr;
  double tr_scale; // 2/k of this phase's iteration (the normalized candidate's scale; 0 at k = 0)
  double w_avg;
};

// Trace ring (TraceRecord src/solver.cpp:271-290): one
// record per traced iteration, written by the controller of CTA 0; the
// iterate z and the partition class of every column (0 N, 1 B1, 2 B2,
// src/diagnostics.cpp:26-43) go to the ring's slot arrays from the phase
// epilogues -- the host drains whole batches, no per-record round trip.
struct TraceRec {
  long long it, n, k;
  double res, kkt[4], cand_norm;
  long long cnt[3];  // |N|, |B1|, |B2|
};

// Controller state.  Lives in global memory between launches; during a
// launch every CTA keeps an identical replica in shared memory.
struct Ctl {
  Roles r;
  long long iteration_limit, check_period, stall_cap, k_star, tau0, trace_period;
  int restart_kind, mode;
  double tol, cert_tol, beta, sigma_used, b_norm, c_norm;
  unsigned long long time_budget_ns;  // remaining wall time for this launch
  long long it, n, k, spmv, batch_end, n_epochs;
  double res_epoch_start, best_kkt, best_err[4];
  int x_best, y_best;
  int status, error, paused, x_best_prev;  // x_best before this iteration's update
  long long last_it, last_n, last_k;
  double last_res, last_kkt[4];
  int last_zx, last_y, last_xp, last_yp, last_xa, last_ya, last_ax, last_axp, last_axa, pad1;
  double final_kkt[4];
  int final_x, final_y;
  int cfinite[4];
  double cinf[4], cmax_u[4], cmax_negu[4], cdot[4], cmax_at[4], cmax_negat[4], cmax_abs_au[4];
  hplp_cert_meta_t cert[2];  // 0 primal, 1 dual
  int cert_cand[2];
  double w_k2, w_k3;  // 1/(k+2), 1/(k+3) of the current iteration
  long long pw_k, pw_max, pw_iters;
  double pw_tol, pw_sigma, pw_sigma_prev, pw_sigma_cur;
  int pw_converged, pw_redraw;
  unsigned long long team_epochs;  // cross-rank barriers passed so far (identical on every rank)
  // team setup modes: kModeKkt totals (||Ax - b||^2, ||[-(c + A^T y)]+||^2,
  // c.x, b.y); kModeScale rounds (sc_ruiz Ruiz rounds, then Pock-Chambolle
  // with sc_alpha when sc_pc) and the scaled ||b||^2, ||c||^2
  double kk_tot[4];
  int sc_ruiz, sc_pc;
  double sc_alpha, sc_bsq, sc_csq;
  // trace ring: records written so far / drained by the host, capacity (0: no
  // ring -- a traced iteration pauses the launch instead), partition tolerances
  long long ring_total, ring_drained;
  int ring_cap, pad_ring;
  double r_tol, tol_active;
  // baseline schemes
  int scheme;          // HPLP_SCHEME_*
  int avg_best;        // average slot holding the best candidate (-1: best is a z in the pools)
  int final_avg;       // final iterate = average slot final_avg (>= 0)
  int last_cand_avg;   // traced candidate = average slot (>= 0) or z (-1)
  int last_y_avg;      // traced z's y lives in an average slot
  int pad4;
  long long avg_count; // iterates in the running average
  double last_res_diff;  // ||T(z) - z|| of the last iteration (TraceRecord::candidate_norm_difference)
};
static_assert(sizeof(Ctl) % 8 == 0, "Ctl copied as 8-byte words");

struct GridBar {
  unsigned long long count;  // monotonic arrivals within one launch
  unsigned abort;            // watchdog fired
  unsigned time_up[2];       // time-limit flag, by iteration parity (CTA 0 writes)
  unsigned pad;
  unsigned long long go;     // team barrier: last cross-rank epoch released to this rank's CTAs
};

// Cross-rank barrier word of one rank of a row-partitioned team, on its own
// 128-byte line.  `arrive` counts the arrivals of every rank's leader CTA and
// is monotonic for the context's lifetime (never reset between launches, so a
// fast peer can arrive before this rank's next launch starts); time_up is the
// time-limit flag, written by rank 0 alone so every rank stops together.
constexpr int kRankRecReplicas = 8;  // copies of the rank records: every CTA reads them (L2 hot spot)
constexpr int kPreReduceRecords = 320;
struct RankBar {
  unsigned long long arrive;
  unsigned time_up[2];
  unsigned long long pad[14];
  // rank records of the main reduction, [parity][source rank][quantity]:
  // each rank's leader reduces its own CTAs' phase A/B records and pushes
  // the 7 totals here on every rank (team_sync with reduce), so a
  // controller sums nranks records instead of nranks * grid
  double rrec[2][kRankRecReplicas][kMaxRanks][8];
};

// Row partition of the team plus the peers' buffers.  Rank r
// owns rows [row0, row1) of A (y, A x, b) and columns [col0, col1) (x, c);
// iterate pools are full length on every rank and every owned slice that a
// peer gathers from (x+, the two y candidates, certificate unit vectors) is
// pushed into the peers' pools by the epilogue that produces it: P2P stores
// over NVLink (CUDA IPC mappings) on a multi-GPU node, or plain stores when
// the ranks are emulated as CTA groups of one launch on one device.
// Per-CTA partial records go to every rank's slot regions the same way, so
// each rank reduces all ranks' records locally in one fixed order and the
// replicated controllers stay bit-identical across ranks.
struct Team {
  int rank, nranks, grp_ctas;
  int sys;                  // 1: some peer is another GPU -> system-scope release/acquire
  int prereduce;            // 1: main reduction through rank records (team_sync reduce)
  int row0, row1, col0, col1;
  double* px[kMaxRanks];    // xpool of every rank (px[rank] = own)
  double* py[kMaxRanks];    // ypool
  double* pu[kMaxRanks];    // upool
  double* ps[kMaxRanks];    // slots
  RankBar* pb[kMaxRanks];   // cross-rank barrier words
  // "needed by" rank masks of the owned elements: bit r of xneed[j - col0]
  // is set when one of rank r's rows has column j (rank r gathers x+_j),
  // bit r of yneed[i - row0] when one of rank r's columns has row i -- a
  // push goes only to the ranks that read the element
  const unsigned char* xneed;
  const unsigned char* yneed;
};

// Slot regions (kMaxQ * grid doubles each).  A CTA may still be reading the
// totals of one reduction while a faster CTA writes the next one, so every
// reduction that can overlap its successor has its own region; phases A and
// B alternate by iteration parity.
enum Region : int { kRegA = 0, kRegB = 2, kRegC1 = 4, kRegC2 = 5, kRegC3 = 6, kRegPA = 7, kRegPB = 8, kRegions = 9 };

struct KParams {
  Sched A;   // rows of A
  Sched AT;  // rows of A^T
  int m, n;
  const double* __restrict__ b;
  const double* __restrict__ c;
  double* xpool;   // kXPool * n
  double* ypool;   // kYPool * m
  double* axpool;  // kAxPool * m
  double* upool;   // [u0: n][u2: n][u1: m][u3: m] certificate unit vectors
  double* slots;   // kMaxQ * grid
  Ctl* ctl;
  GridBar* bar;
  hplp_epoch_t* epochs;  // ring of kEpochCap
  unsigned long long* prof;  // optional per-CTA phase timers [grid][8] (HX_PROFILE=1)
  Team T;                    // row partition + peers (loop_kernel_team only)
  const double* ub;          // box form: column upper bounds (+inf: none); null: standard form
  // baseline schemes (loop_kernel_baseline): kAvgPool slots each
  double* xavg;   // n: mean x
  double* tavg;   // n: mean A^T y
  double* yavg;   // m: mean y
  double* aavg;   // m: mean A x
  double* xbar;   // n: x-part of the PDHG step taken at the average
  // column-blocked phase B (loop_kernel_stream_cb): A split at ncb - 1
  // columns into ncb blocks (device array cbs of their schedules), swept one
  // after the other so each sweep's gathers of x+ stay in L2; bpart carries
  // the leading blocks' row sums.  Indexed at run time: the kernels take
  // KParams as __grid_constant__, so that is a register-indexed constant-bank
  // load, not a local copy
  Sched cbs[kMaxColBlocks];
  int ncb;
  double* bpart;  // m
  // trace ring (TraceRec): records, and per slot z.x (n), z.y (m) and the
  // columns' partition classes (n); a rank writes its own slices (peers read
  // them back through CUDA IPC)
  TraceRec* ring_rec;
  double* ring_x;
  double* ring_y;
  unsigned char* ring_cls;
  double r_tol, tol_active;
};

// z's buffers: pool role, or an average slot after a baseline restart.
__device__ __forceinline__ const double* xsrc_ptr(const KParams* P, const Roles* R) {
  return (R->x_src_avg ? P->xavg : P->xpool) + static_cast<size_t>(R->x_src) * P->n;
}
__device__ __forceinline__ const double* ycur_ptr(const KParams* P, const Roles* R) {
  return (R->y_cur_avg ? P->yavg : P->ypool) + static_cast<size_t>(R->y_cur) * P->m;
}
__device__ __forceinline__ const double* axcur_ptr(const KParams* P, const Roles* R) {
  return (R->ax_cur_avg ? P->aavg : P->axpool) + static_cast<size_t>(R->ax_cur) * P->m;
}

// Where this CTA sits: its index among the CTAs of its rank (cta of nctas)
// and its partial record among all ranks' records (rec of nrec).  Single GPU:
// cta = rec = blockIdx.x, nctas = nrec = gridDim.x.
struct Geo {
  int cta, nctas, rec, nrec;
};

// ---------------------------------------------------------------------------
// device helpers
// ---------------------------------------------------------------------------
__device__ __forceinline__ unsigned long long global_ns() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

// Vectors written inside the kernel are read at L2 (ld.global.cg): no stale
// L1 lines across grid barriers.  The matrix, b and c are read-only (ld.nc).
__device__ __forceinline__ double ldcg(const double* p) { return __ldcg(p); }
__device__ __forceinline__ double ldca(const double* p) { return __ldca(p); }

__device__ __forceinline__ double dmax(double a, double b) { return a < b ? b : a; }

__device__ __forceinline__ unsigned long long ld_acquire_u64(const unsigned long long* p) {
  unsigned long long v;
  asm volatile("ld.acquire.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}



__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}
__device__ __forceinline__ double warp_max(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = dmax(v, __shfl_xor_sync(0xffffffffu, v, o));
  return v;
}

template <int Q, unsigned MaxMask>
__device__ __forceinline__ void acc_init(double (&acc)[Q]) {
#pragma unroll
  for (int q = 0; q < Q; ++q) acc[q] = ((MaxMask >> q) & 1u) ? -INFINITY : 0.0;
}

template <int Q, unsigned MaxMask>
__device__ __forceinline__ void acc_add(double (&acc)[Q], const double (&t)[Q]) {
#pragma unroll
  for (int q = 0; q < Q; ++q) acc[q] = ((MaxMask >> q) & 1u) ? dmax(acc[q], t[q]) : acc[q] + t[q];
}

// One shared scratch for every block_to_slots instantiation.
__device__ __forceinline__ double (*red_buf())[kMaxQ] {
  __shared__ double red[kWarps][kMaxQ];
  return red;
}

// Partial-sum records: each CTA publishes its kMaxQ partials of a reduction
// round as one 128-byte record, written to kReplicas copies of the region so
// the (redundant, every-CTA) readers spread over distinct L2 lines.
constexpr int kReplicas = 4;

__device__ __forceinline__ size_t region_stride(int grid) {
  return static_cast<size_t>(kReplicas) * grid * kMaxQ;
}

// Per-thread accumulators -> this CTA's record in every replica (fixed order);
// standalone kernels (record blockIdx.x of gridDim.x).
template <int Q, unsigned MaxMask>
__device__ void block_to_slots(const double (&acc)[Q], double* region, int grid) {
  double (*red)[kMaxQ] = red_buf();
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
  for (int q = 0; q < Q; ++q) {
    const double v = ((MaxMask >> q) & 1u) ? warp_max(acc[q]) : warp_sum(acc[q]);
    if (lane == 0) red[warp][q] = v;
  }
  __syncthreads();
  if (threadIdx.x < Q * kReplicas) {
    const int q = threadIdx.x % Q, k = threadIdx.x / Q;
    const bool mx = (MaxMask >> q) & 1u;
    double v = red[0][q];
    for (int w = 1; w < kWarps; ++w) v = mx ? dmax(v, red[w][q]) : v + red[w][q];
    region[(static_cast<size_t>(k) * grid + blockIdx.x) * kMaxQ + q] = v;
  }
}

// Loop-kernel version: record g.rec of g.nrec in slot region `region`; a
// ranked CTA writes it into every rank's slots (own included), so all ranks
// hold all records.
template <int Q, unsigned MaxMask, bool RK, class KP>
__device__ void block_to_slots(const double (&acc)[Q], const KP* P, int region, const Geo& g) {
  double (*red)[kMaxQ] = red_buf();
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
  for (int q = 0; q < Q; ++q) {
    const double v = ((MaxMask >> q) & 1u) ? warp_max(acc[q]) : warp_sum(acc[q]);
    if (lane == 0) red[warp][q] = v;
  }
  __syncthreads();
  if (threadIdx.x < Q * kReplicas) {
    const int q = threadIdx.x % Q, k = threadIdx.x / Q;
    const bool mx = (MaxMask >> q) & 1u;
    double v = red[0][q];
    for (int w = 1; w < kWarps; ++w) v = mx ? dmax(v, red[w][q]) : v + red[w][q];
    const size_t off = static_cast<size_t>(region) * region_stride(g.nrec) +
                       (static_cast<size_t>(k) * g.nrec + g.rec) * kMaxQ + q;
    if constexpr (RK) {
      // with rank records the main reduction's records stay local: the leader
      // pre-reduces them at the end-of-iteration barrier (team_sync)
      if (P->T.prereduce && region < kRegC1) P->slots[off] = v;
      else
        for (int r = 0; r < P->T.nranks; ++r) P->T.ps[r][off] = v;
    } else {
      P->slots[off] = v;
    }
  }
}

// Source of one reduced quantity: records of a region (+ optional long-row
// terms), column rq / lq of the 16-wide records.
struct QSrc {
  const double* region;
  int rq;
  const double* lt;
  int n_long;
  int lq;
  bool mx;
};

// Totals of up to kMaxQ quantities, computed by the whole CTA in a fixed
// order: thread t handles quantity t % kMaxQ over records t / kMaxQ + kJ k,
// then thread q combines the kJ partials in index order.  Every CTA computes
// bit-identical totals.  Desc: q -> QSrc.
constexpr int kJ = kThreads / kMaxQ;
// One shared scratch for every block_totals instantiation.
__device__ __forceinline__ double (*part_buf())[kJ][kMaxQ] {
  __shared__ double part[2][kJ][kMaxQ];
  return part;
}

template <class Desc>
__device__ void block_totals(int Q, const Desc& desc, double* tot, const Geo& g) {
  double (*part)[kJ][kMaxQ] = part_buf();
  const int q = threadIdx.x % kMaxQ, j = threadIdx.x / kMaxQ;
  const int G = g.nrec;
  if (q < Q) {
    const QSrc d = desc(q);
    const double* rec = d.region + static_cast<size_t>(g.cta % kReplicas) * G * kMaxQ;
    double v = d.mx ? -INFINITY : 0.0, l = v;
    for (int c = j; c < G; c += kJ) {
      const double x = ldcg(rec + static_cast<size_t>(c) * kMaxQ + d.rq);
      v = d.mx ? dmax(v, x) : v + x;
    }
    if (d.lt)
      for (int c = j; c < d.n_long; c += kJ) {
        const double x = ldcg(d.lt + static_cast<size_t>(c) * kMaxQ + d.lq);
        l = d.mx ? dmax(l, x) : l + x;
      }
    part[0][j][q] = v;
    part[1][j][q] = l;
  }
  __syncthreads();
  if (threadIdx.x < Q) {
    const QSrc d = desc(threadIdx.x);
    double v = part[0][0][threadIdx.x], l = part[1][0][threadIdx.x];
    for (int jj = 1; jj < kJ; ++jj) {
      v = d.mx ? dmax(v, part[0][jj][threadIdx.x]) : v + part[0][jj][threadIdx.x];
      l = d.mx ? dmax(l, part[1][jj][threadIdx.x]) : l + part[1][jj][threadIdx.x];
    }
    tot[threadIdx.x] = d.lt ? (d.mx ? dmax(v, l) : v + l) : v;
  }
  __syncthreads();
}

__device__ __forceinline__ double warp_reduce_strided(const double* p, int count, int stride, bool mx) {
  const int lane = threadIdx.x & 31;
  double v = mx ? -INFINITY : 0.0;
  for (int i = lane; i < count; i += 32) {
    const double s = ldcg(p + static_cast<long long>(i) * stride);
    v = mx ? dmax(v, s) : v + s;
  }
  return mx ? warp_max(v) : warp_sum(v);
}

// ---------------------------------------------------------------------------
// Fused SpMV engine (task kinds in hx_internal.cuh).
//
// Warp w runs tasks w, w + W, ... (static round robin: deterministic and
// statistically balanced).  Per task each lane issues kLoadsPerLane
// independent index/value loads and then as many independent gathers --
// all in registers; B200 measurements (tools/spmv_micro.cu) show register
// loads with a large L1 beat shared-memory staging for random fp64 gathers.
// Stream tasks write the products to a 2 KB per-warp buffer and sum them
// lane-per-row over ascending columns (the reference's order,
// src/sparse_matrix.cpp:108-115, split into even/odd partial sums: HX_RSUM);
// pieces are summed warp-wide.  The row
// epilogue's inputs are loaded before the gathers so their latency overlaps.
// Epi: load(row) / apply(row, sum, inputs, terms[Q]).  Terms of regular rows
// accumulate per thread; a long row's terms are parked in long_terms by
// whichever warp finishes it, so every reduction keeps a fixed order.
// ---------------------------------------------------------------------------
struct alignas(16) WarpStage {
  double prod[kChunk];
};
constexpr size_t kStageBytes = sizeof(WarpStage) * kWarps;

// Index/value registers of one task (kLoadsPerLane per lane).
struct TaskRegs {
  int ci[kLoadsPerLane];
  double cv[kLoadsPerLane];
};

// L2 eviction priority for the matrix streams (createpolicy): they are read
// once per phase, so when the per-iteration working set exceeds what the
// 126 MB L2 keeps (Sched::stream_hint, set at upload), they are loaded
// evict_first and without L1 allocation -- the vectors every SM gathers from
// and the epilogue's pools then stay in L2 between phases.  Measured on
// configs[1] (tools/quick_rate.py A/B): 25.65k -> 26.79k it/s; the box form's
// working set fits in L2 and runs faster without the hint (32.3k vs 30.6k).
__device__ __forceinline__ unsigned long long l2_policy_first() {
  unsigned long long p;
  asm("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
  return p;
}
__device__ __forceinline__ int ldg_stream(const int* p, unsigned long long pol) {
  int v;
  asm volatile("ld.global.nc.L1::no_allocate.L2::cache_hint.s32 %0, [%1], %2;" : "=r"(v) : "l"(p), "l"(pol));
  return v;
}
__device__ __forceinline__ double ldg_stream(const double* p, unsigned long long pol) {
  double v;
  asm volatile("ld.global.nc.L1::no_allocate.L2::cache_hint.f64 %0, [%1], %2;" : "=d"(v) : "l"(p), "l"(pol));
  return v;
}

__device__ __forceinline__ unsigned long long l2_policy_normal() {
  unsigned long long p;
  asm("createpolicy.fractional.L2::evict_normal.b64 %0, 1.0;" : "=l"(p));
  return p;
}

// Epilogue streams of the stream kernel (EF, HX_EPI_EF): 1 loads evict_first,
// 2 loads and stores evict_first -- for working sets far beyond L2, where the
// gather targets should own the cache.
template <int EF>
__device__ __forceinline__ double ld_epi(const double* p) {
  if constexpr (EF >= 1) {
    double v;
    asm volatile("ld.global.cg.L2::cache_hint.f64 %0, [%1], %2;" : "=d"(v) : "l"(p), "l"(l2_policy_first()));
    return v;
  } else {
    return ldcg(p);
  }
}
template <int EF>
__device__ __forceinline__ void st_epi(double* p, double v) {
  if constexpr (EF >= 2) {
    asm volatile("st.global.L2::cache_hint.f64 [%0], %1, %2;" ::"l"(p), "d"(v), "l"(l2_policy_first()) : "memory");
  } else {
    *p = v;
  }
}

// LM: 0 plain read-only loads, 1 evict_first streams, 2 chosen at run time by
// S.stream_hint (one load sequence with a selected policy)
#if HX_VEC
// Vectorised task loads (HX_VEC): the window starts at the even index
// pa = p0 & ~1 and lane l holds elements e = 64 (j / 2) + 2 l + (j & 1) of
// it, loaded as int2 / double2 pairs (half the load instructions); elements
// outside [p0, p1) are zero.  Tasks hold at most kChunk - 1 nonzeros so the
// shifted window fits kChunk slots; the matrix arrays carry a few padding
// elements, so a pair starting at the last nonzero stays in bounds.
__device__ __forceinline__ int vec_e(int j, int lane) { return (j >> 1) * 64 + 2 * lane + (j & 1); }
template <int LM>
__device__ __forceinline__ void load_task(const Sched& S, const int4& tk, int lane, TaskRegs& r) {
  const int p0 = tk.z, pa = p0 & ~1, e0 = p0 - pa, e1 = tk.w - pa;
  HX_CHECK(tk.w - p0 >= 0 && e1 <= kChunk && p0 >= 0, "task nnz range", p0, tk.w - p0);
  [[maybe_unused]] const unsigned long long pol =
      LM == 0 ? 0ull : (LM == 1 || S.stream_hint ? l2_policy_first() : l2_policy_normal());
#pragma unroll
  for (int jj = 0; jj < kLoadsPerLane / 2; ++jj) {
    const int e = jj * 64 + 2 * lane;
    int2 iv = make_int2(0, 0);
    double2 vv = make_double2(0.0, 0.0);
    if (e < e1) {
      const int2* ip = reinterpret_cast<const int2*>(S.idx + pa + e);
      const double2* vp = reinterpret_cast<const double2*>(S.val + pa + e);
      if constexpr (LM == 0) {
        iv = __ldg(ip);
        vv = __ldg(vp);
      } else {
        asm volatile("ld.global.nc.L1::no_allocate.L2::cache_hint.v2.s32 {%0, %1}, [%2], %3;"
                     : "=r"(iv.x), "=r"(iv.y) : "l"(ip), "l"(pol));
        asm volatile("ld.global.nc.L1::no_allocate.L2::cache_hint.v2.f64 {%0, %1}, [%2], %3;"
                     : "=d"(vv.x), "=d"(vv.y) : "l"(vp), "l"(pol));
      }
    }
    const bool v0 = e >= e0 && e < e1, v1 = e + 1 < e1;
    r.ci[2 * jj] = v0 ? iv.x : 0;
    r.cv[2 * jj] = v0 ? vv.x : 0.0;
    r.ci[2 * jj + 1] = v1 ? iv.y : 0;
    r.cv[2 * jj + 1] = v1 ? vv.y : 0.0;
  }
}
#else
template <int LM>
__device__ __forceinline__ void load_task(const Sched& S, const int4& tk, int lane, TaskRegs& r) {
  const int p0 = tk.z, len = tk.w - tk.z;
  HX_CHECK(len >= 0 && len <= kChunk && p0 >= 0, "task nnz range", p0, len);
  if constexpr (LM == 0) {
#pragma unroll
    for (int j = 0; j < kLoadsPerLane; ++j) {
      const int q = j * 32 + lane;
      r.ci[j] = q < len ? __ldg(S.idx + p0 + q) : 0;
      r.cv[j] = q < len ? __ldg(S.val + p0 + q) : 0.0;
    }
  } else {
    const unsigned long long pol = LM == 1 || S.stream_hint ? l2_policy_first() : l2_policy_normal();
#pragma unroll
    for (int j = 0; j < kLoadsPerLane; ++j) {
      const int q = j * 32 + lane;
      r.ci[j] = q < len ? ldg_stream(S.idx + p0 + q, pol) : 0;
      r.cv[j] = q < len ? ldg_stream(S.val + p0 + q, pol) : 0.0;
    }
  }
}
#endif

// The pipeline's head: the first two task descriptors and the first task's
// index/value registers.  They depend only on the (read-only) matrix, so a
// phase's head is loaded before the grid barrier that precedes the phase and
// its latency hides behind the barrier wait.
struct SpmvHead {
  int4 tk, tk1;
  TaskRegs cur;
};

template <int LM = 0>
__device__ __forceinline__ void spmv_head(const Sched& S, int gwarp, int lane, SpmvHead& h) {
  const int W = S.W;
  const int n = S.n_tasks;
  const int4 kNone{0, 0, 0, 0};
  h.tk = gwarp < n ? __ldg(S.tasks + gwarp) : kNone;
  h.tk1 = gwarp + W < n ? __ldg(S.tasks + gwarp + W) : kNone;
  load_task<LM>(S, h.tk, lane, h.cur);
}

// EX: summation order -- 0 the fast order, 1 the reference's (Sched::exact),
// 2 chosen at run time by S.exact (the main loop kernels compile it out: the
// run-time branch costs them registers)
template <int Q, unsigned MaxMask, int LM = 0, int EX = 2, class Src, class Epi>
__device__ __forceinline__ void spmv_rows(const Sched& S, int set, const Src& src, Epi& epi, double (&acc)[Q],
                                          int gwarp, int lane, WarpStage* st, unsigned long long seq,
                                          const SpmvHead& head) {
  const bool exact = EX == 1 || (EX == 2 && S.exact);
  const int W = S.W;
  const int n = S.n_tasks;
  const int4 kNone{0, 0, 0, 0};
  int t = gwarp;
  if (t >= n) return;
  // software pipeline: descriptors two tasks ahead, index/value loads one
  // task ahead of the gathers
  int4 tk = head.tk;
  int4 tk1 = head.tk1;
  TaskRegs cur = head.cur;
  double run_acc = 0.0;  // this lane's partial sum of the current run of long-row pieces
  for (; t < n; t += W) {
    const int4 tk2 = t + 2 * W < n ? __ldg(S.tasks + t + 2 * W) : kNone;
    TaskRegs nxt;
    load_task<LM>(S, tk1, lane, nxt);
    const int r0 = tk.x, r1 = tk.y & kRowMask, kind = task_kind(tk.y);
#if HX_VEC
    const int p0 = tk.z & ~1, len = tk.w - p0;  // the window's base and extent
#else
    const int p0 = tk.z, len = tk.w - tk.z;
#endif
    HX_CHECK(r0 >= 0 && r1 >= r0 && r1 <= S.row_limit, "task rows", r0, r1);
    // stream tasks: up to two rows per lane (lane, lane + 32); their bounds and
    // epilogue inputs are loaded before the gathers so the latencies overlap
    const int nrows = r1 - r0;
    const bool has_row = kind == kTaskStream && lane < nrows;
    const bool has_row2 = kStreamRowsMax > 32 && kind == kTaskStream && lane + 32 < nrows;
    int ra = 0, rb = 0, ra2 = 0, rb2 = 0;
    typename Epi::In in{}, in2{};
    if (has_row) {
      ra = __ldg(S.ptr + r0 + lane);
      rb = min(__ldg(S.ptr + r0 + lane + 1), tk.w);  // a staggered copy's alignment gap ends a task
      HX_CHECK(ra >= p0 && rb >= ra && rb - p0 <= kChunk, "stream row in task", ra - p0, rb - p0);
      in = epi.load(r0 + lane);
    }
#if HX_RSPLIT
    // short task (<= 16 rows): two lanes per row, lane l + 16 sums the tail
    // half of row l (phase B of configs[1]: ~12 rows of ~20 nonzeros)
    const bool split = kind == kTaskStream && nrows <= 16;
    if (split && lane >= 16 && lane - 16 < nrows) {
      ra = __ldg(S.ptr + r0 + lane - 16);
      rb = __ldg(S.ptr + r0 + lane - 15);
    }
#endif
    if (has_row2) {
      ra2 = __ldg(S.ptr + r0 + lane + 32);
      rb2 = min(__ldg(S.ptr + r0 + lane + 33), tk.w);
      HX_CHECK(ra2 >= p0 && rb2 >= ra2 && rb2 - p0 <= kChunk, "stream row 2 in task", ra2 - p0, rb2 - p0);
      in2 = epi.load(r0 + lane + 32);
    }
#pragma unroll
    for (int j = 0; j < kLoadsPerLane; ++j) {
#if HX_VEC
      const int q = vec_e(j, lane);
      const bool live = q >= tk.z - p0 && q < len;
#else
      const int q = j * 32 + lane;
      const bool live = q < len;
#endif
      HX_CHECK(!live || (cur.ci[j] >= 0 && cur.ci[j] < S.cols), "gather index", cur.ci[j], S.cols);
      if (live) cur.cv[j] = cur.cv[j] * src(cur.ci[j]);
    }
    if (kind == kTaskStream) {
#if HX_VEC
#pragma unroll
      for (int jj = 0; jj < kLoadsPerLane / 2; ++jj)
        reinterpret_cast<double2*>(st->prod)[jj * 32 + lane] = make_double2(cur.cv[2 * jj], cur.cv[2 * jj + 1]);
#else
#pragma unroll
      for (int j = 0; j < kLoadsPerLane; ++j) st->prod[j * 32 + lane] = cur.cv[j];
#endif
      __syncwarp();
#if HX_RSUM == 1
      // two interleaved partial sums (even / odd positions), combined at the
      // end: half the dependent-add chain; rows of <= 2 nonzeros keep the
      // reference's exact order.  S.exact: one sequential chain (the
      // reference's order for every row).
      auto row_sum = [&](int qa, int qe) {
        if (exact) {
          double s = 0.0;
          for (int q = qa; q < qe; ++q) s += st->prod[q];
          return s;
        }
        double s0 = 0.0, s1 = 0.0;
        int q = qa;
        for (; q + 4 <= qe; q += 4) {
          const double a0 = st->prod[q], a1 = st->prod[q + 1], a2 = st->prod[q + 2], a3 = st->prod[q + 3];
          s0 += a0;
          s1 += a1;
          s0 += a2;
          s1 += a3;
        }
        if (q + 2 <= qe) {
          const double a0 = st->prod[q], a1 = st->prod[q + 1];
          s0 += a0;
          s1 += a1;
          q += 2;
        }
        if (q < qe) s0 += st->prod[q];
        return s0 + s1;
      };
#elif HX_RSUM == 2
      // four interleaved partial sums (positions mod 4), combined pairwise
      auto row_sum = [&](int qa, int qe) {
        double s0 = 0.0, s1 = 0.0, s2 = 0.0, s3 = 0.0;
        int q = qa;
        for (; q + 4 <= qe; q += 4) {
          const double a0 = st->prod[q], a1 = st->prod[q + 1], a2 = st->prod[q + 2], a3 = st->prod[q + 3];
          s0 += a0;
          s1 += a1;
          s2 += a2;
          s3 += a3;
        }
        if (q < qe) s0 += st->prod[q];
        if (q + 1 < qe) s1 += st->prod[q + 1];
        if (q + 2 < qe) s2 += st->prod[q + 2];
        return (s0 + s1) + (s2 + s3);
      };
#elif HX_RSUM == 3
      // two interleaved partial sums, loads issued 8 ahead
      auto row_sum = [&](int qa, int qe) {
        double s0 = 0.0, s1 = 0.0;
        int q = qa;
        for (; q + 8 <= qe; q += 8) {
          double a[8];
#pragma unroll
          for (int k = 0; k < 8; ++k) a[k] = st->prod[q + k];
#pragma unroll
          for (int k = 0; k < 8; k += 2) {
            s0 += a[k];
            s1 += a[k + 1];
          }
        }
        for (; q + 2 <= qe; q += 2) {
          const double a0 = st->prod[q], a1 = st->prod[q + 1];
          s0 += a0;
          s1 += a1;
        }
        if (q < qe) s0 += st->prod[q];
        return s0 + s1;
      };
#elif HX_RSUM == 4
      // HX_RSUM 1's order (two interleaved partial sums), software-pipelined:
      // the next four products are loaded before the current four are added,
      // so the adds never hold back the next loads
      auto row_sum = [&](int qa, int qe) {
        if (exact) {
          double s = 0.0;
          for (int q = qa; q < qe; ++q) s += st->prod[q];
          return s;
        }
        double s0 = 0.0, s1 = 0.0;
        int q = qa;
        if (q + 4 <= qe) {
          double a0 = st->prod[q], a1 = st->prod[q + 1], a2 = st->prod[q + 2], a3 = st->prod[q + 3];
          for (q += 4; q + 4 <= qe; q += 4) {
            const double b0 = st->prod[q], b1 = st->prod[q + 1], b2 = st->prod[q + 2], b3 = st->prod[q + 3];
            s0 += a0;
            s1 += a1;
            s0 += a2;
            s1 += a3;
            a0 = b0, a1 = b1, a2 = b2, a3 = b3;
          }
          s0 += a0;
          s1 += a1;
          s0 += a2;
          s1 += a3;
        }
        if (q + 2 <= qe) {
          const double a0 = st->prod[q], a1 = st->prod[q + 1];
          s0 += a0;
          s1 += a1;
          q += 2;
        }
        if (q < qe) s0 += st->prod[q];
        return s0 + s1;
      };
#else
      // ascending-order sums (the reference's), loads issued 4 ahead
      auto row_sum = [&](int qa, int qe) {
        double s = 0.0;
        int q = qa;
        for (; q + 4 <= qe; q += 4) {
          const double a0 = st->prod[q], a1 = st->prod[q + 1], a2 = st->prod[q + 2], a3 = st->prod[q + 3];
          s += a0;
          s += a1;
          s += a2;
          s += a3;
        }
        for (; q < qe; ++q) s += st->prod[q];
        return s;
      };
#endif
#if HX_RSPLIT
      if (split) {
        const int qa = ra - p0, qe = rb - p0, qm = qa + ((qe - qa + 1) >> 1);
        double part = 0.0;
        if ((lane & 15) < nrows) part = lane < 16 ? row_sum(qa, qm) : row_sum(qm, qe);
        const double tail = __shfl_down_sync(0xffffffffu, part, 16);
        if (has_row) {
          double tm[Q];
          epi.apply(r0 + lane, part + tail, in, tm);
          acc_add<Q, MaxMask>(acc, tm);
        }
      } else
#endif
#if HX_RSHORT
      // both of a lane's rows of <= 4 nonzeros (slack columns, bound rows):
      // all eight products loaded in one round, summed in HX_RSUM 1's order
      // (s0 = 0 + a0 + a2, s1 = 0 + a1 + a3; a missing product adds +0.0,
      // which leaves the bits alone: s0, s1 start at +0.0)
      if (!exact && rb - ra <= 4 && rb2 - ra2 <= 4) {
        double v[8];
#pragma unroll
        for (int k = 0; k < 4; ++k) {
          v[k] = k < rb - ra ? st->prod[ra - p0 + k] : 0.0;
          v[4 + k] = k < rb2 - ra2 ? st->prod[ra2 - p0 + k] : 0.0;
        }
        if (has_row) {
          double tm[Q];
          epi.apply(r0 + lane, ((0.0 + v[0]) + v[2]) + ((0.0 + v[1]) + v[3]), in, tm);
          acc_add<Q, MaxMask>(acc, tm);
        }
        if (has_row2) {
          double tm[Q];
          epi.apply(r0 + lane + 32, ((0.0 + v[4]) + v[6]) + ((0.0 + v[5]) + v[7]), in2, tm);
          acc_add<Q, MaxMask>(acc, tm);
        }
      } else
#endif
      {
        if (has_row) {
          double tm[Q];
          epi.apply(r0 + lane, row_sum(ra - p0, rb - p0), in, tm);
          acc_add<Q, MaxMask>(acc, tm);
        }
        if (has_row2) {
          double tm[Q];
          epi.apply(r0 + lane + 32, row_sum(ra2 - p0, rb2 - p0), in2, tm);
          acc_add<Q, MaxMask>(acc, tm);
        }
      }
      __syncwarp();
    } else if (exact) {
      // reference order: the products go through the staging buffer and lane 0
      // adds them, in ascending index order, onto the sum the run carries
      // (every long row is a single run in this mode: build_schedule exact)
#pragma unroll
      for (int j = 0; j < kLoadsPerLane; ++j) st->prod[j * 32 + lane] = cur.cv[j];
      __syncwarp();
      if (lane == 0) {
        double a = run_acc;
        for (int q = 0; q < len; ++q) a += st->prod[q];
        run_acc = a;
      }
      __syncwarp();
      if (kind == kTaskPiece && lane == 0) {
        const int4 meta = __ldg(S.meta + t);
        HX_CHECK(meta.y == 1, "exact-order long row split into runs", meta.y, t);
        double tm[Q];
        epi.apply(r0, run_acc, epi.load(r0), tm);
        acc_add<Q, MaxMask>(acc, tm);
      }
      if (kind == kTaskPiece) run_acc = 0.0;
    } else {
#if HX_PSUM
      // pairwise tree over the lane's products (fixed order, short chain)
      double pv[kLoadsPerLane];
#pragma unroll
      for (int j = 0; j < kLoadsPerLane; ++j) pv[j] = cur.cv[j];
#pragma unroll
      for (int w = 1; w < kLoadsPerLane; w *= 2)
#pragma unroll
        for (int j = 0; j + w < kLoadsPerLane; j += 2 * w) pv[j] += pv[j + w];
      double s = pv[0];
#else
      double s = 0.0;
#pragma unroll
      for (int j = 0; j < kLoadsPerLane; ++j) s += cur.cv[j];
#endif
      // a run's pieces: each lane's partial stays in registers until the
      // run's last piece, which reduces it across the warp once
      if (kind == kTaskPieceRun) {
        run_acc += s;
        s = 0.0;
      } else {
        s = warp_sum(run_acc + s);
        run_acc = 0.0;
      }
      if (lane == 0 && kind == kTaskPiece) {
        const int4 meta = __ldg(S.meta + t);  // {slot, nruns, counter, run index}
        HX_CHECK(meta.x >= 0 && meta.x < S.n_slots + (meta.y == 1 ? 1 : 0) && meta.z < S.n_long, "piece slot", meta.x,
                 meta.z);
        if (meta.y == 1) {
          double tm[Q];
          epi.apply(r0, s, epi.load(r0), tm);
          acc_add<Q, MaxMask>(acc, tm);
        } else {
          double* part = S.piece_part(set);
          part[meta.x] = s;
          __threadfence();
          const unsigned old = atomicAdd(S.piece_cnt(set) + meta.z, 1u);
          if (old == static_cast<unsigned>(meta.y - 1)) {
            __threadfence();
            const int first = meta.x - meta.w;
            double tot = 0.0;
            for (int i = 0; i < meta.y; ++i) tot += ldcg(part + first + i);
            S.piece_cnt(set)[meta.z] = 0u;
            double tm[Q];
            epi.apply(r0, tot, epi.load(r0), tm);
            double* lt = S.long_terms(set) + static_cast<long long>(meta.z) * kMaxQ;
#pragma unroll
            for (int q = 0; q < Q; ++q) lt[q] = tm[q];
            // publish to the owner CTA (fold_long): terms before flag
            asm volatile("st.release.gpu.global.u64 [%0], %1;" ::"l"(S.long_flag(set) + meta.z), "l"(seq) : "memory");
          }
        }
      }
    }
    tk = tk1;
    tk1 = tk2;
    cur = nxt;
  }
}

template <int Q, unsigned MaxMask, int LM = 0, int EX = 2, class Src, class Epi>
__device__ __forceinline__ void spmv_rows(const Sched& S, int set, const Src& src, Epi& epi, double (&acc)[Q],
                                          int gwarp, int lane, WarpStage* st, unsigned long long seq = 1) {
  SpmvHead head;
  spmv_head<LM>(S, gwarp, lane, head);
  spmv_rows<Q, MaxMask, LM, EX>(S, set, src, epi, acc, gwarp, lane, st, seq, head);
}

// Owner side of the long-row protocol: warp 0 waits for each owned long row
// of this phase (flag == seq) and folds its terms, in list order, into
// lane 0's accumulators -- a fixed order, so totals stay bit-reproducible.
template <int Q, unsigned MaxMask>
__device__ __forceinline__ void fold_long(const Sched& S, int set, unsigned long long seq, double (&acc)[Q],
                                          int cta, unsigned* abort_flag) {
  if (S.n_long == 0 || threadIdx.x >= 32) return;
  const int lane = threadIdx.x;
  const int b = __ldg(S.owned_ptr + cta), e = __ldg(S.owned_ptr + cta + 1);
  double part[Q];
  acc_init<Q, MaxMask>(part);
  const unsigned long long* flags = S.long_flag(set);
  for (int i = b + lane; i < e; i += 32) {
    const int k = __ldg(S.owned_idx + i);
    const unsigned long long t0 = global_ns();
    while (ld_acquire_u64(flags + k) < seq) {
      if (global_ns() - t0 > 10000000000ull) {  // watchdog: raise the abort flag the next barrier reports
        atomicExch(abort_flag, 1u);
        break;
      }
    }
    const double* lt = S.long_terms(set) + static_cast<long long>(k) * kMaxQ;
    double t[Q];
#pragma unroll
    for (int q = 0; q < Q; ++q) t[q] = ldcg(lt + q);
    acc_add<Q, MaxMask>(part, t);
  }
#pragma unroll
  for (int q = 0; q < Q; ++q) {
    const double v = ((MaxMask >> q) & 1u) ? warp_max(part[q]) : warp_sum(part[q]);
    if (lane == 0) acc[q] = ((MaxMask >> q) & 1u) ? dmax(acc[q], v) : acc[q] + v;
  }
}

// ---- gather sources --------------------------------------------------------
// Kernel-written vectors are gathered through L1 (ld.global.ca would also
// do): every grid barrier's gpu-scope fence invalidates L1 (CCTL.IVALL), so
// no stale line survives into the next phase.
// Gather source.  LAST: loads ask L2 for evict_last (the stream kernel, whose
// matrix streams are evict_first): +0.4% on configs[1].
template <bool LAST = false>
struct SrcVecT {
  const double* v;
  __device__ __forceinline__ double operator()(int j) const {
    if constexpr (LAST) {
      unsigned long long pol;
      asm("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(pol));
      double r;
      asm volatile("ld.global.ca.L2::cache_hint.f64 %0, [%1], %2;" : "=d"(r) : "l"(v + j), "l"(pol));
      return r;
    } else {
      return ldca(v + j);
    }
  }
};
using SrcVec = SrcVecT<false>;
struct SrcDiv {  // power iteration: x = z / ||z|| formed on the fly (same rounding)
  const double* v;
  double d;
  __device__ __forceinline__ double operator()(int j) const { return ldca(v + j) / d; }
};

// ---- epilogues -------------------------------------------------------------
struct NoIn {};

// Ranked epilogues push each owned element a peer gathers into every other
// rank's pool at the same offset (P2P stores on a multi-GPU node).
__device__ __forceinline__ void push_peers(const Team* T, double* const* base, size_t off, double v, unsigned mask) {
  while (mask) {
    const int r = __ffs(mask) - 1;
    mask &= mask - 1;
    base[r][off] = v;
  }
}

// BOX: the box form -- column upper
// bounds u enforced by the projection instead of bound rows: x+ is clamped to
// [0, u], the dual residual counts only columns without a finite bound, and a
// fourth partial carries u_j [-(c + A^T y)_j]^+ (the bound part of the dual
// objective).
// TR: a trace-ring kernel -- a traced iteration (rx non-null) also writes z.x
// and the column's partition class to the ring and adds the class counts and
// ||(2/k)(x - anchor)||^2 as partials NQB..NQB+3.
template <bool RK, bool BOX = false, int EF = 0, bool TR = false>
struct EpiPrimal {  // phase A, rows of A^T
  static constexpr int NQB = BOX ? 4 : 3;
  static constexpr int NQ = NQB + (TR ? 4 : 0);
  const double* xs;
  const double* xa;
  const double* c;
  double* zx;
  double* xp;
  double w, eta;
  int mode;
  const Team* T;   // RK: peers of the x+ push
  size_t xp_off;   // offset of x+ in the x pools
  const double* ub;  // BOX: upper bounds (+inf: none)
  double* rx;             // TR: the ring slot's x (null: iteration not traced)
  unsigned char* rcls;    // TR: the ring slot's partition classes
  double r_tol, tol_active, tr_scale;
  struct In {
    double xs, xa, c, u;
  };
  __device__ __forceinline__ In load(int j) const {
    return In{ld_epi<EF>(xs + j), mode ? ld_epi<EF>(xa + j) : 0.0, EF ? ld_epi<EF>(c + j) : __ldg(c + j),
              BOX ? __ldg(ub + j) : 0.0};
  }
  __device__ __forceinline__ void apply(int j, double aty, const In& in, double (&t)[NQ]) const {
    double x;
    if (mode) {
      const double omw = 1.0 - w;
      x = omw * in.xs + w * in.xa;
    } else {
      x = in.xs;
    }
    st_epi<EF>(zx + j, x);
    const double cj = in.c;
    double xn = x - eta * (aty + cj);
    xn = xn < 0.0 ? 0.0 : xn;
    if constexpr (BOX) xn = xn > in.u ? in.u : xn;
    xp[j] = xn;
    if constexpr (RK)
      if (T->nranks > 1) push_peers(T, T->px, xp_off + j, xn, __ldg(T->xneed + (j - T->col0)));
    double rc = -(cj + aty);
    rc = rc < 0.0 ? 0.0 : rc;
    const double dx = x - xn;
    if constexpr (BOX) {
      const bool bounded = in.u < INFINITY;
      t[0] = bounded ? 0.0 : rc * rc;
      t[3] = bounded ? in.u * rc : 0.0;
    } else {
      t[0] = rc * rc;
    }
    t[1] = cj * x;
    t[2] = dx * dx;
    if constexpr (TR) {
      // partition_estimate_from_reduced_costs (src/diagnostics.cpp:26-43) on
      // the reduced cost c + A^T y (src/solver.cpp:278-279) and z.x
      t[NQB] = t[NQB + 1] = t[NQB + 2] = t[NQB + 3] = 0.0;
      if (rx) {
        rx[j] = x;
        const double r = cj + aty;
        const int cls = r > r_tol ? 0 : (fabs(r) <= r_tol && x > tol_active ? 1 : 2);
        rcls[j] = static_cast<unsigned char>(cls);
        t[NQB + cls] = 1.0;
        const double dxn = tr_scale * (x - in.xa);  // (2/k)(z - anchor), src/solver.cpp:284
        t[NQB + 3] = dxn * dxn;
      }
    }
  }
};

// TR: a traced iteration (ry non-null) writes z.y to the ring and adds the
// normalized candidate's ||dy||^2, dy.d(Ax) as partials 4, 5.
template <bool RK, int EF = 0, bool PART = false, bool TR = false>
struct EpiDual {  // phase B, rows of A
  static constexpr int NQ = TR ? 6 : 4;
  const double* y;
  const double* ax;
  const double* b;
  const double* ya;
  const double* axa;
  double* yp;
  double* axp;
  double* yc;
  double* axc;
  double eta, w;
  const Team* T;          // RK: peers of the y+ / combo push
  size_t yp_off, yc_off;  // offsets of y+ and the combo in the y pools
  const double* part;     // PART: the leading column block's row sums (column-blocked phase B)
  double* ry;             // TR: the ring slot's y (null: iteration not traced)
  double tr_scale;
  struct In {
    double y, ax, b, ya, axa, p;
  };
  __device__ __forceinline__ In load(int i) const {
    return In{ld_epi<EF>(y + i),  ld_epi<EF>(ax + i), EF ? ld_epi<EF>(b + i) : __ldg(b + i), ld_epi<EF>(ya + i),
              ld_epi<EF>(axa + i), PART ? ldcg(part + i) : 0.0};
  }
  __device__ __forceinline__ void apply(int i, double s1, const In& in, double (&t)[NQ]) const {
    // column-blocked: the row's sum is the leading block's plus this block's
    const double s = PART ? in.p + s1 : s1;
    const double yi = in.y;
    const double axi = in.ax;
    const double bi = in.b;
    const double ypi = yi + eta * ((2.0 * s - axi) - bi);
    st_epi<EF>(yp + i, ypi);
    st_epi<EF>(axp + i, s);
    const double omw = 1.0 - w;
    const double yci = omw * ypi + w * in.ya;
    yc[i] = yci;
    // only the combo -- the next y when there is no restart, which phase A
    // gathers speculatively; after a restart the loop pushes y+ itself
    if constexpr (RK)
      if (T->nranks > 1) push_peers(T, T->py, yc_off + i, yci, __ldg(T->yneed + (i - T->row0)));
    st_epi<EF>(axc + i, omw * s + w * in.axa);
    const double d = axi - bi;
    const double dy = yi - ypi;
    const double dax = axi - s;
    t[0] = d * d;
    t[1] = bi * yi;
    t[2] = dy * dy;
    t[3] = dy * dax;
    if constexpr (TR) {
      t[4] = t[5] = 0.0;
      if (ry) {
        ry[i] = yi;
        // (2/k)(z - anchor) and (2/k)(a_x - a_x_anchor), src/solver.cpp:284-286
        const double dyn = tr_scale * (yi - in.ya);
        const double daxn = tr_scale * (axi - in.axa);
        t[4] = dyn * dyn;
        t[5] = dyn * daxn;
      }
    }
  }
};

struct EpiStoreSq {  // out = s, term s^2 (power iteration)
  double* out;
  using In = NoIn;
  __device__ __forceinline__ In load(int) const { return {}; }
  __device__ __forceinline__ void apply(int r, double s, const In&, double (&t)[1]) const {
    out[r] = s;
    t[0] = s * s;
  }
};

// Power iteration in a team: out = s, term s^2, and the entry pushed to the
// peers that gather it (w_i to the owners of the columns in row i, z_j to the
// owners of the rows in column j).
template <bool RK>
struct EpiStoreSqPush {
  double* out;
  const Team* T;
  double* const* base;        // T->py / T->px: the peers' pools
  size_t off;                 // offset of out within the pools
  const unsigned char* need;  // T->yneed / T->xneed
  int lo;                     // row0 / col0
  using In = NoIn;
  __device__ __forceinline__ In load(int) const { return {}; }
  __device__ __forceinline__ void apply(int r, double s, const In&, double (&t)[1]) const {
    out[r] = s;
    t[0] = s * s;
    if constexpr (RK)
      if (T->nranks > 1) push_peers(T, base, off + r, s, __ldg(need + (r - lo)));
  }
};

// kModeKkt (teams): kkt_error_with_products at z with fresh products,
// src/pdhg_core.cpp:57-68.  Rows of A^T: [-(c + A^T y)]+^2 and c.x with x
// formed as in phase A; rows of A: (Ax - b)^2 and b.y.
struct SrcComb {  // x = x_src, or (1 - w) x_src + w anchor (the rounding phase A uses)
  const double* xs;
  const double* xa;
  double w;
  int mode;
  __device__ __forceinline__ double operator()(int j) const {
    return mode ? (1.0 - w) * ldca(xs + j) + w * ldca(xa + j) : ldca(xs + j);
  }
};
struct EpiKktA {
  SrcComb x;
  const double* c;
  struct In {
    double x, c;
  };
  __device__ __forceinline__ In load(int j) const { return In{x(j), __ldg(c + j)}; }
  __device__ __forceinline__ void apply(int, double aty, const In& in, double (&t)[2]) const {
    double rc = -(in.c + aty);
    rc = rc < 0.0 ? 0.0 : rc;
    t[0] = rc * rc;
    t[1] = in.c * in.x;
  }
};
struct EpiKktB {
  const double* b;
  const double* y;
  struct In {
    double b, y;
  };
  __device__ __forceinline__ In load(int i) const { return In{__ldg(b + i), ldcg(y + i)}; }
  __device__ __forceinline__ void apply(int, double ax, const In& in, double (&t)[2]) const {
    const double d = ax - in.b;
    t[0] = d * d;
    t[1] = in.b * in.y;
  }
};

struct EpiStore {
  double* out;
  using In = NoIn;
  __device__ __forceinline__ In load(int) const { return {}; }
  __device__ __forceinline__ void apply(int r, double s, const In&, double (&t)[1]) const {
    out[r] = s;
    t[0] = 0.0;
  }
};

// Column-blocked sweeps before the last: out = s on the first, out + s after
// (a row's sum is ((s_0 + s_1) + s_2) + ..., each block's part in ascending
// column order; the last sweep adds its own through EpiDual's PART input).
struct EpiAccum {
  double* out;
  int first;
  using In = NoIn;
  __device__ __forceinline__ In load(int) const { return {}; }
  __device__ __forceinline__ void apply(int r, double s, const In&, double (&t)[1]) const {
    out[r] = first ? s : ldcg(out + r) + s;
    t[0] = 0.0;
  }
};

struct EpiPosNeg {  // primal certificate: max(A^T u), max(-A^T u)
  using In = NoIn;
  __device__ __forceinline__ In load(int) const { return {}; }
  __device__ __forceinline__ void apply(int, double s, const In&, double (&t)[2]) const {
    t[0] = s;
    t[1] = -s;
  }
};

struct EpiAbs {  // dual certificate: max |A u|
  using In = NoIn;
  __device__ __forceinline__ In load(int) const { return {}; }
  __device__ __forceinline__ void apply(int, double s, const In&, double (&t)[1]) const { t[0] = fabs(s); }
};

// ---------------------------------------------------------------------------
// Grid barrier: one monotonic 64-bit arrival counter per launch (reset by
// the host before each launch), so a barrier is a single release atomic per
// CTA plus an acquire spin until count >= (barriers passed) * grid.  A 10 s
// watchdog turns a hang into HPLP_ETIMEOUT instead of a dead GPU.  The
// gpu-scope fence after the spin also invalidates this SM's L1
// (CCTL.IVALL), so L1-cached gathers never see stale lines.
// ---------------------------------------------------------------------------
__device__ bool grid_sync(GridBar* bar, unsigned long long& target) {
  __shared__ int s_ok;
  __syncthreads();
  target += gridDim.x;
  if (threadIdx.x == 0) {
    s_ok = 1;
    // release: this CTA's writes (ordered before by bar.sync) become visible
    // before the arrival (SASS: MEMBAR.ALL.GPU + REDG, no return)
    asm volatile("red.release.gpu.global.add.u64 [%0], %1;" ::"l"(&bar->count), "l"(1ull) : "memory");
    const unsigned long long t0 = global_ns();
    unsigned spins = 0;
    // poll, then acquire (SASS: LDG.STRONG.GPU + CCTL.IVALL): later reads,
    // L1-cached ones included, see every CTA's released writes
#if HX_BAR_RELAXED
    // relaxed polls (no L1 invalidation per poll), one acquire load at the end
    while (*reinterpret_cast<volatile unsigned long long*>(&bar->count) < target) {
#else
    while (ld_acquire_u64(&bar->count) < target) {
#endif
      if ((++spins & 255u) == 0u) {
        if (*reinterpret_cast<volatile unsigned*>(&bar->abort)) {
          s_ok = 0;
          break;
        }
        if (global_ns() - t0 > 10000000000ull) {
          atomicExch(&bar->abort, 1u);
          s_ok = 0;
          break;
        }
      }
    }
#if HX_BAR_RELAXED
    (void)ld_acquire_u64(&bar->count);
#endif
  }
  __syncthreads();
  return s_ok != 0;
}

__device__ __forceinline__ unsigned long long ld_acquire_sys_u64(const unsigned long long* p) {
  unsigned long long v;
  asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}

// Team barrier (row-partitioned ranks), two levels:
//  1. every CTA of this rank arrives on the rank's local counter with a
//     system-scope release, which orders its P2P stores into peers' memory
//     (x+ / y slices, partial records) before the arrival;
//  2. the rank's leader (CTA 0) waits for all local CTAs, then bumps the
//     monotonic `arrive` word of every rank (system-scope release, one P2P
//     atomic per peer), waits until its own word shows all ranks' leaders for
//     this epoch, and releases its CTAs through `go`.
// Causality is transitive along peer CTA -> peer leader -> this leader ->
// this CTA, so after the barrier every slice a peer pushed is visible here,
// and the acquire spins invalidate L1 as in grid_sync.  `repoch` (cross-rank
// barriers passed) continues across launches and is identical on all ranks.
// Each spin has the same 10 s watchdog; a rank whose peer died stops with
// HPLP_ETIMEOUT instead of hanging the GPU.
//
// With `reduce` >= 0 (the end-of-iteration barrier; value = iteration
// parity) the leader's warp, once every local CTA has arrived, also sums
// the rank's own phase A/B records (slot regions kRegA/kRegB + parity,
// local records only, fixed order) and stores the 7 totals into every
// rank's RankBar::rrec[parity][rank] before its arrival, which releases
// them with the rest.
__device__ bool team_sync(GridBar* bar, const Team& T, const Geo& g, unsigned long long& target,
                          unsigned long long& repoch, const double* slots = nullptr, int reduce = -1,
                          bool box = false) {
  __shared__ int s_ok;
  __syncthreads();
  target += g.nctas;
  repoch += 1;
  if (reduce >= 0 && g.cta == 0) {
    // whole leader CTA: thread (k, q) sums quantity q over local records
    // k, k + 64, ...; warp q folds the 64 partials (fixed order)
    __shared__ double part[64][8];
    if (threadIdx.x == 0) {
      s_ok = 1;
      if (T.sys) asm volatile("red.release.sys.global.add.u64 [%0], %1;" ::"l"(&bar->count), "l"(1ull) : "memory");
      else asm volatile("red.release.gpu.global.add.u64 [%0], %1;" ::"l"(&bar->count), "l"(1ull) : "memory");
      const unsigned long long t0 = global_ns();
      unsigned spins = 0;
      while ((T.sys ? ld_acquire_sys_u64(&bar->count) : ld_acquire_u64(&bar->count)) < target) {
        if ((++spins & 255u) != 0u) continue;
        if (*reinterpret_cast<volatile unsigned*>(&bar->abort) || global_ns() - t0 > 10000000000ull) {
          atomicExch(&bar->abort, 1u);
          s_ok = 0;
          break;
        }
      }
    }
    __syncthreads();
    if (s_ok) {
      // q 0..2: phase A, 3..6: phase B, 7: the box term (phase A's fourth)
      static_assert(kThreads == 512, "the leader reduction below fills part[64][8] with 512 threads");
      const int q = threadIdx.x & 7, k = threadIdx.x >> 3;  // 512 threads: k < 64
      {
        const size_t stride = region_stride(g.nrec);
        const double* rg = slots + static_cast<size_t>(q < 3 || q == 7 ? kRegA + reduce : kRegB + reduce) * stride +
                           (q < 3 ? q : q == 7 ? 3 : q - 3);
        const size_t r0 = static_cast<size_t>(T.rank) * g.nctas;
        double v = 0.0;
        if (q < 7 || box)
          for (int c = k; c < g.nctas; c += 64) v += ldcg(rg + (r0 + c) * kMaxQ);
        part[k][q] = v;
      }
      __syncthreads();
      const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
      if (warp < 8) {
        const double v = warp_sum(part[lane][warp] + part[lane + 32][warp]);
        for (int d = lane; d < T.nranks * kRankRecReplicas; d += 32)
          T.pb[d % T.nranks]->rrec[reduce][d / T.nranks][T.rank][warp] = v;
        if (T.sys) asm volatile("fence.acq_rel.sys;" ::: "memory");
        else __threadfence();
      }
    }
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    const bool counted = reduce >= 0 && g.cta == 0;  // the leader arrived above
    if (!counted) s_ok = 1;
    // peers on other GPUs see this CTA's P2P stores only through a
    // system-scope release; ranks sharing one device need gpu scope only
    if (!counted) {
      if (T.sys) asm volatile("red.release.sys.global.add.u64 [%0], %1;" ::"l"(&bar->count), "l"(1ull) : "memory");
      else asm volatile("red.release.gpu.global.add.u64 [%0], %1;" ::"l"(&bar->count), "l"(1ull) : "memory");
    }
    const unsigned long long t0 = global_ns();
    unsigned spins = 0;
    auto alive = [&]() -> bool {
      if ((++spins & 255u) != 0u) return true;
      if (*reinterpret_cast<volatile unsigned*>(&bar->abort)) return false;
      if (global_ns() - t0 > 10000000000ull) {
        atomicExch(&bar->abort, 1u);
        return false;
      }
      return true;
    };
    if (g.cta == 0) {
      if (!counted)
        while ((T.sys ? ld_acquire_sys_u64(&bar->count) : ld_acquire_u64(&bar->count)) < target)
          if (!alive()) {
            s_ok = 0;
            break;
          }
      if (s_ok) {
        for (int r = 0; r < T.nranks; ++r) {
          if (T.sys)
            asm volatile("red.release.sys.global.add.u64 [%0], %1;" ::"l"(&T.pb[r]->arrive), "l"(1ull) : "memory");
          else
            asm volatile("red.release.gpu.global.add.u64 [%0], %1;" ::"l"(&T.pb[r]->arrive), "l"(1ull) : "memory");
        }
        const unsigned long long want = repoch * static_cast<unsigned long long>(T.nranks);
        while ((T.sys ? ld_acquire_sys_u64(&T.pb[T.rank]->arrive) : ld_acquire_u64(&T.pb[T.rank]->arrive)) < want)
          if (!alive()) {
            s_ok = 0;
            break;
          }
      }
      if (s_ok) asm volatile("st.release.gpu.global.u64 [%0], %1;" ::"l"(&bar->go), "l"(repoch) : "memory");
    } else {
      while (ld_acquire_u64(&bar->go) < repoch)
        if (!alive()) {
          s_ok = 0;
          break;
        }
    }
  }
  __syncthreads();
  return s_ok != 0;
}

// ---------------------------------------------------------------------------
// Controller logic (thread 0 of every CTA, on its shared replica).  Only CTA 0
// (writer) touches global memory (epoch ring).
// ---------------------------------------------------------------------------
__device__ int pick_free(int pool, int e0, int e1, int e2, int e3, int e4 = -1, int e5 = -1) {
  for (int i = 0; i < pool; ++i)
    if (i != e0 && i != e1 && i != e2 && i != e3 && i != e4 && i != e5) return i;
  return -1;
}

// should_restart, src/solver.cpp:162-174.
__device__ bool should_restart(const Ctl& C, long long n, long long k, double now, double start) {
  switch (C.restart_kind) {
    case HPLP_RESTART_FIXED:
      return k >= C.k_star;
    case HPLP_RESTART_ADAPTIVE:
      if (n == 0) return k > C.tau0;
      return now <= C.beta * start;
    default:
      return false;
  }
}

__device__ void set_final_limit(Ctl& C, int status) {
  C.status = status;
  if (C.best_kkt < INFINITY) {  // isfinite(best_kkt): it only ever decreases from +inf
    C.final_x = C.x_best;
    C.final_y = C.y_best;
    C.final_avg = C.avg_best;  // averaged baselines: the best is an average slot
    for (int q = 0; q < 4; ++q) C.final_kkt[q] = C.best_err[q];
  } else {
    C.final_x = -1;  // host evaluates kkt_error(z) with fresh products
    C.final_y = -1;
    C.final_avg = -1;
  }
  C.r.stop = 1;
}

// Ring slot of iteration `it` (-1: not traced or no ring).
__host__ __device__ inline int ring_slot(const Ctl& C, long long it) {
  return C.ring_cap > 0 && C.trace_period > 0 && it % C.trace_period == 0
             ? static_cast<int>((it / C.trace_period) % C.ring_cap)
             : -1;
}

// Restart decision + Halpern bookkeeping + next roles + limits
// (src/solver.cpp:319-341 and the loop-top checks :242-254).
__device__ void finish_iteration(Ctl& C, hplp_epoch_t* epochs, bool writer, double res, bool time_up) {
  // C.w_k2 = 1/(k+2), C.w_k3 = 1/(k+3) were computed in parallel (warp 0)
  Roles& R = C.r;
  bool restart = should_restart(C, C.n, C.k, res, C.res_epoch_start);
  if (!restart && C.restart_kind == HPLP_RESTART_ADAPTIVE && C.stall_cap > 0 && C.k >= C.stall_cap)
    restart = true;
  if (restart) {
    if (writer && C.n_epochs > 0) epochs[(C.n_epochs - 1) % kEpochCap].restart_length = C.k;
    R.x_src = R.xp_out;
    R.x_mode = 0;
    R.x_anchor = R.xp_out;
    R.y_cur = R.yp_out;
    R.y_anchor = R.yp_out;
    R.ax_cur = R.axp_out;
    R.ax_anchor = R.axp_out;
    R.w_x = 0.0;
    R.y_unpushed = 1;
    C.n += 1;
    C.k = 0;
  } else {
    const double w = C.w_k2;  // 1.0 / (k + 2)
    R.x_src = R.xp_out;
    R.x_mode = 1;
    R.w_x = w;
    R.y_cur = R.yc_out;
    R.ax_cur = R.axc_out;
    R.y_unpushed = 0;
    C.k += 1;
  }
  R.check = 0;
  C.it += 1;
  R.tr_slot = ring_slot(C, C.it);
  if (R.tr_slot >= 0) R.tr_scale = C.k >= 1 ? 2.0 / static_cast<double>(C.k) : 0.0;
  // x outputs avoid this iteration's T(z) and the best iterate before and
  // after its update too, so that without a restart the picks equal the
  // speculative ones (make_spec), which cannot know the update yet
  R.zx_out = pick_free(kXPool, R.x_src, R.x_anchor, C.x_best, C.last_zx, C.x_best_prev);
  R.xp_out = pick_free(kXPool, R.x_src, R.x_anchor, C.x_best, C.last_zx, C.x_best_prev, R.zx_out);
  R.yp_out = pick_free(kYPool, R.y_cur, R.y_anchor, C.y_best, -1);
  R.yc_out = pick_free(kYPool, R.y_cur, R.y_anchor, C.y_best, R.yp_out);
  R.axp_out = pick_free(kAxPool, R.ax_cur, R.ax_anchor, -1, -1);
  R.axc_out = pick_free(kAxPool, R.ax_cur, R.ax_anchor, R.axp_out, -1);
  R.w_next = restart ? 0.5 : C.w_k3;  // 1.0 / (k_new + 2)
  if (C.it >= C.iteration_limit) {
    set_final_limit(C, HPLP_STATUS_ITERATION_LIMIT);
  } else if (time_up) {
    set_final_limit(C, HPLP_STATUS_TIME_LIMIT);
  }
  if (C.trace_period > 0 && C.last_it % C.trace_period == 0) {
    // no ring: the host takes each record between launches; a ring pauses
    // only when one more record could overwrite an undrained one (the next
    // traced phase A writes its slot speculatively)
    if (C.ring_cap == 0 || C.ring_total - C.ring_drained >= C.ring_cap - 1) {
      C.paused = 1;
      R.stop = 1;
    }
  }
  if (C.it >= C.batch_end) R.stop = 1;
}

// After phases A+B: KKT, residual, epochs, best, termination, scan or finish.
// pre[0..2]: KKT components (kkt_error_with_products, src/pdhg_core.cpp:57-68),
// pre[3] = dx2/eta, pre[4] = dy2/eta, computed one per lane of warp 0.
// ring / trt: the trace ring's records and this iteration's trace totals
// (|N|, |B1|, |B2|, and the normalized candidate's ||dx||^2, ||dy||^2,
// dy.d(Ax)) when the iteration is traced into a ring, else null.
__device__ void main_logic(Ctl& C, const double* tot, const double* pre, hplp_epoch_t* epochs, bool writer,
                           bool time_up, TraceRec* ring = nullptr, const double* trt = nullptr, bool check_due = false) {
  Roles& R = C.r;
  const double dx2 = tot[2], dy2 = tot[5], dyax = tot[6];
  double kkt[4];
  kkt[0] = pre[0];
  kkt[1] = pre[1];
  kkt[2] = pre[2];
  double mx = kkt[0];
  if (mx < kkt[1]) mx = kkt[1];
  if (mx < kkt[2]) mx = kkt[2];
  kkt[3] = mx;
  // canonical_norm_with_product, src/pdhg_core.cpp:37-51
  const double eta = R.eta;
  const double q = pre[3] - 2.0 * dyax + pre[4];
  double res;
  if (q < 0.0) {
    const double scale = (dx2 + dy2) / eta;
    if (q < -1e-9 * scale) {
      C.error = HPLP_EDOMAIN;
      R.stop = 1;
      return;
    }
    res = 0.0;
  } else {
    res = sqrt(q);
  }
  C.spmv += 2;
  if (C.k == 0) {  // src/solver.cpp:261-264
    C.res_epoch_start = res;
    if (writer) {
      hplp_epoch_t& e = epochs[C.n_epochs % kEpochCap];
      e.epoch = C.n;
      e.restart_length = 0;
      e.residual_at_start = res;
      e.kkt_at_start = {kkt[0], kkt[1], kkt[2], kkt[3]};
    }
    C.n_epochs += 1;
  }
  C.x_best_prev = C.x_best;
  if (kkt[3] < C.best_kkt) {  // :265-269
    C.best_kkt = kkt[3];
    for (int i = 0; i < 4; ++i) C.best_err[i] = kkt[i];
    C.x_best = R.zx_out;
    C.y_best = R.y_cur;
  }
  C.last_it = C.it;
  C.last_n = C.n;
  C.last_k = C.k;
  C.last_res = res;
  C.last_res_diff = res;  // ||T(z) - z|| == ||z - T(z)||
  for (int i = 0; i < 4; ++i) C.last_kkt[i] = kkt[i];
  C.last_zx = R.zx_out;
  C.last_xp = R.xp_out;
  C.last_y = R.y_cur;
  C.last_yp = R.yp_out;
  C.last_xa = R.x_anchor;
  C.last_ya = R.y_anchor;
  C.last_ax = R.ax_cur;
  C.last_axp = R.axp_out;
  C.last_axa = R.ax_anchor;
  if (ring && trt) {  // TraceRecord of this iteration (src/solver.cpp:271-290)
    const int slot = ring_slot(C, C.it);
    if (writer && slot >= 0) {
      TraceRec& t = ring[slot];
      t.it = C.it, t.n = C.n, t.k = C.k;
      t.res = res;
      for (int i = 0; i < 4; ++i) t.kkt[i] = kkt[i];
      // canonical_norm_with_product of the normalized candidate (2/k)(z -
      // anchor), src/solver.cpp:283-286; NaN at k = 0 or a clearly negative form
      double cn = __longlong_as_double(0x7ff8000000000000ll);
      if (C.k >= 1) {
        const double qn = trt[3] / eta - 2.0 * trt[5] + trt[4] / eta;
        if (qn >= 0.0) cn = sqrt(qn);
        else if (qn >= -1e-9 * ((trt[3] + trt[4]) / eta)) cn = 0.0;
      }
      t.cand_norm = cn;
      for (int i = 0; i < 3; ++i) t.cnt[i] = static_cast<long long>(trt[i]);
    }
    C.ring_total += 1;
  }
  if (kkt[3] <= C.tol) {  // :292-295, returns z
    C.status = HPLP_STATUS_OPTIMAL;
    C.final_x = R.zx_out;
    C.final_y = R.y_cur;
    for (int i = 0; i < 4; ++i) C.final_kkt[i] = kkt[i];
    R.stop = 1;
    if (C.trace_period > 0 && C.last_it % C.trace_period == 0) C.paused = 1;
    return;
  }
  // check_due: C.it % C.check_period == 0, a 64-bit remainder warp 0 forms
  // on another lane beside the KKT divides
  if (C.check_period > 0 && C.it > 0 && (check_due || C.k == 0)) {  // :297-298
    R.check = 1;
    R.cand_scale = C.k >= 1 ? 2.0 / static_cast<double>(C.k) : 0.0;
    return;
  }
  finish_iteration(C, epochs, writer, res, time_up);
}

// validate_primal_infeasibility, src/infeasibility.cpp:41-67, from reductions.
__device__ bool eval_primal(const Ctl& C, int c, hplp_cert_meta_t& rep) {
  const double tol = C.cert_tol;
  double inf_u = C.cinf[c];
  if (inf_u < 0.0) inf_u = 0.0;
  const double threshold = tol * dmax(1.0, inf_u * C.sigma_used);
  double best_res = INFINITY;
  bool valid = false;
  for (int si = 0; si < 2; ++si) {
    const double s = si == 0 ? 1.0 : -1.0;
    const double residual = dmax(0.0, si == 0 ? C.cmax_at[c] : C.cmax_negat[c]);
    const double margin = s * C.cdot[c];
    const bool ok = residual <= threshold && margin > 0.0 && margin >= tol * C.b_norm;
    if (ok || (!valid && residual < best_res)) {
      best_res = residual;
      rep.residual = residual;
      rep.margin = margin;
      rep.orientation = si == 0 ? HPLP_ORIENT_AS_IS : HPLP_ORIENT_NEGATED;
    }
    if (ok) {
      valid = true;
      break;
    }
  }
  return valid;
}

// validate_dual_infeasibility, src/infeasibility.cpp:76-106, from reductions.
__device__ bool eval_dual(const Ctl& C, int c, hplp_cert_meta_t& rep) {
  const double tol = C.cert_tol;
  double inf_u = C.cinf[c];
  if (inf_u < 0.0) inf_u = 0.0;
  const double threshold = tol * dmax(1.0, inf_u * C.sigma_used);
  const double nonneg_threshold = tol * dmax(1.0, inf_u);
  const double margin_threshold = -tol * dmax(1.0, C.c_norm);
  const double ray = dmax(0.0, C.cmax_abs_au[c]);
  double best_res = INFINITY;
  bool valid = false;
  for (int si = 0; si < 2; ++si) {
    const double s = si == 0 ? 1.0 : -1.0;
    const double sign = dmax(0.0, si == 0 ? C.cmax_negu[c] : C.cmax_u[c]);
    const double residual = dmax(ray, sign);
    const double margin = s * C.cdot[c];
    const bool ok = ray <= threshold && sign <= nonneg_threshold && margin <= margin_threshold;
    if (ok || (!valid && residual < best_res)) {
      best_res = residual;
      rep.residual = residual;
      rep.margin = margin;
      rep.orientation = si == 0 ? HPLP_ORIENT_AS_IS : HPLP_ORIENT_NEGATED;
    }
    if (ok) {
      valid = true;
      break;
    }
  }
  return valid;
}

// Whether candidate c can still validate once its product is known: the
// parts of eval_primal / eval_dual that do not need the SpMV, operand for
// operand (a y-candidate's margin test; an x-candidate's sign and margin
// tests).  False means the evaluation fails whatever the product is.
__device__ bool cert_may_pass(const Ctl& C, int c) {
  const double tol = C.cert_tol;
  if (c & 1) {  // y-candidate: primal certificate, margin s (b . u) > 0 and >= tol ||b||
    for (int si = 0; si < 2; ++si) {
      const double margin = (si == 0 ? 1.0 : -1.0) * C.cdot[c];
      if (margin > 0.0 && margin >= tol * C.b_norm) return true;
    }
    return false;
  }
  double inf_u = C.cinf[c];  // x-candidate: dual certificate
  if (inf_u < 0.0) inf_u = 0.0;
  const double nonneg_threshold = tol * dmax(1.0, inf_u);
  const double margin_threshold = -tol * dmax(1.0, C.c_norm);
  for (int si = 0; si < 2; ++si) {
    const double sign = dmax(0.0, si == 0 ? C.cmax_negu[c] : C.cmax_u[c]);
    const double margin = (si == 0 ? 1.0 : -1.0) * C.cdot[c];
    if (sign <= nonneg_threshold && margin <= margin_threshold) return true;
  }
  return false;
}

__device__ void finish_iteration_baseline(Ctl& C, hplp_epoch_t* epochs, bool writer, double res, bool time_up);

// CertificateScan::check semantics, src/solver.cpp:108-135 (+ :300-317).
// Candidates: 0 v_x diff, 1 v_y diff, 2 v_x normalized, 3 v_y normalized.
__device__ void scan_logic(Ctl& C, hplp_epoch_t* epochs, bool writer, bool time_up) {
  Roles& R = C.r;
  hplp_cert_meta_t prim{}, dual{};
  bool have_p = false, have_d = false;
  for (int src = 0; src < 2; ++src) {  // difference first, then normalized
    if (src == 1 && (C.last_k < 1 || C.scheme != HPLP_SCHEME_RHPDHG)) break;  // baselines: difference only
    const int cy = src == 0 ? 1 : 3, cx = src == 0 ? 0 : 2;
    const int source = src == 0 ? HPLP_SOURCE_ITERATE_DIFFERENCE : HPLP_SOURCE_NORMALIZED_ITERATE;
    if (!have_p && R.cn2[cy] > 0.0) {
      C.spmv += 1;
      hplp_cert_meta_t rep{};
      if (C.cfinite[cy] && eval_primal(C, cy, rep)) {
        have_p = true;
        prim = rep;
        prim.present = 1;
        prim.source = source;
        prim.at_iteration = C.last_it;
        C.cert_cand[0] = cy;
      }
    }
    if (!have_d && R.cn2[cx] > 0.0) {
      C.spmv += 1;
      hplp_cert_meta_t rep{};
      if (C.cfinite[cx] && eval_dual(C, cx, rep)) {
        have_d = true;
        dual = rep;
        dual.present = 1;
        dual.source = source;
        dual.at_iteration = C.last_it;
        C.cert_cand[1] = cx;
      }
    }
  }
  if (have_p || have_d) {
    C.cert[0] = prim;
    C.cert[1] = dual;
    C.status = have_p && have_d ? HPLP_STATUS_PRIMAL_DUAL_INFEASIBLE
               : have_p         ? HPLP_STATUS_PRIMAL_INFEASIBLE
                                : HPLP_STATUS_DUAL_INFEASIBLE;
    C.final_x = C.last_zx;
    C.final_y = C.last_y;
    C.final_avg = C.last_cand_avg;  // baselines return the candidate (the average when averaged)
    for (int i = 0; i < 4; ++i) C.final_kkt[i] = C.last_kkt[i];
    R.stop = 1;
    if (C.trace_period > 0 && C.last_it % C.trace_period == 0) C.paused = 1;
    return;
  }
  if (C.scheme != HPLP_SCHEME_RHPDHG) finish_iteration_baseline(C, epochs, writer, C.last_res, time_up);
  else finish_iteration(C, epochs, writer, C.last_res, time_up);
}

// Roles of phase A for iteration it+1 assuming no restart and no stop
// (finish_iteration's no-restart branch), known before the controller runs.
// The x outputs avoid T(z) of iteration it and the current best, the two
// candidates for the best after the update, so they equal finish_iteration's
// picks whenever no restart happens.
__device__ void make_spec(const Ctl& C, Roles& S) {
  const Roles& R = C.r;
  S = R;
  S.x_src = R.xp_out;
  S.x_mode = 1;
  S.w_x = 1.0 / static_cast<double>(C.k + 2);
  S.y_cur = R.yc_out;
  S.zx_out = pick_free(kXPool, S.x_src, S.x_anchor, C.x_best, R.zx_out);
  S.tr_slot = ring_slot(C, C.it + 1);
  S.tr_scale = 2.0 / static_cast<double>(C.k + 1);  // k + 1 >= 1 without a restart
  S.xp_out = pick_free(kXPool, S.x_src, S.x_anchor, C.x_best, R.zx_out, S.zx_out);
}

// Did the speculative phase A compute exactly what phase A with roles R would?
__device__ __forceinline__ bool same_phase_a(const Roles& R, const Roles& S) {
  return R.x_mode == S.x_mode && R.x_src == S.x_src && R.x_anchor == S.x_anchor && R.zx_out == S.zx_out &&
         R.xp_out == S.xp_out && R.y_cur == S.y_cur && R.w_x == S.w_x && R.eta == S.eta && R.tr_slot == S.tr_slot &&
         (R.tr_slot < 0 || R.tr_scale == S.tr_scale);
}

__device__ void ctl_load(const Ctl* g, Ctl& s) {
  const unsigned long long* src = reinterpret_cast<const unsigned long long*>(g);
  unsigned long long* dst = reinterpret_cast<unsigned long long*>(&s);
  for (int i = threadIdx.x; i < static_cast<int>(sizeof(Ctl) / 8); i += blockDim.x) dst[i] = __ldcg(src + i);
  __syncthreads();
}

__device__ void ctl_store(const Ctl& s, Ctl* g) {
  __syncthreads();
  const unsigned long long* src = reinterpret_cast<const unsigned long long*>(&s);
  unsigned long long* dst = reinterpret_cast<unsigned long long*>(g);
  for (int i = threadIdx.x; i < static_cast<int>(sizeof(Ctl) / 8); i += blockDim.x) dst[i] = src[i];
}

// ---------------------------------------------------------------------------
// Phases.  Each is a separate (noinline) function so the register allocator
// sees one SpMV instantiation at a time; KParams lives in global memory.
// ---------------------------------------------------------------------------
__device__ __forceinline__ double* region_ptr(const KParams* P, int r, int nrec) {
  return P->slots + static_cast<size_t>(r) * region_stride(nrec);
}

__device__ __forceinline__ int gwarp_id(const Geo& g) { return g.cta * kWarps + (threadIdx.x >> 5); }

// phase A: A^T y, primal step (+ Halpern formation of x), primal partials
template <bool RK, bool BOX, int LM = 2, int EX = 2, bool TR = false>
__device__ HX_PHASE_INLINE void phase_primal_t(const KParams* P, const Roles* R, int par, WarpStage* stage,
                                               unsigned long long seq, const SpmvHead& head, const Geo& g) {
  constexpr int NQ = EpiPrimal<RK, BOX, 0, TR>::NQ;
  const int n = P->n, m = P->m;
  double acc[NQ];
  acc_init<NQ, 0>(acc);
  const bool traced = TR && R->tr_slot >= 0;
  EpiPrimal<RK, BOX, LM == 1 ? HX_EPI_EF : 0, TR> e{xsrc_ptr(P, R),
                       P->xpool + static_cast<size_t>(R->x_anchor) * n,
                       P->c,
                       P->xpool + static_cast<size_t>(R->zx_out) * n,
                       P->xpool + static_cast<size_t>(R->xp_out) * n,
                       R->w_x,
                       R->eta,
                       R->x_mode,
                       &P->T,
                       static_cast<size_t>(R->xp_out) * n,
                       P->ub,
                       traced ? P->ring_x + static_cast<size_t>(R->tr_slot) * n : nullptr,
                       traced ? P->ring_cls + static_cast<size_t>(R->tr_slot) * n : nullptr,
                       P->r_tol,
                       P->tol_active,
                       R->tr_scale};
  const Sched S = P->AT;
#ifdef HX_WPROF
  const unsigned long long w0 = clock64();
#endif
  spmv_rows<NQ, 0, LM, EX>(S, par, SrcVecT<LM == 1 && HX_GATHER_LAST>{ycur_ptr(P, R)}, e, acc, gwarp_id(g),
                       threadIdx.x & 31, stage, seq, head);
#ifdef HX_WPROF
  if constexpr (!RK)
    if (P->prof && (threadIdx.x & 31) == 0) P->prof[gridDim.x * 16 + gwarp_id(g)] += clock64() - w0;
#endif
  fold_long<NQ, 0>(S, par, seq, acc, g.cta, &P->bar->abort);
  block_to_slots<NQ, 0, RK>(acc, P, kRegA + par, g);
}

// phase B: A x+, dual step, speculative Halpern combos, dual partials
template <bool RK, int LM = 2, bool CB = false, int EX = 2, bool TR = false>
__device__ HX_PHASE_INLINE bool phase_dual(const KParams* P, const Roles* R, int par, WarpStage* stage,
                                           unsigned long long seq, const SpmvHead& head, const Geo& g,
                                           unsigned long long* target = nullptr) {
  const int n = P->n, m = P->m;
  constexpr int QD = TR ? 6 : 4;
  double acc[QD];
  acc_init<QD, 0>(acc);
  const bool traced = TR && R->tr_slot >= 0;
  EpiDual<RK, LM == 1 ? HX_EPI_EF : 0, CB, TR> e{ycur_ptr(P, R),
            axcur_ptr(P, R),
            P->b,
            P->ypool + static_cast<size_t>(R->y_anchor) * m,
            P->axpool + static_cast<size_t>(R->ax_anchor) * m,
            P->ypool + static_cast<size_t>(R->yp_out) * m,
            P->axpool + static_cast<size_t>(R->axp_out) * m,
            P->ypool + static_cast<size_t>(R->yc_out) * m,
            P->axpool + static_cast<size_t>(R->axc_out) * m,
            R->eta,
            R->w_next,
            &P->T,
            static_cast<size_t>(R->yp_out) * m,
            static_cast<size_t>(R->yc_out) * m,
            P->bpart,
            traced ? P->ring_y + static_cast<size_t>(R->tr_slot) * m : nullptr,
            R->tr_scale};
  const double* xsrc = P->xpool + static_cast<size_t>(R->xp_out) * n;
  SpmvHead h1;
  if constexpr (CB) {
    // sweeps 0 .. ncb - 2: the leading column blocks' row sums carried in
    // bpart, a grid barrier after each; then the last block with the full
    // epilogue
    double a0[1] = {0.0};
    h1 = head;
    for (int k = 0; k + 1 < P->ncb; ++k) {
      const Sched Sk = P->cbs[k];
      EpiAccum st0{P->bpart, k == 0};
      spmv_rows<1, 0, LM, EX>(Sk, par, SrcVecT<LM == 1 && HX_GATHER_LAST>{xsrc}, st0, a0, gwarp_id(g),
                              threadIdx.x & 31, stage, seq, h1);
      const Sched Sn = P->cbs[k + 1];
      spmv_head<LM>(Sn, gwarp_id(g), threadIdx.x & 31, h1);
      // abort / watchdog: leave before the next sweep (its long rows would
      // wait on pieces that never come)
      if (!grid_sync(P->bar, *target)) return false;
    }
  }
  const Sched S = CB ? P->cbs[P->ncb - 1] : P->A;
#ifdef HX_WPROF
  const unsigned long long w0 = clock64();
#endif
  spmv_rows<QD, 0, LM, EX>(S, par, SrcVecT<LM == 1 && HX_GATHER_LAST>{xsrc}, e, acc, gwarp_id(g), threadIdx.x & 31, stage,
                      seq, CB ? h1 : head);
#ifdef HX_WPROF
  if constexpr (!RK)
    if (P->prof && (threadIdx.x & 31) == 0) P->prof[gridDim.x * (16 + kWarps) + gwarp_id(g)] += clock64() - w0;
#endif
  fold_long<QD, 0>(S, par, seq, acc, g.cta, &P->bar->abort);
  block_to_slots<QD, 0, RK>(acc, P, kRegB + par, g);
  return true;
}

// Totals of phases A+B -> t[0..6], computed by warp 0 alone (the other warps
// are in the speculative phase A by then).  Lane l reads record l / 2 + 16 k
// of phase A's (even lanes) or phase B's (odd lanes) region as one 256-bit
// load of quantities 0..3: all 148 records of a single GPU in one round of
// 10 independent loads per lane (one L2 round trip; the loads queue behind
// the speculative phase A's gathers, so each extra round trip costs ~0.7 us
// -- configs[2]: lane-per-record scalar loads 3.7 us, this ~1.5).  Each lane
// sums its records in order, then a xor butterfly over the 16 lanes of a
// region finishes -- a fixed order, so every CTA holds bit-identical totals.
// t[0..2]: phase A partials, t[3..6]: phase B, t[7]: the box form's bound
// term of the dual objective (phase A's fourth partial; 0 in standard form)
constexpr int kTotBatch = 10;  // records per lane per round: 16 * 10 = 160 >= 148
template <bool BOX>
__device__ __forceinline__ void warp_totals_main(const KParams* P, int par, double (&t)[8], const Geo& g) {
  const int lane = threadIdx.x & 31, G = g.nrec;
  const size_t rep = static_cast<size_t>(g.cta % kReplicas) * G * kMaxQ;
  const double* base = region_ptr(P, (lane & 1) ? kRegB + par : kRegA + par, G) + rep;
  double s[4] = {0.0, 0.0, 0.0, 0.0};
  for (int c0 = lane >> 1; c0 < G; c0 += 16 * kTotBatch) {
    double v[kTotBatch][4];
#pragma unroll
    for (int k = 0; k < kTotBatch; ++k) {
      const int c = c0 + 16 * k;
      if (c < G) {
        asm volatile("ld.global.cg.v4.f64 {%0, %1, %2, %3}, [%4];"
                     : "=d"(v[k][0]), "=d"(v[k][1]), "=d"(v[k][2]), "=d"(v[k][3])
                     : "l"(base + static_cast<size_t>(c) * kMaxQ));
      } else {
        v[k][0] = v[k][1] = v[k][2] = v[k][3] = 0.0;
      }
    }
#pragma unroll
    for (int k = 0; k < kTotBatch; ++k)
#pragma unroll
      for (int q = 0; q < 4; ++q) s[q] += v[k][q];
  }
#pragma unroll
  for (int m = 2; m < 32; m *= 2)
#pragma unroll
    for (int q = 0; q < 4; ++q) s[q] += __shfl_xor_sync(0xffffffffu, s[q], m);
  t[0] = __shfl_sync(0xffffffffu, s[0], 0);
  t[1] = __shfl_sync(0xffffffffu, s[1], 0);
  t[2] = __shfl_sync(0xffffffffu, s[2], 0);
  t[7] = BOX ? __shfl_sync(0xffffffffu, s[3], 0) : 0.0;
#pragma unroll
  for (int q = 0; q < 4; ++q) t[3 + q] = __shfl_sync(0xffffffffu, s[q], 1);
}

// Trace totals of a traced iteration (every rank's records, fixed order).
__device__ __forceinline__ void warp_totals_trace(const KParams* P, int par, double (&t)[6], const Geo& g) {
  const int lane = threadIdx.x & 31, G = g.nrec;
  const size_t rep = static_cast<size_t>(g.cta % kReplicas) * G * kMaxQ;
  const double* ra = region_ptr(P, kRegA + par, G) + rep;
  const double* rb = region_ptr(P, kRegB + par, G) + rep;
  for (int c = lane; c < G; c += 32) {
    const double* a = ra + static_cast<size_t>(c) * kMaxQ;
    const double* b = rb + static_cast<size_t>(c) * kMaxQ;
#pragma unroll
    for (int q = 0; q < 4; ++q) t[q] += ldcg(a + 3 + q);
    t[4] += ldcg(b + 4);
    t[5] += ldcg(b + 5);
  }
#pragma unroll
  for (int q = 0; q < 6; ++q) t[q] = warp_sum(t[q]);
}

// Team totals: the nranks rank records of this parity, summed in rank order
// (every lane, identical on every rank).
__device__ __forceinline__ void warp_totals_ranks(const KParams* P, int par, double (&t)[8], int cta) {
  const double (*rr)[8] = P->T.pb[P->T.rank]->rrec[par][cta % kRankRecReplicas];
#pragma unroll
  for (int q = 0; q < 8; ++q) t[q] = ldcg(&rr[0][q]);
  for (int r = 1; r < P->T.nranks; ++r)
#pragma unroll
    for (int q = 0; q < 8; ++q) t[q] += ldcg(&rr[r][q]);
}

// power iteration halves: w = A x (x = x0 or z / zn), z = A^T w
// (a team: every rank its own rows of w = A x and columns of z = A^T w,
// pushed to the peers that gather them; the norms reduced over all ranks'
// records -- identical on every rank)
template <int LM = 0, int EX = 2, bool RK = false>
__device__ HX_PHASE_INLINE void power_a(const KParams* P, const Roles* R, WarpStage* stage, unsigned long long seq,
                                        const Geo& g) {
  double acc[1];
  acc_init<1, 0>(acc);
  EpiStoreSqPush<RK> e{P->ypool, &P->T, P->T.py, 0, P->T.yneed, P->T.row0};
  const Sched S = P->A;
  if (R->pw_mode == 0) spmv_rows<1, 0, LM, EX>(S, 0, SrcVec{P->xpool}, e, acc, gwarp_id(g), threadIdx.x & 31, stage, seq);
  else
    spmv_rows<1, 0, LM, EX>(S, 0, SrcDiv{P->xpool + P->n, R->pw_zn}, e, acc, gwarp_id(g), threadIdx.x & 31, stage, seq);
  fold_long<1, 0>(S, 0, seq, acc, g.cta, &P->bar->abort);
  block_to_slots<1, 0, RK>(acc, P, kRegPA, g);
}

template <int LM = 0, int EX = 2, bool RK = false>
__device__ HX_PHASE_INLINE void power_b(const KParams* P, WarpStage* stage, unsigned long long seq, const Geo& g) {
  double acc[1];
  acc_init<1, 0>(acc);
  EpiStoreSqPush<RK> e{P->xpool + P->n, &P->T, P->T.px, static_cast<size_t>(P->n), P->T.xneed, P->T.col0};
  const Sched S = P->AT;
  spmv_rows<1, 0, LM, EX>(S, 0, SrcVec{P->ypool}, e, acc, gwarp_id(g), threadIdx.x & 31, stage, seq);
  fold_long<1, 0>(S, 0, seq, acc, g.cta, &P->bar->abort);
  block_to_slots<1, 0, RK>(acc, P, kRegPB, g);
}

// kModeKkt (teams): this rank's columns (A^T y) and rows (A x), partials into
// region C1 (4 quantities), every rank's records on every rank.
template <int LM, int EX>
__device__ HX_PHASE_INLINE void team_kkt(const KParams* P, const Roles* R, WarpStage* stage, unsigned long long seq,
                                         const Geo& g) {
  const int n = P->n, m = P->m;
  const SrcComb xf{xsrc_ptr(P, R), P->xpool + static_cast<size_t>(R->x_anchor) * n, R->w_x, R->x_mode};
  const double* y = ycur_ptr(P, R);
  double a2[2], b2[2];
  acc_init<2, 0>(a2);
  acc_init<2, 0>(b2);
  EpiKktA ea{xf, P->c};
  spmv_rows<2, 0, LM, EX>(P->AT, 0, SrcVec{y}, ea, a2, gwarp_id(g), threadIdx.x & 31, stage, seq);
  fold_long<2, 0>(P->AT, 0, seq, a2, g.cta, &P->bar->abort);
  EpiKktB eb{P->b, y};
  spmv_rows<2, 0, LM, EX>(P->A, 1, xf, eb, b2, gwarp_id(g), threadIdx.x & 31, stage, seq + 1);
  fold_long<2, 0>(P->A, 1, seq + 1, b2, g.cta, &P->bar->abort);
  (void)m;
  const double a4[4] = {b2[0], a2[0], a2[1], b2[1]};
  block_to_slots<4, 0, true>(a4, P, kRegC1, g);
}

// kModeScale (teams), one round of hx_precondition on this rank's blocks:
// the row / column norms of the rows and columns it owns (row_norm_kernel's
// formulas), their inverse square roots into the u-pool regions (u1: d_row,
// u0: d_col, peers' copies through pushes), accumulated into R (u3) / C (u2).
__device__ void team_scale_norms(const KParams* P, const Geo& g, int kind, double prow, double pcol) {
  const Team& T = P->T;
  const int n = P->n, m = P->m;
  double* dcol = P->upool;
  double* ccum = P->upool + n;
  double* drow = P->upool + 2 * static_cast<size_t>(n);
  double* rcum = drow + m;
  const int tid = g.cta * kThreads + threadIdx.x, nth = g.nctas * kThreads;
  auto norm = [&](const Sched& S, int r, double pw) {
    double acc = 0.0;
    for (int p = __ldg(S.ptr + r); p < __ldg(S.ptr + r + 1); ++p) {
      const double a = fabs(ldcg(S.val + p));
      if (kind == 0) acc = a > acc ? a : acc;
      else acc += pw == 1.0 ? a : pow(a, pw);
    }
    return acc > 0.0 ? 1.0 / sqrt(acc) : 1.0;
  };
  for (int i = T.row0 + tid; i < T.row1; i += nth) {
    const double f = norm(P->A, i, prow);
    drow[i] = f;
    rcum[i] = rcum[i] * f;
    if (T.nranks > 1) push_peers(&T, T.pu, 2 * static_cast<size_t>(n) + i, f, __ldg(T.yneed + (i - T.row0)));
  }
  for (int j = T.col0 + tid; j < T.col1; j += nth) {
    const double f = norm(P->AT, j, pcol);
    dcol[j] = f;
    ccum[j] = ccum[j] * f;
    if (T.nranks > 1) push_peers(&T, T.pu, static_cast<size_t>(j), f, __ldg(T.xneed + (j - T.col0)));
  }
}

// ... then (after a team barrier) this rank's blocks scaled with the
// scale_csr_kernel rounding (v d_row) d_col, its b and c entries with
// scale_vec_kernel's.
__device__ void team_scale_apply(const KParams* P, const Geo& g) {
  const Team& T = P->T;
  const int n = P->n;
  const double* dcol = P->upool;
  const double* drow = P->upool + 2 * static_cast<size_t>(n);
  const int tid = g.cta * kThreads + threadIdx.x, nth = g.nctas * kThreads;
  double* av = const_cast<double*>(P->A.val);
  double* tv = const_cast<double*>(P->AT.val);
  double* b = const_cast<double*>(P->b);
  double* c = const_cast<double*>(P->c);
  for (int i = T.row0 + tid; i < T.row1; i += nth) {
    const double di = drow[i];
    for (int p = __ldg(P->A.ptr + i); p < __ldg(P->A.ptr + i + 1); ++p) av[p] = (av[p] * di) * dcol[__ldg(P->A.idx + p)];
    b[i] = b[i] * di;
  }
  for (int j = T.col0 + tid; j < T.col1; j += nth) {
    const double dj = dcol[j];
    for (int p = __ldg(P->AT.ptr + j); p < __ldg(P->AT.ptr + j + 1); ++p)
      tv[p] = (tv[p] * drow[__ldg(P->AT.idx + p)]) * dj;
    c[j] = c[j] * dj;
  }
}

// certificate scan C1: candidate norms and finiteness
// Element ranges a CTA sweeps: the owned column / row blocks of its rank.
template <bool RK>
__device__ __forceinline__ void owned_ranges(const KParams* P, int& c0, int& c1, int& r0, int& r1) {
  if constexpr (RK) {
    c0 = P->T.col0, c1 = P->T.col1, r0 = P->T.row0, r1 = P->T.row1;
  } else {
    c0 = 0, c1 = P->n, r0 = 0, r1 = P->m;
  }
}

template <bool RK>
__device__ HX_PHASE_INLINE void cert_norms(const KParams* P, const Roles* R, const Geo& g) {
  const int n = P->n, m = P->m;
  const int gtid = g.cta * kThreads + threadIdx.x, gs = g.nctas * kThreads;
  int c0, c1, r0, r1;
  owned_ranges<RK>(P, c0, c1, r0, r1);
  const double* zx = P->xpool + static_cast<size_t>(R->zx_out) * n;
  const double* xp = P->xpool + static_cast<size_t>(R->xp_out) * n;
  const double* xa = P->xpool + static_cast<size_t>(R->x_anchor) * n;
  const double* yc = ycur_ptr(P, R);
  const double* yp = P->ypool + static_cast<size_t>(R->yp_out) * m;
  const double* ya = P->ypool + static_cast<size_t>(R->y_anchor) * m;
  double acc[8];
  acc_init<8, 0>(acc);
  const double s = R->cand_scale;
  for (int j = c0 + gtid; j < c1; j += gs) {
    const double x = ldcg(zx + j);
    const double vd = ldcg(xp + j) - x;
    const double vn = s * (x - ldcg(xa + j));
    acc[0] += vd * vd;
    acc[2] += vn * vn;
    acc[4] += isfinite(vd) ? 0.0 : 1.0;
    acc[6] += isfinite(vn) ? 0.0 : 1.0;
  }
  for (int i = r0 + gtid; i < r1; i += gs) {
    const double y = ldcg(yc + i);
    const double vd = ldcg(yp + i) - y;
    const double vn = s * (y - ldcg(ya + i));
    acc[1] += vd * vd;
    acc[3] += vn * vn;
    acc[5] += isfinite(vd) ? 0.0 : 1.0;
    acc[7] += isfinite(vn) ? 0.0 : 1.0;
  }
  block_to_slots<8, 0, RK>(acc, P, kRegC1, g);
}

// certificate scan C2: unit vectors u = v / ||v|| and their reductions
template <bool RK>
__device__ HX_PHASE_INLINE void cert_units(const KParams* P, const Roles* R, const Geo& g) {
  const int n = P->n, m = P->m;
  const int gtid = g.cta * kThreads + threadIdx.x, gs = g.nctas * kThreads;
  int c0, c1, r0, r1;
  owned_ranges<RK>(P, c0, c1, r0, r1);
  // u vectors are SpMV gather sources of the validation products: a ranked
  // CTA pushes its owned slices to the peers (same upool offsets)
  auto put = [&](double* base, size_t off, double v, unsigned mask) {
    base[off] = v;
    if constexpr (RK) push_peers(&P->T, P->T.pu, off, v, mask);
  };
  auto xmask = [&](int j) -> unsigned {
    if constexpr (RK) return __ldg(P->T.xneed + (j - P->T.col0));
    else return 0u;
  };
  auto ymask = [&](int i) -> unsigned {
    if constexpr (RK) return __ldg(P->T.yneed + (i - P->T.row0));
    else return 0u;
  };
  const double* zx = P->xpool + static_cast<size_t>(R->zx_out) * n;
  const double* xp = P->xpool + static_cast<size_t>(R->xp_out) * n;
  const double* xa = P->xpool + static_cast<size_t>(R->x_anchor) * n;
  const double* yc = ycur_ptr(P, R);
  const double* yp = P->ypool + static_cast<size_t>(R->yp_out) * m;
  const double* ya = P->ypool + static_cast<size_t>(R->y_anchor) * m;
  double acc[12];
  acc_init<12, 0x577u>(acc);
  const double s = R->cand_scale;
  for (int j = c0 + gtid; j < c1; j += gs) {
    const double x = ldcg(zx + j);
    const double cj = __ldg(P->c + j);
    if (R->cand_on[0]) {
      const double u = (ldcg(xp + j) - x) / R->cn2[0];
      put(P->upool, static_cast<size_t>(j), u, xmask(j));
      acc[0] = dmax(acc[0], fabs(u));
      acc[1] = dmax(acc[1], u);
      acc[2] = dmax(acc[2], -u);
      acc[3] += cj * u;
    }
    if (R->cand_on[2]) {
      const double u = (s * (x - ldcg(xa + j))) / R->cn2[2];
      put(P->upool, static_cast<size_t>(n) + j, u, xmask(j));
      acc[4] = dmax(acc[4], fabs(u));
      acc[5] = dmax(acc[5], u);
      acc[6] = dmax(acc[6], -u);
      acc[7] += cj * u;
    }
  }
  for (int i = r0 + gtid; i < r1; i += gs) {
    const double y = ldcg(yc + i);
    const double bi = __ldg(P->b + i);
    if (R->cand_on[1]) {
      const double u = (ldcg(yp + i) - y) / R->cn2[1];
      put(P->upool, 2 * static_cast<size_t>(n) + i, u, ymask(i));
      acc[8] = dmax(acc[8], fabs(u));
      acc[9] += bi * u;
    }
    if (R->cand_on[3]) {
      const double u = (s * (y - ldcg(ya + i))) / R->cn2[3];
      put(P->upool, 2 * static_cast<size_t>(n) + m + i, u, ymask(i));
      acc[10] = dmax(acc[10], fabs(u));
      acc[11] += bi * u;
    }
  }
  block_to_slots<12, 0x577u, RK>(acc, P, kRegC2, g);
}

// certificate scan C3: the validation SpMVs, up to four independent products
template <bool RK, int LM = 0, int EX = 2>
__device__ HX_PHASE_INLINE void cert_products(const KParams* P, const Roles* R, WarpStage* stage,
                                              unsigned long long seq, const Geo& g) {
  const int n = P->n, m = P->m;
  double acc[6];
  acc_init<6, 0x3Fu>(acc);
  const double* u0 = P->upool;
  const double* u2 = P->upool + n;
  const double* u1 = P->upool + 2 * static_cast<size_t>(n);
  const double* u3 = u1 + m;
  const int gw = gwarp_id(g), lane = threadIdx.x & 31;
  const Sched AT = P->AT;
  const Sched A = P->A;
  for (int k = 0; k < 2; ++k) {
    if (R->cand_on[1 + 2 * k]) {
      double a2[2];
      acc_init<2, 3u>(a2);
      EpiPosNeg e;
      spmv_rows<2, 3u, LM, EX>(AT, 2 + k, SrcVec{k ? u3 : u1}, e, a2, gw, lane, stage, seq);
      fold_long<2, 3u>(AT, 2 + k, seq, a2, g.cta, &P->bar->abort);
      acc[2 * k] = a2[0], acc[2 * k + 1] = a2[1];
    }
    if (R->cand_on[2 * k]) {
      double a1[1];
      acc_init<1, 1u>(a1);
      EpiAbs e;
      spmv_rows<1, 1u, LM, EX>(A, 2 + k, SrcVec{k ? u2 : u0}, e, a1, gw, lane, stage, seq);
      fold_long<1, 1u>(A, 2 + k, seq, a1, g.cta, &P->bar->abort);
      acc[4 + k] = a1[0];
    }
  }
  block_to_slots<6, 0x3Fu, RK>(acc, P, kRegC3, g);
}

// ---------------------------------------------------------------------------
// Baseline schemes: solve_baseline (src/solver.cpp:344-509) on the device.
// Vanilla PDHG runs the same fused phases as rHPDHG with z <- T(z) roles;
// the averaged schemes fold the running average (update_average,
// src/baselines.cpp:20-31, and the products' means, solver.cpp:404-416) into
// the phase epilogues out of place (average slot avg_cur -> avg_out), so the
// KKT at the average (solver.cpp:418-421) needs no extra pass; the residual
// at the average (restarted average every iteration, averaged at epoch
// starts and traced iterations, :424-433) takes two more fused phases: the
// PDHG step at the average.  One thread-0 controller per CTA, replicated as
// in the main loop; no speculation (phase A follows the controller).
// ---------------------------------------------------------------------------
struct EpiPrimalAvg {  // phase A + average update of x and A^T y
  const double* xs;
  const double* c;
  double* zx;
  double* xp;
  const double* xa_in;
  const double* ta_in;
  double* xa_out;
  double* ta_out;
  double eta, w;
  int copy;
  struct In {
    double xs, c, xa, ta;
  };
  __device__ __forceinline__ In load(int j) const {
    return In{ldcg(xs + j), __ldg(c + j), copy ? 0.0 : ldcg(xa_in + j), copy ? 0.0 : ldcg(ta_in + j)};
  }
  __device__ __forceinline__ void apply(int j, double aty, const In& in, double (&t)[3]) const {
    const double x = in.xs;
    zx[j] = x;
    double xn = x - eta * (aty + in.c);
    xn = xn < 0.0 ? 0.0 : xn;
    xp[j] = xn;
    const double xa = copy ? x : in.xa + w * (x - in.xa);
    const double ta = copy ? aty : in.ta + w * (aty - in.ta);
    xa_out[j] = xa;
    ta_out[j] = ta;
    double rc = -(in.c + ta);  // dual residual at the average
    rc = rc < 0.0 ? 0.0 : rc;
    const double dx = x - xn;
    t[0] = rc * rc;
    t[1] = in.c * xa;
    t[2] = dx * dx;
  }
};

struct EpiDualAvg {  // phase B + average update of y and A x
  const double* y;
  const double* ax;
  const double* b;
  double* yp;
  double* axp;
  const double* ya_in;
  const double* aa_in;
  double* ya_out;
  double* aa_out;
  double eta, w;
  int copy;
  struct In {
    double y, ax, b, ya, aa;
  };
  __device__ __forceinline__ In load(int i) const {
    return In{ldcg(y + i), ldcg(ax + i), __ldg(b + i), copy ? 0.0 : ldcg(ya_in + i), copy ? 0.0 : ldcg(aa_in + i)};
  }
  __device__ __forceinline__ void apply(int i, double s, const In& in, double (&t)[4]) const {
    const double ypi = in.y + eta * ((2.0 * s - in.ax) - in.b);
    yp[i] = ypi;
    axp[i] = s;
    const double ya = copy ? in.y : in.ya + w * (in.y - in.ya);
    const double aa = copy ? in.ax : in.aa + w * (in.ax - in.aa);
    ya_out[i] = ya;
    aa_out[i] = aa;
    const double d = aa - in.b;  // primal residual at the average
    const double dy = in.y - ypi;
    const double dax = in.ax - s;
    t[0] = d * d;
    t[1] = in.b * ya;
    t[2] = dy * dy;
    t[3] = dy * dax;
  }
};

struct EpiAvgStepPrimal {  // PDHG step at the average, primal half
  const double* xa;
  const double* c;
  double* xbar;
  double eta;
  struct In {
    double xa, c;
  };
  __device__ __forceinline__ In load(int j) const { return In{ldcg(xa + j), __ldg(c + j)}; }
  __device__ __forceinline__ void apply(int j, double at, const In& in, double (&t)[1]) const {
    double xn = in.xa - eta * (at + in.c);
    xn = xn < 0.0 ? 0.0 : xn;
    xbar[j] = xn;
    const double d = in.xa - xn;
    t[0] = d * d;
  }
};

struct EpiAvgStepDual {  // PDHG step at the average, dual half (products only)
  const double* ya;
  const double* aa;
  const double* b;
  double eta;
  struct In {
    double ya, aa, b;
  };
  __device__ __forceinline__ In load(int i) const { return In{ldcg(ya + i), ldcg(aa + i), __ldg(b + i)}; }
  __device__ __forceinline__ void apply(int, double s, const In& in, double (&t)[2]) const {
    const double ypn = in.ya + eta * ((2.0 * s - in.aa) - in.b);
    const double dy = in.ya - ypn;
    const double dax = in.aa - s;
    t[0] = dy * dy;
    t[1] = dy * dax;
  }
};

__device__ HX_PHASE_INLINE void phase_primal_avg(const KParams* P, const Roles* R, int par, WarpStage* stage,
                                                 unsigned long long seq, const SpmvHead& head, const Geo& g) {
  const int n = P->n;
  double acc[3];
  acc_init<3, 0>(acc);
  const int cur = R->avg_cur < 0 ? 0 : R->avg_cur;
  EpiPrimalAvg e{xsrc_ptr(P, R),
                 P->c,
                 P->xpool + static_cast<size_t>(R->zx_out) * n,
                 P->xpool + static_cast<size_t>(R->xp_out) * n,
                 P->xavg + static_cast<size_t>(cur) * n,
                 P->tavg + static_cast<size_t>(cur) * n,
                 P->xavg + static_cast<size_t>(R->avg_out) * n,
                 P->tavg + static_cast<size_t>(R->avg_out) * n,
                 R->eta,
                 R->w_avg,
                 R->avg_mode == 1};
  spmv_rows<3, 0>(P->AT, par, SrcVec{ycur_ptr(P, R)}, e, acc, gwarp_id(g), threadIdx.x & 31, stage, seq, head);
  fold_long<3, 0>(P->AT, par, seq, acc, g.cta, &P->bar->abort);
  block_to_slots<3, 0, false>(acc, P, kRegA + par, g);
}

__device__ HX_PHASE_INLINE void phase_dual_avg(const KParams* P, const Roles* R, int par, WarpStage* stage,
                                               unsigned long long seq, const SpmvHead& head, const Geo& g) {
  const int n = P->n, m = P->m;
  double acc[4];
  acc_init<4, 0>(acc);
  const int cur = R->avg_cur < 0 ? 0 : R->avg_cur;
  EpiDualAvg e{ycur_ptr(P, R),
               axcur_ptr(P, R),
               P->b,
               P->ypool + static_cast<size_t>(R->yp_out) * m,
               P->axpool + static_cast<size_t>(R->axp_out) * m,
               P->yavg + static_cast<size_t>(cur) * m,
               P->aavg + static_cast<size_t>(cur) * m,
               P->yavg + static_cast<size_t>(R->avg_out) * m,
               P->aavg + static_cast<size_t>(R->avg_out) * m,
               R->eta,
               R->w_avg,
               R->avg_mode == 1};
  spmv_rows<4, 0>(P->A, par, SrcVec{P->xpool + static_cast<size_t>(R->xp_out) * n}, e, acc, gwarp_id(g),
                  threadIdx.x & 31, stage, seq, head);
  fold_long<4, 0>(P->A, par, seq, acc, g.cta, &P->bar->abort);
  block_to_slots<4, 0, false>(acc, P, kRegB + par, g);
}

__device__ HX_PHASE_INLINE void phase_avgstep_a(const KParams* P, const Roles* R, WarpStage* stage,
                                                unsigned long long seq, const Geo& g) {
  const int n = P->n, m = P->m;
  double acc[1];
  acc_init<1, 0>(acc);
  EpiAvgStepPrimal e{P->xavg + static_cast<size_t>(R->avg_out) * n, P->c, P->xbar, R->eta};
  spmv_rows<1, 0>(P->AT, 0, SrcVec{P->yavg + static_cast<size_t>(R->avg_out) * m}, e, acc, gwarp_id(g),
                  threadIdx.x & 31, stage, seq);
  fold_long<1, 0>(P->AT, 0, seq, acc, g.cta, &P->bar->abort);
  block_to_slots<1, 0, false>(acc, P, kRegPA, g);
}

__device__ HX_PHASE_INLINE void phase_avgstep_b(const KParams* P, const Roles* R, WarpStage* stage,
                                                unsigned long long seq, const Geo& g) {
  const int m = P->m;
  double acc[2];
  acc_init<2, 0>(acc);
  EpiAvgStepDual e{P->yavg + static_cast<size_t>(R->avg_out) * m, P->aavg + static_cast<size_t>(R->avg_out) * m,
                   P->b, R->eta};
  spmv_rows<2, 0>(P->A, 1, SrcVec{P->xbar}, e, acc, gwarp_id(g), threadIdx.x & 31, stage, seq);
  fold_long<2, 0>(P->A, 1, seq, acc, g.cta, &P->bar->abort);
  block_to_slots<2, 0, false>(acc, P, kRegPB, g);
}

// canonical_norm_with_product, src/pdhg_core.cpp:37-51, from the three sums;
// *bad = 1 on the domain_error branch.
__device__ double canonical_from(double dx2, double dy2, double dyax, double eta, int* bad) {
  const double q = dx2 / eta - 2.0 * dyax + dy2 / eta;
  if (q < 0.0) {
    if (q < -1e-9 * ((dx2 + dy2) / eta)) *bad = 1;
    return 0.0;
  }
  return sqrt(q);
}

__device__ __forceinline__ bool tracing_at(const Ctl& C, long long it) {
  return C.trace_period > 0 && it % C.trace_period == 0;
}

// Restart / next roles / limits of a baseline (src/solver.cpp:483-508).
__device__ void finish_iteration_baseline(Ctl& C, hplp_epoch_t* epochs, bool writer, double res, bool time_up) {
  Roles& R = C.r;
  const bool averaged = C.scheme != HPLP_SCHEME_VANILLA;
  bool restart = false;
  if (C.scheme == HPLP_SCHEME_RESTARTED_AVERAGE) {
    restart = should_restart(C, C.n, C.k, res, C.res_epoch_start);
    if (!restart && C.restart_kind == HPLP_RESTART_ADAPTIVE && C.stall_cap > 0 && C.k >= C.stall_cap) restart = true;
  }
  const int avg_now = R.avg_out;  // the average after this iteration's update
  if (averaged) C.avg_count = R.avg_mode == 1 ? 1 : C.avg_count + 1;
  if (restart) {  // z <- z-bar, a_x <- a_x_avg, empty average (:490-497)
    if (writer && C.n_epochs > 0) epochs[(C.n_epochs - 1) % kEpochCap].restart_length = C.k;
    R.x_src = avg_now, R.x_src_avg = 1;
    R.y_cur = avg_now, R.y_cur_avg = 1;
    R.ax_cur = avg_now, R.ax_cur_avg = 1;
    R.avg_mode = 1;
    R.avg_cur = -1;
    C.avg_count = 0;
    C.n += 1;
    C.k = 0;
  } else {  // z <- T(z), a_x <- A x+ (:498-502)
    R.x_src = R.xp_out, R.x_src_avg = 0;
    R.y_cur = R.yp_out, R.y_cur_avg = 0;
    R.ax_cur = R.axp_out, R.ax_cur_avg = 0;
    if (averaged) {
      R.avg_mode = 2;
      R.avg_cur = avg_now;
      R.w_avg = 1.0 / static_cast<double>(C.avg_count + 1);
    }
    C.k += 1;
  }
  R.x_mode = 0;
  R.w_x = 0.0;
  R.check = 0;
  C.it += 1;
  const int xs = R.x_src_avg ? -1 : R.x_src, yc = R.y_cur_avg ? -1 : R.y_cur, ac = R.ax_cur_avg ? -1 : R.ax_cur;
  R.zx_out = pick_free(kXPool, xs, C.x_best, C.last_zx, -1);
  R.xp_out = pick_free(kXPool, xs, C.x_best, C.last_zx, R.zx_out);
  R.yp_out = pick_free(kYPool, yc, C.y_best, C.last_y_avg ? -1 : C.last_y, -1);
  R.yc_out = pick_free(kYPool, yc, C.y_best, C.last_y_avg ? -1 : C.last_y, R.yp_out);
  R.axp_out = pick_free(kAxPool, ac, -1, -1, -1);
  R.axc_out = pick_free(kAxPool, ac, R.axp_out, -1, -1);
  if (averaged) R.avg_out = pick_free(kAvgPool, R.avg_cur, C.avg_best, R.x_src_avg ? R.x_src : -1, avg_now);
  R.w_next = 0.0;
  R.avg_step = C.scheme == HPLP_SCHEME_RESTARTED_AVERAGE ||
               (C.scheme == HPLP_SCHEME_AVERAGED && (C.k == 0 || tracing_at(C, C.it)));
  if (C.it >= C.iteration_limit) set_final_limit(C, HPLP_STATUS_ITERATION_LIMIT);
  else if (time_up) set_final_limit(C, HPLP_STATUS_TIME_LIMIT);
  if (tracing_at(C, C.last_it)) {
    C.paused = 1;
    R.stop = 1;
  }
  if (C.it >= C.batch_end) R.stop = 1;
}

// One baseline iteration's decisions (src/solver.cpp:418-489): t[0..6] as
// in the main loop (KKT terms at the candidate; z's own step terms), a[0..2]
// the step at the average (when R.avg_step).
__device__ void main_logic_baseline(Ctl& C, const double* t, const double* a, hplp_epoch_t* epochs, bool writer,
                                    bool time_up) {
  Roles& R = C.r;
  const bool averaged = C.scheme != HPLP_SCHEME_VANILLA;
  double kkt[4];
  kkt[0] = sqrt(t[3]) / (1.0 + C.b_norm);
  kkt[1] = sqrt(t[0]) / (1.0 + C.c_norm);
  kkt[2] = fabs(t[1] + t[4]) / (1.0 + fabs(t[1]) + fabs(t[4]));
  kkt[3] = dmax(dmax(kkt[0], kkt[1]), kkt[2]);
  const double eta = R.eta;
  int bad = 0;
  const double res_z = canonical_from(t[2], t[5], t[6], eta, &bad);  // ||z - T(z)||, with products
  double res;
  C.spmv += 2;
  if (averaged && R.avg_step) {
    res = canonical_from(a[0], a[1], a[2], eta, &bad);
    C.spmv += 2;
  } else if (!averaged) {
    res = res_z;
  } else {
    res = NAN;
  }
  if (bad) {
    C.error = HPLP_EDOMAIN;
    R.stop = 1;
    return;
  }
  if (C.k == 0) {
    C.res_epoch_start = res;
    if (writer) {
      hplp_epoch_t& e = epochs[C.n_epochs % kEpochCap];
      e.epoch = C.n;
      e.restart_length = 0;
      e.residual_at_start = res;
      e.kkt_at_start = {kkt[0], kkt[1], kkt[2], kkt[3]};
    }
    C.n_epochs += 1;
  }
  C.x_best_prev = C.x_best;
  if (kkt[3] < C.best_kkt) {  // candidate: z, or the average slot just written
    C.best_kkt = kkt[3];
    for (int i = 0; i < 4; ++i) C.best_err[i] = kkt[i];
    if (averaged) {
      C.avg_best = R.avg_out;
      C.x_best = C.y_best = -1;
    } else {
      C.x_best = R.zx_out;
      C.y_best = R.y_cur;
      C.avg_best = -1;
    }
  }
  C.last_it = C.it;
  C.last_n = C.n;
  C.last_k = C.k;
  C.last_res = res;
  C.last_res_diff = res_z;
  for (int i = 0; i < 4; ++i) C.last_kkt[i] = kkt[i];
  C.last_zx = R.zx_out;
  C.last_xp = R.xp_out;
  C.last_y = R.y_cur;
  C.last_y_avg = R.y_cur_avg;
  C.last_yp = R.yp_out;
  C.last_xa = R.x_anchor;
  C.last_ya = R.y_anchor;
  C.last_ax = R.ax_cur;
  C.last_axp = R.axp_out;
  C.last_cand_avg = averaged ? R.avg_out : -1;
  if (kkt[3] <= C.tol) {  // :462-465, returns the candidate
    C.status = HPLP_STATUS_OPTIMAL;
    C.final_x = R.zx_out;
    C.final_y = R.y_cur;
    C.final_avg = C.last_cand_avg;
    for (int i = 0; i < 4; ++i) C.final_kkt[i] = kkt[i];
    R.stop = 1;
    if (tracing_at(C, C.last_it)) C.paused = 1;
    return;
  }
  if (C.check_period > 0 && C.it > 0 && C.it % C.check_period == 0) {  // :467-481, difference candidate only
    R.check = 1;
    R.cand_scale = 0.0;
    return;
  }
  finish_iteration_baseline(C, epochs, writer, res, time_up);
}

__device__ __forceinline__ void loop_body_baseline(const KParams* P, const Geo& g) {
  __shared__ Ctl C;
  __shared__ double tot[kMaxQ];
  __shared__ double atot[4];
  extern __shared__ __align__(16) unsigned char dyn_smem[];
  const int lane = threadIdx.x & 31;
  const int warp = threadIdx.x >> 5;
  const bool writer = g.cta == 0;
  WarpStage* stage = reinterpret_cast<WarpStage*>(dyn_smem) + warp;
  const unsigned long long t_start = global_ns();
  ctl_load(P->ctl, C);
  const unsigned long long budget = C.time_budget_ns;
  const Roles* R = &C.r;
  GridBar* bar = P->bar;
  unsigned long long target = 0;
  unsigned long long seq = 1;
  const bool vanilla = C.scheme == HPLP_SCHEME_VANILLA;
  while (!R->stop) {
    const int par = static_cast<int>(C.it & 1);
    SpmvHead head;
    spmv_head(P->AT, gwarp_id(g), lane, head);
    if (vanilla) phase_primal_t<false, false>(P, R, par, stage, ++seq, head, g);
    else phase_primal_avg(P, R, par, stage, ++seq, head, g);
    if (writer && threadIdx.x == 0 && budget != 0ull)
      bar->time_up[par] = (global_ns() - t_start) > budget ? 1u : 0u;
    spmv_head(P->A, gwarp_id(g), lane, head);
    if (!grid_sync(bar, target)) return;
    if (vanilla) phase_dual<false>(P, R, par, stage, ++seq, head, g);
    else phase_dual_avg(P, R, par, stage, ++seq, head, g);
    if (!grid_sync(bar, target)) return;
    if (R->avg_step) {  // the PDHG step at the average (:424-433)
      phase_avgstep_a(P, R, stage, ++seq, g);
      if (!grid_sync(bar, target)) return;
      phase_avgstep_b(P, R, stage, ++seq, g);
      if (!grid_sync(bar, target)) return;
      {
        const double* ra = region_ptr(P, kRegPA, g.nrec);
        const double* rb = region_ptr(P, kRegPB, g.nrec);
        block_totals(3, [&](int q) { return QSrc{q == 0 ? ra : rb, q == 0 ? 0 : q - 1, nullptr, 0, 0, false}; },
                     atot, g);
      }
    }
    if (warp == 0) {
      double t[8];
      warp_totals_main<false>(P, par, t, g);
      if (lane == 0) {
        for (int i = 0; i < 7; ++i) tot[i] = t[i];
        const bool time_up = budget != 0ull && *reinterpret_cast<volatile unsigned*>(&bar->time_up[par]) != 0u;
        main_logic_baseline(C, tot, atot, P->epochs, writer, time_up);
      }
    }
    __syncthreads();
    if (R->check) {  // certificate scan, iterate-difference candidate (:467-481)
      cert_norms<false>(P, R, g);
      if (!grid_sync(bar, target)) return;
      {
        const double* rg = region_ptr(P, kRegC1, g.nrec);
        block_totals(8, [&](int q) { return QSrc{rg, q, nullptr, 0, 0, false}; }, tot, g);
      }
      if (threadIdx.x == 0) {
        int any = 0;
        for (int c = 0; c < 4; ++c) {
          C.r.cn2[c] = sqrt(tot[c]);
          C.cfinite[c] = tot[4 + c] == 0.0;
          C.r.cand_on[c] = c < 2 && C.r.cn2[c] > 0.0 && C.cfinite[c];
          any |= C.r.cand_on[c];
        }
        if (!any) scan_logic(C, P->epochs, writer, false);
      }
      __syncthreads();
      if (R->check) {
        cert_units<false>(P, R, g);
        if (!grid_sync(bar, target)) return;
        {
          const double* rg = region_ptr(P, kRegC2, g.nrec);
          block_totals(12, [&](int q) { return QSrc{rg, q, nullptr, 0, 0, ((0x577u >> q) & 1u) != 0}; }, tot, g);
        }
        if (threadIdx.x == 0) {
          C.cinf[0] = tot[0], C.cmax_u[0] = tot[1], C.cmax_negu[0] = tot[2], C.cdot[0] = tot[3];
          C.cinf[1] = tot[8], C.cdot[1] = tot[9];
        }
        __syncthreads();
        cert_products<false>(P, R, stage, ++seq, g);
        if (!grid_sync(bar, target)) return;
        {
          const double* rg = region_ptr(P, kRegC3, g.nrec);
          block_totals(6, [&](int q) { return QSrc{rg, q, nullptr, 0, 0, true}; }, tot, g);
        }
        if (threadIdx.x == 0) {
          C.cmax_at[1] = tot[0], C.cmax_negat[1] = tot[1];
          C.cmax_abs_au[0] = tot[4];
          const bool time_up = budget != 0ull && *reinterpret_cast<volatile unsigned*>(&bar->time_up[par]) != 0u;
          scan_logic(C, P->epochs, writer, time_up);
        }
        __syncthreads();
      }
    }
    if (R->stop) break;
    if (!grid_sync(bar, target)) return;  // phase A of the next iteration rewrites this one's long-row counters
  }
  if (writer) ctl_store(C, P->ctl);
}

__global__ void __launch_bounds__(kThreads, kMinBlocks) loop_kernel_baseline(const __grid_constant__ KParams KP) {
  const Geo g{static_cast<int>(blockIdx.x), static_cast<int>(gridDim.x), static_cast<int>(blockIdx.x),
              static_cast<int>(gridDim.x)};
  loop_body_baseline(&KP, g);
}

// ---------------------------------------------------------------------------
// The persistent loop kernel.
// ---------------------------------------------------------------------------
// RK = false: one GPU, P in the constant bank (loop_kernel).  RK = true: one
// rank of a row-partitioned team (loop_kernel_team), P in shared memory.
// SU (teams): the setup modes (power iteration, KKT, preconditioning) in their
// own kernel (team_setup_kernel), so the loop's register allocation is not
// charged for them.
// TR: the trace-ring kernels (loop_kernel_trace / loop_kernel_team_trace).
template <bool RK, bool BOX = false, int LM = 2, bool CB = false, int EX = 2, bool SU = false, bool TR = false>
__device__ __forceinline__ void loop_body(const KParams* P, const Geo& g) {
  __shared__ Ctl C;
  __shared__ double tot[kMaxQ];
  __shared__ int s_time_up;
  extern __shared__ __align__(16) unsigned char dyn_smem[];
  const int lane = threadIdx.x & 31;
  const int warp = threadIdx.x >> 5;
  const bool writer = g.cta == 0;
  WarpStage* stage = reinterpret_cast<WarpStage*>(dyn_smem) + warp;
  const unsigned long long t_start = global_ns();
  ctl_load(P->ctl, C);
  const unsigned long long budget = C.time_budget_ns;
  const Roles* R = &C.r;
  GridBar* bar = P->bar;
  unsigned long long target = 0;
  unsigned long long seq = 1;  // phase sequence number (long-row flags; reset per launch)
  unsigned long long repoch = C.team_epochs;  // team barriers passed (continues across launches)
  const bool solo = !RK || P->T.nranks == 1;  // a team of one needs no cross-rank step
  auto sync = [&]() -> bool {
    if constexpr (RK) {
      if (!solo) return team_sync(bar, P->T, g, target, repoch);
    }
    return grid_sync(bar, target);
  };
  // end-of-iteration barrier: a team also forms the rank records of the
  // main reduction there
  auto sync_reduce = [&](int pr) -> bool {
    if constexpr (RK) {
      if (!solo) return team_sync(bar, P->T, g, target, repoch, P->slots, P->T.prereduce ? pr : -1, BOX);
    }
    return grid_sync(bar, target);
  };
  // time-limit flag: decided by rank 0 alone so every rank stops together
  auto set_time_up = [&](int pr, unsigned v) {
    if constexpr (RK) {
      if (P->T.rank == 0)
        for (int r = 0; r < P->T.nranks; ++r) *reinterpret_cast<volatile unsigned*>(&P->T.pb[r]->time_up[pr]) = v;
    } else {
      bar->time_up[pr] = v;
    }
  };
  auto get_time_up = [&](int pr) -> unsigned {
    if constexpr (RK) return *reinterpret_cast<volatile unsigned*>(&P->T.pb[P->T.rank]->time_up[pr]);
    else return *reinterpret_cast<volatile unsigned*>(&bar->time_up[pr]);
  };

  if ((!RK || SU) && C.mode == kModePower) {
    // power_iteration loop body, src/sparse_matrix.cpp:153-177 (a team: each
    // rank its rows / columns, the norms over every rank's records)
    while (!R->stop) {
      power_a<LM, EX, RK>(P, R, stage, ++seq, g);
      if (!sync()) return;
      {
        const double* rg = region_ptr(P, kRegPA, g.nrec);
        block_totals(1, [&](int) { return QSrc{rg, 0, nullptr, 0, 0, false}; }, tot, g);
      }
      if (threadIdx.x == 0) {
        const double sigma = sqrt(tot[0]);
        C.pw_iters = C.pw_k + 1;
        C.pw_sigma_cur = sigma;
        if (sigma == 0.0) {
          C.pw_redraw = 1;
          C.r.stop = 1;
        }
      }
      __syncthreads();
      if (R->stop) break;
      power_b<LM, EX, RK>(P, stage, ++seq, g);
      if (!sync()) return;
      {
        const double* rg = region_ptr(P, kRegPB, g.nrec);
        block_totals(1, [&](int) { return QSrc{rg, 0, nullptr, 0, 0, false}; }, tot + 1, g);
      }
      if (threadIdx.x == 0) {
        const double sigma = C.pw_sigma_cur;
        C.pw_sigma = sigma;
        if (C.pw_k > 0 && fabs(sigma - C.pw_sigma_prev) <= C.pw_tol * sigma) {
          C.pw_converged = 1;
          C.r.stop = 1;
        } else {
          C.pw_sigma_prev = sigma;
          const double zn = sqrt(tot[1]);
          if (zn == 0.0) {
            C.pw_converged = 1;
            C.r.stop = 1;
          } else {
            C.r.pw_mode = 1;
            C.r.pw_zn = zn;
            C.pw_k += 1;
            if (C.pw_k >= C.pw_max) C.r.stop = 1;
          }
        }
      }
      __syncthreads();
    }
    if (threadIdx.x == 0) C.team_epochs = repoch;
    if (writer) ctl_store(C, P->ctl);
    return;
  }
  if constexpr (RK && SU) {
    if (C.mode == kModeKkt) {
      team_kkt<LM, EX>(P, R, stage, seq + 1, g);
      seq += 2;
      if (!sync()) return;
      const double* rg = region_ptr(P, kRegC1, g.nrec);
      block_totals(4, [&](int q) { return QSrc{rg, q, nullptr, 0, 0, false}; }, tot, g);
      if (threadIdx.x == 0) {
        for (int q = 0; q < 4; ++q) C.kk_tot[q] = tot[q];
        C.team_epochs = repoch;
      }
      if (writer) ctl_store(C, P->ctl);
      return;
    }
    if (C.mode == kModeScale) {
      // hx_precondition on the team: ruiz rounds, then the
      // Pock-Chambolle round; every exchange is a push + team barrier
      const Team& T = P->T;
      const int n = P->n, m = P->m;
      const int tid = g.cta * kThreads + threadIdx.x, nth = g.nctas * kThreads;
      for (int i = T.row0 + tid; i < T.row1; i += nth) P->upool[2 * static_cast<size_t>(n) + m + i] = 1.0;
      for (int j = T.col0 + tid; j < T.col1; j += nth) P->upool[n + j] = 1.0;
      for (int k = 0; k < C.sc_ruiz + C.sc_pc; ++k) {
        const bool ruiz = k < C.sc_ruiz;
        team_scale_norms(P, g, ruiz ? 0 : 1, ruiz ? 1.0 : 2.0 - C.sc_alpha, ruiz ? 1.0 : C.sc_alpha);
        if (!sync()) return;
        team_scale_apply(P, g);
        if (!sync()) return;
      }
      double a2[2] = {0.0, 0.0};
      for (int i = T.row0 + tid; i < T.row1; i += nth) {
        const double v = ldcg(P->b + i);
        a2[0] += v * v;
      }
      for (int j = T.col0 + tid; j < T.col1; j += nth) {
        const double v = ldcg(P->c + j);
        a2[1] += v * v;
      }
      block_to_slots<2, 0, true>(a2, P, kRegC1, g);
      if (!sync()) return;
      const double* rg = region_ptr(P, kRegC1, g.nrec);
      block_totals(2, [&](int q) { return QSrc{rg, q, nullptr, 0, 0, false}; }, tot, g);
      if (threadIdx.x == 0) {
        C.sc_bsq = tot[0];
        C.sc_csq = tot[1];
        C.team_epochs = repoch;
      }
      if (writer) ctl_store(C, P->ctl);
      return;
    }
    return;  // no loop in the setup kernel
  }

  unsigned long long* prof = (!RK && P->prof) ? P->prof + blockIdx.x * 16 : nullptr;
  // phase timers live in shared memory (thread 0 only): per-thread arrays would
  // hold registers across the whole loop in every thread
  __shared__ unsigned long long pacc[8], pacc2[3], tp;
  if (threadIdx.x == 0) {
    for (int k = 0; k < 8; ++k) pacc[k] = 0;
    for (int k = 0; k < 3; ++k) pacc2[k] = 0;
    tp = clock64();
  }
  auto mark = [&](int k) {  // SM cycles (clock64); the host converts with the SM clock
    if (prof && threadIdx.x == 0) {
      const unsigned long long t = clock64();
      pacc[k] += t - tp;
      tp = t;
    }
  };
  // Phase A of iteration it+1 runs speculatively (roles of "no restart,
  // no stop": make_spec) in warps 1..15 while warp 0 reduces the partials
  // and runs the controller of iteration it; warp 0 then runs its own,
  // lighter, share of the tasks (the schedule's lead).  When the decision
  // differs from the speculation (a restart, a stop), every CTA waits for
  // the speculative phase to finish everywhere and phase A is redone with
  // the real roles.  The speculative outputs go to buffers no live role
  // uses, so a discarded speculation leaves no trace.
  __shared__ Roles SR;
  bool spec_done = false;
  while (!R->stop) {
    const int par = static_cast<int>(C.it & 1);
    SpmvHead head;
    if (!spec_done) {
      spmv_head<LM>(P->AT, gwarp_id(g), lane, head);
      phase_primal_t<RK, BOX, LM, EX, TR>(P, R, par, stage, ++seq, head, g);
      if (writer && threadIdx.x == 0 && budget != 0ull) set_time_up(par, (global_ns() - t_start) > budget ? 1u : 0u);
    }
    mark(0);
    spmv_head<LM>(CB ? P->cbs[0] : P->A, gwarp_id(g), lane, head);
    if (!sync()) return;
    mark(1);
    if (!phase_dual<RK, LM, CB, EX, TR>(P, R, par, stage, ++seq, head, g, &target)) return;
    if (threadIdx.x == 0) make_spec(C, SR);
    mark(2);
    spmv_head<LM>(P->AT, gwarp_id(g), lane, head);
    if (!sync_reduce(par)) return;
    mark(3);
    if (warp == 0) {
      unsigned long long cA = clock64(), cB = 0, cC = 0;
      // (issuing these loads before the other warps start the speculative
      // phase A -- a named barrier -- measured slower: the 40 registers they
      // hold across the barrier spill)
      double t[8];
      if (solo || !P->T.prereduce) warp_totals_main<BOX>(P, par, t, g);
      else warp_totals_ranks(P, par, t, g.cta);
      // the independent fp64 divides / square roots, one per lane, executed
      // uniformly (operands selected per lane, one sqrt + one divide)
      double num = 1.0, den = 1.0;
      if (lane == 0) num = t[3], den = 1.0 + C.b_norm;
      else if (lane == 1) num = t[0], den = 1.0 + C.c_norm;
      else if (lane == 2) num = fabs(t[1] + (t[4] + t[7])), den = 1.0 + fabs(t[1]) + fabs(t[4] + t[7]);
      else if (lane == 3) num = t[2], den = C.r.eta;
      else if (lane == 4) num = t[5], den = C.r.eta;
      else if (lane == 5) den = static_cast<double>(C.k + 2);
      else if (lane == 6) den = static_cast<double>(C.k + 3);
      const double sq = sqrt(num);
      const double v = (lane < 2 ? sq : num) / den;
      double pre[7];
#pragma unroll
      for (int i = 0; i < 7; ++i) pre[i] = __shfl_sync(0xffffffffu, v, i);
      const int due = __shfl_sync(0xffffffffu, lane == 7 && C.check_period > 0 && C.it % C.check_period == 0, 7);
      cB = clock64();
      // a traced iteration of a trace-ring kernel: the classes' counts and
      // the normalized candidate's sums (phase A partials 3..6, phase B 4..5)
      double trt[6] = {0.0, 0.0, 0.0, 0.0, 0.0, 0.0};
      const bool traced = TR && ring_slot(C, C.it) >= 0;
      if (traced) warp_totals_trace(P, par, trt, g);
      if (lane == 0) {
#pragma unroll
        for (int i = 0; i < 7; ++i) tot[i] = t[i];
        s_time_up = budget != 0ull && get_time_up(par) != 0u;
        C.w_k2 = pre[5];
        C.w_k3 = pre[6];
        main_logic(C, tot, pre, P->epochs, writer, s_time_up != 0, traced ? P->ring_rec : nullptr,
                   traced ? trt : nullptr, due != 0);
      }
      cC = clock64();
      __syncwarp();
      if (prof && threadIdx.x == 0) {
        pacc2[0] += cB - cA;
        pacc2[1] += cC - cB;
      }
    }
    mark(4);
    // speculative phase A of iteration it+1 (measured: worth ~10% against
    // running phase A after the controller)
    phase_primal_t<RK, BOX, LM, EX, TR>(P, &SR, par ^ 1, stage, ++seq, head, g);
    if (writer && threadIdx.x == 0 && budget != 0ull)
      set_time_up(par ^ 1, (global_ns() - t_start) > budget ? 1u : 0u);
    __syncthreads();
    mark(0);
    if (prof && threadIdx.x == 0) pacc[5] += 1;

    if (R->check) {
      // ---- certificate scan (src/solver.cpp:297-317) ----
      cert_norms<RK>(P, R, g);
      if (!sync()) return;
      {
        const double* rg = region_ptr(P, kRegC1, g.nrec);
        block_totals(8, [&](int q) { return QSrc{rg, q, nullptr, 0, 0, false}; }, tot, g);
      }
      if (threadIdx.x == 0) {
        int any = 0;
        for (int c = 0; c < 4; ++c) {
          C.r.cn2[c] = sqrt(tot[c]);
          C.cfinite[c] = tot[4 + c] == 0.0;
          const bool normalized = c >= 2;
          C.r.cand_on[c] = (!normalized || C.last_k >= 1) && C.r.cn2[c] > 0.0 && C.cfinite[c];
          any |= C.r.cand_on[c];
        }
        if (!any) scan_logic(C, P->epochs, writer, s_time_up != 0);  // nothing to validate
      }
      __syncthreads();
      if (R->check) {
        cert_units<RK>(P, R, g);
        if (!sync()) return;
        {
          const double* rg = region_ptr(P, kRegC2, g.nrec);
          block_totals(12, [&](int q) { return QSrc{rg, q, nullptr, 0, 0, ((0x577u >> q) & 1u) != 0}; }, tot, g);
        }
        __shared__ int s_skip;  // candidates whose validation SpMV is skipped (bit c)
        if (threadIdx.x == 0) {
          C.cinf[0] = tot[0], C.cmax_u[0] = tot[1], C.cmax_negu[0] = tot[2], C.cdot[0] = tot[3];
          C.cinf[2] = tot[4], C.cmax_u[2] = tot[5], C.cmax_negu[2] = tot[6], C.cdot[2] = tot[7];
          C.cinf[1] = tot[8], C.cdot[1] = tot[9];
          C.cinf[3] = tot[10], C.cdot[3] = tot[11];
          // a candidate whose margin / sign tests already fail cannot pass
          // whatever its product: no SpMV for it (cert_may_pass)
          int skip = 0;
          for (int c = 0; c < 4; ++c)
            if (C.r.cand_on[c] && !cert_may_pass(C, c)) {
              C.r.cand_on[c] = 0;
              skip |= 1 << c;
            }
          s_skip = skip;
        }
        __syncthreads();
        const bool products = R->cand_on[0] || R->cand_on[1] || R->cand_on[2] || R->cand_on[3];
        if (products) {
          cert_products<RK, LM, EX>(P, R, stage, ++seq, g);
          if (!sync()) return;
          const double* rg = region_ptr(P, kRegC3, g.nrec);
          block_totals(6, [&](int q) { return QSrc{rg, q, nullptr, 0, 0, true}; }, tot, g);
        }
        if (threadIdx.x == 0) {
          if (products) {
            C.cmax_at[1] = tot[0], C.cmax_negat[1] = tot[1];
            C.cmax_at[3] = tot[2], C.cmax_negat[3] = tot[3];
            C.cmax_abs_au[0] = tot[4], C.cmax_abs_au[2] = tot[5];
          }
          // a skipped candidate's residual reads +inf: it fails as it would have
          const int sk = s_skip;
          if (sk & 2) C.cmax_at[1] = C.cmax_negat[1] = INFINITY;
          if (sk & 8) C.cmax_at[3] = C.cmax_negat[3] = INFINITY;
          if (sk & 1) C.cmax_abs_au[0] = INFINITY;
          if (sk & 4) C.cmax_abs_au[2] = INFINITY;
          scan_logic(C, P->epochs, writer, s_time_up != 0);
        }
        __syncthreads();
      }
    }
    spec_done = same_phase_a(*R, SR);
    bool synced = false;
    if constexpr (RK) {
      // a restart makes y+ the next y, but phase B pushed only the combo: push
      // this rank's rows of y+ now, and barrier before anyone reads them --
      // also when this launch ends here (the next launch starts with phase A)
      if (R->y_unpushed && !solo) {
        const double* yv = P->ypool + static_cast<size_t>(R->y_cur) * P->m;
        const size_t off = static_cast<size_t>(R->y_cur) * P->m;
        for (int i = P->T.row0 + g.cta * kThreads + threadIdx.x; i < P->T.row1; i += g.nctas * kThreads)
          push_peers(&P->T, P->T.py, off + i, ldcg(yv + i), __ldg(P->T.yneed + (i - P->T.row0)));
        if (!sync()) return;
        synced = true;
      }
      __syncthreads();  // every thread has read y_unpushed before it is cleared
      if (threadIdx.x == 0) C.r.y_unpushed = 0;
    }
    if (R->stop) break;
    // a redo reuses this parity's long-row counters: wait until every CTA's
    // speculative phase A is complete
    if (!spec_done && !synced && !sync()) return;
    mark(6);
  }
  if (prof && threadIdx.x == 0) {
    for (int k = 0; k < 6; ++k) prof[k] += pacc[k];
    prof[7] += pacc[6];
    for (int k = 0; k < 3; ++k) prof[8 + k] += pacc2[k];
    unsigned smid;
    asm volatile("mov.u32 %0, %%smid;" : "=r"(smid));
    prof[6] = smid;
  }
  if (threadIdx.x == 0) C.team_epochs = repoch;
  if (writer) ctl_store(C, P->ctl);
}

__global__ void __launch_bounds__(kThreads, kMinBlocks) loop_kernel(const __grid_constant__ KParams KP) {
  // constant bank; no local copy (grid_constant)
  const Geo g{static_cast<int>(blockIdx.x), static_cast<int>(gridDim.x), static_cast<int>(blockIdx.x),
              static_cast<int>(gridDim.x)};
  loop_body<false, false, 0, false, 0>(&KP, g);
}

// The same loop with the matrix streams loaded evict_first (working set
// beyond L2: Sched::stream_hint).
__global__ void __launch_bounds__(kThreads, kMinBlocks) loop_kernel_stream(const __grid_constant__ KParams KP) {
  const Geo g{static_cast<int>(blockIdx.x), static_cast<int>(gridDim.x), static_cast<int>(blockIdx.x),
              static_cast<int>(gridDim.x)};
  loop_body<false, false, 1, false, 0>(&KP, g);
}

// The reference summation order (hx_set_sum_order): every row one
// sequential chain; matrix-stream policy chosen at run time.
__global__ void __launch_bounds__(kThreads, kMinBlocks) loop_kernel_exact(const __grid_constant__ KParams KP) {
  const Geo g{static_cast<int>(blockIdx.x), static_cast<int>(gridDim.x), static_cast<int>(blockIdx.x),
              static_cast<int>(gridDim.x)};
  loop_body<false, false, 2, false, 1>(&KP, g);
}

// The trace-ring kernel (hx_setup with a trace period): traced iterations go
// to the device ring instead of pausing the launch.
__global__ void __launch_bounds__(kThreads, kMinBlocks) loop_kernel_trace(const __grid_constant__ KParams KP) {
  const Geo g{static_cast<int>(blockIdx.x), static_cast<int>(gridDim.x), static_cast<int>(blockIdx.x),
              static_cast<int>(gridDim.x)};
  loop_body<false, false, 2, false, 2, false, true>(&KP, g);
}

// The stream kernel with phase B swept in two column blocks (hx_upload_csr
// enables it when x+ is far larger than L2: configs[4]).
__global__ void __launch_bounds__(kThreads, kMinBlocks) loop_kernel_stream_cb(const __grid_constant__ KParams KP) {
  const Geo g{static_cast<int>(blockIdx.x), static_cast<int>(gridDim.x), static_cast<int>(blockIdx.x),
              static_cast<int>(gridDim.x)};
  loop_body<false, false, 1, true, 0>(&KP, g);
}

// The box form (hx_set_box) as its own kernel: the standard loop keeps its code.
__global__ void __launch_bounds__(kThreads, kMinBlocks) loop_kernel_box(const __grid_constant__ KParams KP) {
  const Geo g{static_cast<int>(blockIdx.x), static_cast<int>(gridDim.x), static_cast<int>(blockIdx.x),
              static_cast<int>(gridDim.x)};
  loop_body<false, true, 0>(&KP, g);
}

static_assert(sizeof(KParams) % 8 == 0, "KParams copied as 8-byte words");

// One launch runs every rank of `team` that lives on this device: CTAs
// [r * grp_ctas, (r + 1) * grp_ctas) are rank team[r].T.rank.  On a
// multi-GPU node each device launches its own rank (one group); on one
// device a whole team is emulated as groups of one cooperative launch (their
// CTAs wait on one another, so they must be co-resident -- never separate
// launches).
struct TeamLaunch {
  KParams p[kMaxRanks];  // the ranks of this launch (one on a multi-GPU node)
  int ranks, grp_ctas;
};
static_assert(sizeof(TeamLaunch) < 32000, "TeamLaunch must fit the kernel parameter space");

__global__ void __launch_bounds__(kThreads, kMinBlocks) loop_kernel_team(const __grid_constant__ TeamLaunch L) {
  // parameters stay in the constant bank (like loop_kernel), indexed by group
  const int group = blockIdx.x / L.grp_ctas;
  const KParams* P = &L.p[group];
  const int cta = blockIdx.x % L.grp_ctas;
  const Geo g{cta, L.grp_ctas, P->T.rank * L.grp_ctas + cta, P->T.nranks * L.grp_ctas};
  loop_body<true, false, 2>(P, g);
}

// The team loop with the matrix streams loaded evict_first at compile time
// (Sched::stream_hint: the rank's working set is beyond L2), like
// loop_kernel_stream -- the run-time policy choice costs ~2%.
__global__ void __launch_bounds__(kThreads, kMinBlocks) loop_kernel_team_stream(const __grid_constant__ TeamLaunch L) {
  const int group = blockIdx.x / L.grp_ctas;
  const KParams* P = &L.p[group];
  const int cta = blockIdx.x % L.grp_ctas;
  const Geo g{cta, L.grp_ctas, P->T.rank * L.grp_ctas + cta, P->T.nranks * L.grp_ctas};
  loop_body<true, false, 1>(P, g);
}

// The team's trace-ring loop.
__global__ void __launch_bounds__(kThreads, kMinBlocks) loop_kernel_team_trace(const __grid_constant__ TeamLaunch L) {
  const int group = blockIdx.x / L.grp_ctas;
  const KParams* P = &L.p[group];
  const int cta = blockIdx.x % L.grp_ctas;
  const Geo g{cta, L.grp_ctas, P->T.rank * L.grp_ctas + cta, P->T.nranks * L.grp_ctas};
  loop_body<true, false, 2, false, 2, false, true>(P, g);
}

// The team's setup modes (kModePower / kModeKkt / kModeScale), launched like
// loop_kernel_team.
__global__ void __launch_bounds__(kThreads, kMinBlocks) team_setup_kernel(const __grid_constant__ TeamLaunch L) {
  const int group = blockIdx.x / L.grp_ctas;
  const KParams* P = &L.p[group];
  const int cta = blockIdx.x % L.grp_ctas;
  const Geo g{cta, L.grp_ctas, P->T.rank * L.grp_ctas + cta, P->T.nranks * L.grp_ctas};
  loop_body<true, false, 2, false, 2, true>(P, g);
}

// ---------------------------------------------------------------------------
// Standalone kernels (setup, boundary SpMVs, results)
// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(kThreads, kMinBlocks) spmv_store_kernel(Sched S, const double* x, double* out) {
  extern __shared__ __align__(16) unsigned char dyn_smem[];
  double acc[1];
  acc_init<1, 0>(acc);
  EpiStore e{out};
  spmv_rows<1, 0>(S, 0, SrcVec{x}, e, acc, blockIdx.x * kWarps + (threadIdx.x >> 5), threadIdx.x & 31,
                  reinterpret_cast<WarpStage*>(dyn_smem) + (threadIdx.x >> 5));
}

__global__ void combine_kernel(int len, double w, const double* a, const double* b, double* out) {
  const double omw = 1.0 - w;
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < len; i += gridDim.x * blockDim.x)
    out[i] = omw * a[i] + w * b[i];
}

// make_certificate, src/solver.cpp:89-101: (s / ||raw||) * raw, raw rebuilt
// from the iterate buffers exactly as the scan formed it.
__global__ void cert_kernel(int len, int normalized, double scale, double factor, const double* p,
                            const double* q, double* out) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < len; i += gridDim.x * blockDim.x) {
    const double raw = normalized ? scale * (p[i] - q[i]) : q[i] - p[i];
    out[i] = factor * raw;
  }
}

// Fixed-order partial sums for the setup norms and kkt_current.
__global__ void __launch_bounds__(kThreads, kMinBlocks)
kkt_partials_kernel(int m, int n, const double* ax, const double* b, const double* aty,
                    const double* c, const double* x, const double* y, double* slots, const double* ub = nullptr) {
  double acc[7];
  acc_init<7, 0>(acc);
  const int gtid = blockIdx.x * kThreads + threadIdx.x, gs = gridDim.x * kThreads;
  for (int i = gtid; i < m; i += gs) {
    const double bi = b[i];
    if (ax) {
      const double d = ax[i] - bi;
      acc[0] += d * d;
      acc[3] += bi * y[i];
    }
    acc[4] += bi * bi;
  }
  for (int j = gtid; j < n; j += gs) {
    const double cj = c[j];
    if (aty) {
      double r = -(cj + aty[j]);
      r = r < 0.0 ? 0.0 : r;
      const double u = ub ? ub[j] : INFINITY;  // box form: bounded columns enter the dual objective
      if (u < INFINITY) acc[6] += u * r;
      else acc[1] += r * r;
      acc[2] += cj * x[j];
    }
    acc[5] += cj * cj;
  }
  block_to_slots<7, 0>(acc, slots, gridDim.x);
}

// Trace diagnostics (src/solver.cpp:283-287): sums of the normalized
// candidate s (z - anchor) with its product s (a_x - a_x_anchor):
// ||dx||^2, ||dy||^2, dy . d(Ax), each term rounded as the reference forms it.
__global__ void __launch_bounds__(kThreads, kMinBlocks)
cand_norm_kernel(int m, int n, double s, const double* zx, const double* xa, const double* y, const double* ya,
                 const double* ax, const double* axa, double* slots) {
  double acc[3];
  acc_init<3, 0>(acc);
  const int gtid = blockIdx.x * kThreads + threadIdx.x, gs = gridDim.x * kThreads;
  for (int j = gtid; j < n; j += gs) {
    const double d = s * (zx[j] - xa[j]);
    acc[0] += d * d;
  }
  for (int i = gtid; i < m; i += gs) {
    const double dy = s * (y[i] - ya[i]);
    const double da = s * (ax[i] - axa[i]);
    acc[1] += dy * dy;
    acc[2] += dy * da;
  }
  block_to_slots<3, 0>(acc, slots, gridDim.x);
}

__global__ void final_reduce_kernel(const double* region, int grid, int q_count, double* out) {
  const int wq = threadIdx.x >> 5;
  for (int q = wq; q < q_count; q += blockDim.x / 32) {
    const double t = warp_reduce_strided(region + q, grid, kMaxQ, false);  // replica 0
    if ((threadIdx.x & 31) == 0) out[q] = t;
  }
}

// Device-side CSR validation (src/sparse_matrix.cpp:27-53): flags
// 1 out-of-range column, 2 non-finite value, 4 unsorted row, 8 duplicate,
// 16 non-monotone row pointer.
__global__ void validate_kernel(int m, int n, const long long* rp, const int* ci, const double* v,
                                unsigned* flags) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < m; i += gridDim.x * blockDim.x) {
    const long long p0 = rp[i], p1 = rp[i + 1];
    unsigned f = 0;
    if (p1 < p0) f |= 16u;
    for (long long p = p0; p < p1; ++p) {
      const int col = ci[p];
      if (col < 0 || col >= n) f |= 1u;
      if (!isfinite(v[p])) f |= 2u;
      if (p > p0) {
        if (col < ci[p - 1]) f |= 4u;
        if (col == ci[p - 1]) f |= 8u;
      }
    }
    if (f) atomicOr(flags, f);
  }
}

// The bank-staggered copy of a CSR matrix (build_schedule's stagger), one
// warp per row: row r's entries at pptr[r], then its pad slots up to
// pptr[r + 1] with value 0 and the column of the row's last entry (the lane
// before a pad gathers the same line, so a pad costs no extra wavefront);
// an empty row's pads take the next row's first column.
__global__ void pad_copy_kernel(int rows, const int* ptr, const int* idx, const double* val, const int* pptr,
                                int* pidx, double* pval) {
  const int lane = threadIdx.x & 31;
  const int nnz = ptr[rows];
  for (int r = (blockIdx.x * blockDim.x + threadIdx.x) >> 5; r < rows; r += (gridDim.x * blockDim.x) >> 5) {
    const int a = ptr[r], e = ptr[r + 1], pa = pptr[r], pe = pptr[r + 1];
    for (int k = lane; k < e - a; k += 32) {
      pidx[pa + k] = idx[a + k];
      pval[pa + k] = val[a + k];
    }
    const int fill = e > a ? idx[e - 1] : e < nnz ? idx[e] : 0;
    for (int k = pa + (e - a) + lane; k < pe; k += 32) {
      pidx[k] = fill;
      pval[k] = 0.0;
    }
  }
}

__global__ void narrow_ptr_kernel(int len, const long long* src, int* dst) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < len; i += gridDim.x * blockDim.x)
    dst[i] = static_cast<int>(src[i]);
}

__global__ void row_of_kernel(int m, const int* rp, int* row_of, int* iota) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < m; i += gridDim.x * blockDim.x)
    for (int p = rp[i]; p < rp[i + 1]; ++p) {
      row_of[p] = i;
      iota[p] = p;
    }
}

// Column blocks of A (column-blocked phase B): per row, the split point in
// its ascending columns, then the two halves copied to their CSR arrays (one
// warp per row).  cnt0 / cnt1 have m + 1 entries, [0] = 0, so an inclusive
// scan gives the row pointers.
// Column blocks of A (phase B of loop_kernel_stream_cb): block k holds the
// columns [split[k - 1], split[k]) (split[-1] = 0, split[K - 1] = n), rows
// kept whole and ascending inside each block.
struct ColSplit {
  int K;
  int split[kMaxColBlocks];  // exclusive upper column of each block
  int* cnt[kMaxColBlocks];   // per row counts at [i + 1] (inclusive-scanned into the block's row pointers)
  const int* ptr[kMaxColBlocks];
  int* idx[kMaxColBlocks];
  double* val[kMaxColBlocks];
};

__global__ void split_count_kernel(int m, const int* ptr, const int* idx, ColSplit sp) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < m; i += gridDim.x * blockDim.x) {
    const int lo = ptr[i], hi = ptr[i + 1];
    int prev = lo;
    for (int k = 0; k < sp.K; ++k) {
      int a = prev, b = hi;
      if (k + 1 < sp.K) {
        while (a < b) {
          const int mid = (a + b) >> 1;
          if (idx[mid] < sp.split[k]) a = mid + 1;
          else b = mid;
        }
      } else {
        a = hi;
      }
      sp.cnt[k][i + 1] = a - prev;
      prev = a;
    }
  }
}

__global__ void split_copy_kernel(int m, const int* ptr, const int* idx, const double* val, ColSplit sp) {
  const int lane = threadIdx.x & 31;
  for (int i = (blockIdx.x * blockDim.x + threadIdx.x) >> 5; i < m; i += (gridDim.x * blockDim.x) >> 5) {
    const int a = ptr[i], len = ptr[i + 1] - a;
    for (int q = lane; q < len; q += 32) {
      const int col = idx[a + q];
      int k = 0, before = 0;  // block of this entry, entries of the row in earlier blocks
      while (k + 1 < sp.K && col >= sp.split[k]) {
        before += sp.ptr[k][i + 1] - sp.ptr[k][i];
        ++k;
      }
      const int o = sp.ptr[k][i] + q - before;
      sp.idx[k][o] = col;
      sp.val[k][o] = val[a + q];
    }
  }
}

__global__ void col_count_kernel(int nnz, const int* ci, int* count) {
  for (int p = blockIdx.x * blockDim.x + threadIdx.x; p < nnz; p += gridDim.x * blockDim.x)
    atomicAdd(count + ci[p], 1);
}

__global__ void gather_t_kernel(int nnz, const int* perm, const int* row_of, const double* val, int* t_idx,
                                double* t_val) {
  for (int k = blockIdx.x * blockDim.x + threadIdx.x; k < nnz; k += gridDim.x * blockDim.x) {
    const int p = perm[k];
    t_idx[k] = row_of[p];
    t_val[k] = val[p];
  }
}

// ---------------------------------------------------------------------------
// Diagonal preconditioning (Ruiz equilibration + Pock-Chambolle), an instance
// transform A' = R A C, b' = R b, c' = C c applied to both stored copies with
// identical rounding ((a * r_i) * c_j).  Setup-time kernels, thread per row.
// ---------------------------------------------------------------------------
// kind 0: max |a_ij| over the row, kind 1: sum |a_ij|^p (p = 2 - alpha for
// rows of A, alpha for rows of A^T, passed as `power`).
__global__ void row_norm_kernel(int rows, const int* rp, const double* v, int kind, double power, double* out) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < rows; i += gridDim.x * blockDim.x) {
    double acc = 0.0;
    for (int p = rp[i]; p < rp[i + 1]; ++p) {
      const double a = fabs(v[p]);
      if (kind == 0) acc = a > acc ? a : acc;
      else acc += power == 1.0 ? a : pow(a, power);
    }
    out[i] = acc;
  }
}

// d = 1/sqrt(norm) (1 where the norm is 0); acc *= d.
__global__ void inv_sqrt_kernel(int len, double* d, double* acc) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < len; i += gridDim.x * blockDim.x) {
    const double nrm = d[i];
    const double f = nrm > 0.0 ? 1.0 / sqrt(nrm) : 1.0;
    d[i] = f;
    acc[i] = acc[i] * f;
  }
}

// val(row i, col j) = (val * dr[i]) * dc[j]; `transposed` swaps the roles.
__global__ void scale_csr_kernel(int rows, const int* rp, const int* ci, double* v, const double* d_row,
                                 const double* d_col, int transposed) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < rows; i += gridDim.x * blockDim.x)
    for (int p = rp[i]; p < rp[i + 1]; ++p) {
      const int j = ci[p];
      v[p] = transposed ? (v[p] * d_row[j]) * d_col[i] : (v[p] * d_row[i]) * d_col[j];
    }
}

__global__ void div_vec_kernel(int len, double* v, const double* d) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < len; i += gridDim.x * blockDim.x) v[i] /= d[i];
}

__global__ void scale_vec_kernel(int len, double* v, const double* d) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < len; i += gridDim.x * blockDim.x) v[i] = v[i] * d[i];
}

}  // namespace hx

// ===========================================================================
// Host side
// ===========================================================================
using namespace hx;

namespace {

constexpr int kProfWords = 16 + 2 * kWarps;  // per CTA: phase timers + per-warp SpMV timers

struct DevSched {
  int4* tasks = nullptr;
  int4* meta = nullptr;
  double* part = nullptr;    // 4 * n_slots
  unsigned* cnt = nullptr;   // 4 * n_long
  double* terms = nullptr;   // 4 * n_long * kMaxQ
  int* owned_ptr = nullptr;
  int* owned_idx = nullptr;
  unsigned long long* flags = nullptr;  // 4 * n_long
  // bank-staggered copy of the matrix the tasks index (SchedHost::pptr);
  // null: the view reads the CSR arrays themselves
  int* pptr = nullptr;
  int* pidx = nullptr;
  double* pval = nullptr;
  Sched view;
  double max_cost = 0, mean_cost = 0;
};

}  // namespace

struct hx_ctx {
  int device = 0;
  cudaStream_t stream = nullptr;
  cudaEvent_t ev0 = nullptr, ev1 = nullptr;
  int sm_count = 0;
  int grid = 0;
  std::string err;
  int64_t m = 0, n = 0, nnz = 0;
  int64_t nnz_a = 0, nnz_t = 0;  // nonzeros this context stores of A and A^T (a rank: its blocks)
  bool uploaded = false, setup_done = false;
  int sum_order = 0;  // hx_set_sum_order: 1 = the reference's sequential row sums
  int64_t launches = 0;
  // device data
  int* a_ptr = nullptr;
  int* a_idx = nullptr;
  double* a_val = nullptr;
  int* t_ptr = nullptr;
  int* t_idx = nullptr;
  double* t_val = nullptr;
  double* b = nullptr;
  double* c = nullptr;
  DevSched sa, st;
  // column-blocked phase B (loop_kernel_stream_cb): A's leading / trailing
  // column blocks as CSR with their schedules, and the leading block's row sums
  int colblock = 0;  // column blocks of phase B (0: none)
  int* cb_ptr[kMaxColBlocks] = {};
  int* cb_idx[kMaxColBlocks] = {};
  double* cb_val[kMaxColBlocks] = {};
  DevSched sb[kMaxColBlocks];
  double* bpart = nullptr;
  double* xpool = nullptr;
  double* ypool = nullptr;
  double* axpool = nullptr;
  double* upool = nullptr;
  double* xavg = nullptr;  // baseline schemes: kAvgPool slots (allocated at hx_setup)
  double* tavg = nullptr;
  double* yavg = nullptr;
  double* aavg = nullptr;
  double* xbar = nullptr;
  double* ub = nullptr;  // box form: column upper bounds (hx_set_box)
  double* slots = nullptr;
  double* scratch = nullptr;  // kMaxQ doubles
  Ctl* ctl = nullptr;
  GridBar* bar = nullptr;
  KParams* kparams = nullptr;
  unsigned long long* prof = nullptr;  // HX_PROFILE=1: per-CTA phase timers
  hplp_epoch_t* epochs = nullptr;
  Ctl h;  // host mirror
  double b_norm = 0, c_norm = 0;
  double b_sq = 0, u_sq = 0;  // ||b||^2 of the device problem; box form: sum of finite u_j^2
  double time_limit_s = 0, loop_elapsed_s = 0;  // SolverConfig::time_limit_seconds budget of the loop
  // Row-partitioned team (hx_set_partition / hx_team_*).  The
  // context keeps the full problem (setup kernels, power iteration and the
  // boundary SpMVs run on it unchanged -- every rank computes the same
  // values); the loop kernel runs the partition schedules pa / pt.
  bool ranked = false;
  Team team{};                       // own range + every rank's buffers
  int pcol0[kMaxRanks] = {}, pcol1[kMaxRanks] = {};  // every rank's column block (result assembly)
  int prow0[kMaxRanks] = {}, prow1[kMaxRanks] = {};  // every rank's row block
  DevSched pa, pt;                   // rows [row0,row1) of A, [col0,col1) of A^T
  RankBar* rbar = nullptr;
  unsigned char* xneed = nullptr;    // masks of Team::xneed / yneed (device)
  unsigned char* yneed = nullptr;
  unsigned long long team_epochs = 0;
  std::vector<hx_ctx*> local_team;   // ranks launched together (same device), rank order
  std::vector<void*> ipc_open;       // peer mappings to close
  // trace ring (KParams::ring_*): one allocation, ring_layout(); a rank's is
  // CUDA-IPC memory (peers' mappings in peer_ring, own included)
  unsigned char* ring = nullptr;
  int ring_cap = 0;
  unsigned char* peer_ring[kMaxRanks] = {};
  double r_tol = 0.0, tol_active = 0.0;
};

namespace {
// Trace ring layout: cap slots of z.x (n doubles), z.y (m doubles), classes
// (n bytes), then cap records.  Capacity from a memory budget
// (HPLP_TRACE_RING_MB, default 256 MB), 2..1024 slots.
struct RingLayout {
  size_t x, y, cls, rec, bytes;
};
RingLayout ring_layout(int cap, int64_t n, int64_t m) {
  RingLayout L{};
  L.x = 0;
  L.y = L.x + static_cast<size_t>(cap) * n * sizeof(double);
  L.cls = L.y + static_cast<size_t>(cap) * m * sizeof(double);
  L.rec = (L.cls + static_cast<size_t>(cap) * n + 15) & ~size_t{15};
  L.bytes = L.rec + static_cast<size_t>(cap) * sizeof(TraceRec);
  return L;
}
int ring_capacity(int64_t n, int64_t m) {
  double mb = 256.0;
  if (const char* e = std::getenv("HPLP_TRACE_RING_MB")) mb = std::atof(e);
  const double per = 8.0 * static_cast<double>(n + m) + static_cast<double>(n) + sizeof(TraceRec);
  const double cap = mb * 1048576.0 / std::max(per, 1.0);
  return static_cast<int>(std::max(2.0, std::min(1024.0, cap)));
}
}  // namespace

namespace {

thread_local std::string g_create_err;

int set_err(hx_ctx* ctx, int code, const std::string& msg) {
  if (ctx) ctx->err = msg;
  else g_create_err = msg;
  return code;
}

#define HX_CUDA(ctx, expr)                                                                    \
  do {                                                                                        \
    cudaError_t e_ = (expr);                                                                  \
    if (e_ != cudaSuccess)                                                                    \
      return set_err(ctx, e_ == cudaErrorMemoryAllocation ? HPLP_ENOMEM : HPLP_ECUDA,         \
                     std::string(#expr) + ": " + cudaGetErrorString(e_));                     \
  } while (0)

// Device memory comes from the device's stream-ordered pool with an
// unlimited release threshold, so repeated solves reuse memory instead of
// mapping and unmapping it: plain cudaMalloc / cudaFree of the ~100 MB a
// configs[1] problem needs took 0.03-0.5 s per call on the B200 boxes, more
// than the solve.  Buffers peers map through CUDA IPC must be cudaMalloc
// memory (dalloc_ipc); dfree tells them apart.
std::mutex g_mem_mu;
std::unordered_set<void*> g_ipc_blocks;
std::unordered_set<int> g_pool_ready;

cudaError_t pool_ready() {
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return e;
  std::lock_guard<std::mutex> lk(g_mem_mu);
  if (g_pool_ready.count(dev)) return cudaSuccess;
  cudaMemPool_t pool;
  e = cudaDeviceGetDefaultMemPool(&pool, dev);
  if (e != cudaSuccess) return e;
  uint64_t keep = ~uint64_t{0};
  e = cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &keep);
  if (e == cudaSuccess) g_pool_ready.insert(dev);
  return e;
}

template <typename T>
cudaError_t dalloc(T** p, size_t count) {
  cudaError_t e = pool_ready();
  if (e != cudaSuccess) return e;
  e = cudaMallocAsync(reinterpret_cast<void**>(p), std::max<size_t>(count, 1) * sizeof(T), 0);
  return e != cudaSuccess ? e : cudaStreamSynchronize(0);
}

template <typename T>
cudaError_t dalloc_ipc(T** p, size_t count) {
  cudaError_t e = cudaMalloc(reinterpret_cast<void**>(p), std::max<size_t>(count, 1) * sizeof(T));
  if (e == cudaSuccess) {
    std::lock_guard<std::mutex> lk(g_mem_mu);
    g_ipc_blocks.insert(*p);
  }
  return e;
}

// Callers free only memory no pending work uses (the context's stream is
// synchronized first).
void dfree(void* p) {
  if (!p) return;
  bool ipc;
  {
    std::lock_guard<std::mutex> lk(g_mem_mu);
    ipc = g_ipc_blocks.erase(p) > 0;
  }
  if (ipc) cudaFree(p);
  else cudaFreeAsync(p, 0);
}

// Frees a device temporary when the scope ends (error returns included).
struct DevFree {
  void** p;
  ~DevFree() {
    if (*p) dfree(*p);
    *p = nullptr;
  }
};

void free_sched(DevSched& s) {
  dfree(s.tasks), dfree(s.meta), dfree(s.owned_ptr), dfree(s.owned_idx), dfree(s.flags);
  dfree(s.part), dfree(s.cnt), dfree(s.terms);
  dfree(s.pptr), dfree(s.pidx), dfree(s.pval);
  s = DevSched{};
}

void free_problem(hx_ctx* c) {
  if (c->stream) cudaStreamSynchronize(c->stream);
  dfree(c->a_ptr), dfree(c->a_idx), dfree(c->a_val), dfree(c->t_ptr), dfree(c->t_idx), dfree(c->t_val);
  dfree(c->b), dfree(c->c), dfree(c->xpool), dfree(c->ypool), dfree(c->axpool), dfree(c->upool);
  dfree(c->xavg), dfree(c->tavg), dfree(c->yavg), dfree(c->aavg), dfree(c->xbar), dfree(c->ub);
  c->xavg = c->tavg = c->yavg = c->aavg = c->xbar = c->ub = nullptr;
  free_sched(c->sa);
  free_sched(c->st);
  free_sched(c->pa);
  free_sched(c->pt);
  for (int k = 0; k < kMaxColBlocks; ++k) {
    free_sched(c->sb[k]);
    dfree(c->cb_ptr[k]), dfree(c->cb_idx[k]), dfree(c->cb_val[k]);
    c->cb_ptr[k] = c->cb_idx[k] = nullptr;
    c->cb_val[k] = nullptr;
  }

  dfree(c->bpart);
  c->bpart = nullptr;
  dfree(c->ring);
  c->ring = nullptr;
  c->ring_cap = 0;
  c->colblock = 0;
  c->a_ptr = c->a_idx = c->t_ptr = c->t_idx = nullptr;
  c->a_val = c->t_val = c->b = c->c = c->xpool = c->ypool = c->axpool = c->upool = nullptr;
  c->uploaded = c->setup_done = false;
}

// Schedule of rows [row0, row0 + rows) of a CSR matrix (the whole matrix by
// default; a rank's block in a team), built on the host (h) and uploaded.
// Task rows stay global indices.
int upload_built_sched(hx_ctx* ctx, DevSched& d, SchedHost h, int rows, int cols, const int* dptr, const int* didx,
                       const double* dval, int row0) {
  if (row0)
    for (int4& t : h.tasks)
      if (t.x != t.y || t.z != t.w) {
        const int kind = task_kind(t.y);
        t.x += row0;
        t.y = task_y((t.y & kRowMask) + row0, kind);
      }
  HX_CUDA(ctx, dalloc(&d.tasks, h.tasks.size()));
  HX_CUDA(ctx, dalloc(&d.meta, h.meta.size()));
  HX_CUDA(ctx, dalloc(&d.part, 4 * static_cast<size_t>(h.n_slots)));
  HX_CUDA(ctx, dalloc(&d.cnt, 4 * static_cast<size_t>(h.n_long)));
  HX_CUDA(ctx, dalloc(&d.terms, 4 * static_cast<size_t>(h.n_long) * kMaxQ));
  HX_CUDA(ctx, dalloc(&d.owned_ptr, h.owned_ptr.size()));
  HX_CUDA(ctx, dalloc(&d.owned_idx, h.owned_idx.size()));
  HX_CUDA(ctx, dalloc(&d.flags, 4 * static_cast<size_t>(h.n_long)));
  auto cp = [&](void* dst, const void* src, size_t bytes) {
    return bytes ? cudaMemcpyAsync(dst, src, bytes, cudaMemcpyHostToDevice, ctx->stream) : cudaSuccess;
  };
  HX_CUDA(ctx, cp(d.tasks, h.tasks.data(), h.tasks.size() * sizeof(int4)));
  HX_CUDA(ctx, cp(d.owned_ptr, h.owned_ptr.data(), h.owned_ptr.size() * sizeof(int)));
  HX_CUDA(ctx, cp(d.owned_idx, h.owned_idx.data(), h.owned_idx.size() * sizeof(int)));
  HX_CUDA(ctx, cp(d.meta, h.meta.data(), h.meta.size() * sizeof(int4)));
  HX_CUDA(ctx, cudaMemsetAsync(d.cnt, 0, std::max<size_t>(1, 4 * static_cast<size_t>(h.n_long)) * sizeof(unsigned),
                               ctx->stream));
  if (!h.pptr.empty()) {
    // the staggered copy: row r's entries at pptr[r], its trailing pads zero
    const int64_t pn = h.padded_nnz;
    HX_CUDA(ctx, dalloc(&d.pptr, h.pptr.size()));
    HX_CUDA(ctx, dalloc(&d.pidx, pn + kMatrixPad));
    HX_CUDA(ctx, dalloc(&d.pval, pn + kMatrixPad));
    HX_CUDA(ctx, cp(d.pptr, h.pptr.data(), h.pptr.size() * sizeof(int)));
    HX_CUDA(ctx, cudaMemsetAsync(d.pidx, 0, (pn + kMatrixPad) * sizeof(int), ctx->stream));
    HX_CUDA(ctx, cudaMemsetAsync(d.pval, 0, (pn + kMatrixPad) * sizeof(double), ctx->stream));
    pad_copy_kernel<<<4 * ctx->sm_count, 256, 0, ctx->stream>>>(rows, dptr, didx, dval, d.pptr, d.pidx, d.pval);
    HX_CUDA(ctx, cudaGetLastError());
    ctx->launches += 1;
    dptr = d.pptr;
    didx = d.pidx;
    dval = d.pval;
  }
  HX_CUDA(ctx, cudaStreamSynchronize(ctx->stream));  // host vectors go out of scope
  Sched& v = d.view;
  v.rows = rows;
  v.cols = cols;
  v.W = ctx->grid * kWarps;
  v.ptr = dptr;
  v.idx = didx;
  v.val = dval;
  v.tasks = d.tasks;
  v.n_tasks = static_cast<int>(h.tasks.size());
  v.meta = d.meta;
  v.n_long = h.n_long;
  v.part_base = d.part;
  v.cnt_base = d.cnt;
  v.terms_base = d.terms;
  v.n_slots = h.n_slots;
  v.owned_ptr = d.owned_ptr;
  v.owned_idx = d.owned_idx;
  v.flag_base = d.flags;
  d.max_cost = h.max_warp_cost;
  d.mean_cost = h.mean_warp_cost;
  return HPLP_OK;
}

// HX_COSTS="rowT,taskT,rowA,taskA": schedule cost constants for the rows of
// A^T (phase A) and of A (phase B), in nnz units (experiments)
void sched_costs(bool transposed, double& row_cost, double& task_cost) {
  row_cost = kRowCost, task_cost = kTaskCost;
  if (const char* e = std::getenv("HX_COSTS")) {
    double v[4] = {kRowCost, kTaskCost, kRowCost, kTaskCost};
    std::sscanf(e, "%lf,%lf,%lf,%lf", &v[0], &v[1], &v[2], &v[3]);
    row_cost = transposed ? v[0] : v[2];
    task_cost = transposed ? v[1] : v[3];
  }
}

int upload_sched(hx_ctx* ctx, DevSched& d, const int* ptr_host, int rows, int cols, const int* dptr,
                 const int* didx, const double* dval, double lead = 0.0, int row0 = 0, bool transposed = false) {
  double rc, tc;
  sched_costs(transposed, rc, tc);
  return upload_built_sched(ctx, d,
                            build_schedule(ptr_host + row0, rows, ctx->grid * kWarps, lead, rc, tc, ctx->sum_order == 1),
                            rows, cols, dptr, didx, dval, row0);
}

KParams params(hx_ctx* c) {
  KParams P{};
  P.A = c->sa.view;
  P.AT = c->st.view;
  P.m = static_cast<int>(c->m);
  P.n = static_cast<int>(c->n);
  P.b = c->b;
  P.c = c->c;
  P.xpool = c->xpool;
  P.ypool = c->ypool;
  P.axpool = c->axpool;
  P.upool = c->upool;
  P.slots = c->slots;
  P.ub = c->ub;
  P.ctl = c->ctl;
  P.bar = c->bar;
  P.epochs = c->epochs;
  P.prof = c->prof;
  P.xavg = c->xavg, P.tavg = c->tavg, P.yavg = c->yavg, P.aavg = c->aavg, P.xbar = c->xbar;
  for (int k = 0; k < c->colblock; ++k) P.cbs[k] = c->sb[k].view;
  P.ncb = c->colblock;
  P.bpart = c->bpart;
  if (c->ring) {
    const RingLayout L = ring_layout(c->ring_cap, c->n, c->m);
    P.ring_x = reinterpret_cast<double*>(c->ring + L.x);
    P.ring_y = reinterpret_cast<double*>(c->ring + L.y);
    P.ring_cls = c->ring + L.cls;
    P.ring_rec = reinterpret_cast<TraceRec*>(c->ring + L.rec);
  }
  P.r_tol = c->r_tol;
  P.tol_active = c->tol_active;
  return P;
}

int launch_loop(hx_ctx* c) {
  KParams P = params(c);
  void* args[] = {&P};
  HX_CUDA(c, cudaMemcpyAsync(c->ctl, &c->h, sizeof(Ctl), cudaMemcpyHostToDevice, c->stream));
  HX_CUDA(c, cudaMemsetAsync(c->bar, 0, sizeof(GridBar), c->stream));
  for (int k = -2; k < c->colblock; ++k) {  // long-row flags restart with the per-launch sequence
    const DevSched* d = k == -2 ? &c->sa : k == -1 ? &c->st : &c->sb[k];
    if (d->view.n_long)
      HX_CUDA(c, cudaMemsetAsync(d->flags, 0, 4 * static_cast<size_t>(d->view.n_long) * sizeof(unsigned long long),
                                 c->stream));
  }
  const void* kernel = c->h.mode == kModeLoop && c->h.scheme != HPLP_SCHEME_RHPDHG
                           ? reinterpret_cast<const void*>(loop_kernel_baseline)
                           : c->ub                     ? reinterpret_cast<const void*>(loop_kernel_box)
                           : c->h.ring_cap > 0 && c->h.mode == kModeLoop ? reinterpret_cast<const void*>(loop_kernel_trace)
                           : c->sum_order == HX_SUM_REFERENCE ? reinterpret_cast<const void*>(loop_kernel_exact)
                           : c->sa.view.stream_hint && c->colblock && c->h.mode == kModeLoop
                               ? reinterpret_cast<const void*>(loop_kernel_stream_cb)
                           : c->sa.view.stream_hint    ? reinterpret_cast<const void*>(loop_kernel_stream)
                                                       : reinterpret_cast<const void*>(loop_kernel);
  HX_CUDA(c, cudaLaunchCooperativeKernel(kernel, dim3(c->grid), dim3(kThreads), args, kStageBytes, c->stream));
  c->launches += 1;
  HX_CUDA(c, cudaMemcpyAsync(&c->h, c->ctl, sizeof(Ctl), cudaMemcpyDeviceToHost, c->stream));
  GridBar gb;
  HX_CUDA(c, cudaMemcpyAsync(&gb, c->bar, sizeof(GridBar), cudaMemcpyDeviceToHost, c->stream));
  HX_CUDA(c, cudaStreamSynchronize(c->stream));
  HX_CUDA(c, cudaGetLastError());
  if (gb.abort) {
    return set_err(c, HPLP_ETIMEOUT, "hx: grid barrier watchdog fired (device hang avoided)");
  }
  return HPLP_OK;
}

// ---- row-partitioned team ---------------------------------------------------
// Launch parameters of one rank: its partition schedules plus the team.
KParams team_params(hx_ctx* c) {
  KParams P = params(c);
  P.A = c->pa.view;
  P.AT = c->pt.view;
  P.prof = nullptr;
  P.T = c->team;
  if (c->h.ring_cap > 0) P.T.prereduce = 0;  // the trace totals need every rank's records
  return P;
}

// Issue one loop launch for the ranks of `ranks` that share a device (rank
// order): a single cooperative launch of ranks.size() * grid CTAs on the
// first rank's stream.  No host wait here (device-to-pageable copies block,
// so they wait for team_complete): a process driving several devices issues
// every device's launch before any rank can stall on a peer.
int team_issue(const std::vector<hx_ctx*>& ranks, std::vector<KParams>& hp) {
  hx_ctx* lead = ranks.front();
  cudaStream_t s = lead->stream;
  HX_CUDA(lead, cudaSetDevice(lead->device));
  hp.clear();
  for (hx_ctx* c : ranks) {
    hp.push_back(team_params(c));
    c->h.team_epochs = c->team_epochs;
    HX_CUDA(lead, cudaMemcpyAsync(c->ctl, &c->h, sizeof(Ctl), cudaMemcpyHostToDevice, s));
    HX_CUDA(lead, cudaMemsetAsync(c->bar, 0, sizeof(GridBar), s));
    for (DevSched* d : {&c->pa, &c->pt})
      if (d->view.n_long)
        HX_CUDA(lead, cudaMemsetAsync(d->flags, 0, 4 * static_cast<size_t>(d->view.n_long) * sizeof(unsigned long long),
                                      s));
  }
  static_assert(std::is_trivially_copyable<TeamLaunch>::value, "TeamLaunch");
  auto tl = std::make_unique<TeamLaunch>();
  std::memset(tl.get(), 0, sizeof(TeamLaunch));
  for (size_t i = 0; i < hp.size(); ++i) tl->p[i] = hp[i];
  tl->ranks = static_cast<int>(hp.size());
  tl->grp_ctas = lead->grid;
  void* args[] = {tl.get()};
  bool stream = true;  // every rank of the launch streams its blocks evict_first
  for (hx_ctx* c : ranks) stream = stream && c->pa.view.stream_hint && c->pt.view.stream_hint;
  const void* kernel = lead->h.mode != kModeLoop ? reinterpret_cast<const void*>(team_setup_kernel)
                      : lead->h.ring_cap > 0   ? reinterpret_cast<const void*>(loop_kernel_team_trace)
                      : stream                 ? reinterpret_cast<const void*>(loop_kernel_team_stream)
                                               : reinterpret_cast<const void*>(loop_kernel_team);
  HX_CUDA(lead, cudaLaunchCooperativeKernel(kernel,
                                            dim3(static_cast<unsigned>(lead->grid * ranks.size())), dim3(kThreads),
                                            args, kStageBytes, s));
  lead->launches += 1;
  return HPLP_OK;
}

int team_complete(const std::vector<hx_ctx*>& ranks) {
  hx_ctx* lead = ranks.front();
  HX_CUDA(lead, cudaSetDevice(lead->device));
  std::vector<GridBar> gb(ranks.size());
  for (size_t i = 0; i < ranks.size(); ++i) {
    HX_CUDA(lead, cudaMemcpyAsync(&ranks[i]->h, ranks[i]->ctl, sizeof(Ctl), cudaMemcpyDeviceToHost, lead->stream));
    HX_CUDA(lead, cudaMemcpyAsync(&gb[i], ranks[i]->bar, sizeof(GridBar), cudaMemcpyDeviceToHost, lead->stream));
  }
  HX_CUDA(lead, cudaStreamSynchronize(lead->stream));
  HX_CUDA(lead, cudaGetLastError());
  bool aborted = false;
  for (size_t i = 0; i < ranks.size(); ++i) {
    ranks[i]->team_epochs = ranks[i]->h.team_epochs;
    aborted |= gb[i].abort != 0;
  }
  if (aborted) {
    for (hx_ctx* c : ranks) c->team.nranks = 0;  // barrier words out of step: the team is unusable
    return set_err(lead, HPLP_ETIMEOUT, "hx: team barrier watchdog fired (a rank stalled; device hang avoided)");
  }
  return HPLP_OK;
}

// One loop launch of a whole team known to this process, grouped by device.
int team_launch(const std::vector<hx_ctx*>& all) {
  std::vector<std::vector<hx_ctx*>> groups;
  for (hx_ctx* c : all) {
    bool placed = false;
    for (auto& g : groups)
      if (g.front()->device == c->device) {
        g.push_back(c);
        placed = true;
      }
    if (!placed) groups.push_back({c});
  }
  std::vector<std::vector<KParams>> hp(groups.size());
  int rc = HPLP_OK;
  size_t issued = 0;
  for (; issued < groups.size() && rc == HPLP_OK; ++issued) rc = team_issue(groups[issued], hp[issued]);
  for (size_t k = 0; k < issued; ++k) {
    const int r2 = team_complete(groups[k]);
    if (rc == HPLP_OK) rc = r2;
    if (r2 != HPLP_OK)
      for (hx_ctx* c : all) c->err = groups[k].front()->err;
  }
  return rc;
}

// Result assembly: the x pool vector `role` holds valid values only on each
// rank's own column block (x+ and everything formed from it are pushed to
// every rank, the x formed in phase A is not); copy the peers' blocks in.
int assemble_x(hx_ctx* c, int role) {
  if (!c->ranked || role < 0) return HPLP_OK;
  for (int r = 0; r < c->team.nranks; ++r) {
    const int64_t len = c->pcol1[r] - c->pcol0[r];
    if (r == c->team.rank || len <= 0) continue;
    const size_t off = static_cast<size_t>(role) * c->n + c->pcol0[r];
    HX_CUDA(c, cudaMemcpyAsync(c->xpool + off, c->team.px[r] + off, len * sizeof(double), cudaMemcpyDefault,
                               c->stream));
  }
  return HPLP_OK;
}

// The same for a y pool vector: y+ is pushed to the peers only on restarts,
// so a y+ role read back for results is assembled from the peers' rows.
int assemble_y(hx_ctx* c, int role) {
  if (!c->ranked || role < 0) return HPLP_OK;
  for (int r = 0; r < c->team.nranks; ++r) {
    const int64_t len = c->prow1[r] - c->prow0[r];
    if (r == c->team.rank || len <= 0) continue;
    const size_t off = static_cast<size_t>(role) * c->m + c->prow0[r];
    HX_CUDA(c, cudaMemcpyAsync(c->ypool + off, c->team.py[r] + off, len * sizeof(double), cudaMemcpyDefault,
                               c->stream));
  }
  return HPLP_OK;
}

// A x (A^T y): a rank computes its own rows (columns) only -- the blocks it stores.
int spmv_dev(hx_ctx* c, bool transpose, const double* x, double* out) {
  const Sched& S = c->ranked ? (transpose ? c->pt.view : c->pa.view) : (transpose ? c->st.view : c->sa.view);
  spmv_store_kernel<<<c->grid, kThreads, kStageBytes, c->stream>>>(S, x, out);
  c->launches += 1;
  HX_CUDA(c, cudaGetLastError());
  return HPLP_OK;
}

double* xbuf(hx_ctx* c, int i) { return c->xpool + static_cast<size_t>(i) * c->n; }
// baseline schemes: a vector that may live in an average slot
double* xbuf2(hx_ctx* c, int i, int avg) { return (avg ? c->xavg : c->xpool) + static_cast<size_t>(i) * c->n; }
double* ybuf2(hx_ctx* c, int i, int avg) { return (avg ? c->yavg : c->ypool) + static_cast<size_t>(i) * c->m; }
double* ybuf(hx_ctx* c, int i) { return c->ypool + static_cast<size_t>(i) * c->m; }
double* axbuf(hx_ctx* c, int i) { return c->axpool + static_cast<size_t>(i) * c->m; }

void fill_progress(hx_ctx* c, hx_progress_t* p) {
  if (!p) return;
  const Ctl& C = c->h;
  p->it = C.it;
  p->n = C.n;
  p->k = C.k;
  p->spmv_count = C.spmv;
  p->status = C.status;
  p->error = C.error;
  p->paused = C.paused;
  p->best_valid = C.best_kkt < std::numeric_limits<double>::infinity();
  p->res_epoch_start = C.res_epoch_start;
  p->best_kkt = C.best_kkt;
  p->best_err = {C.best_err[0], C.best_err[1], C.best_err[2], C.best_err[3]};
  p->trace_it = C.last_it;
  p->trace_n = C.last_n;
  p->trace_k = C.last_k;
  p->trace_res = C.last_res;
  p->trace_res_diff = C.last_res_diff;
  p->trace_kkt = {C.last_kkt[0], C.last_kkt[1], C.last_kkt[2], C.last_kkt[3]};
  p->final_kkt = {C.final_kkt[0], C.final_kkt[1], C.final_kkt[2], C.final_kkt[3]};
  p->n_epochs = C.n_epochs;
  p->primal_cert = C.cert[0];
  p->dual_cert = C.cert[1];
}

}  // namespace

extern "C" {

namespace {
// Summation order new contexts start with: hx_set_default_sum_order, else
// the environment (HPLP_SUM_ORDER=reference), else HX_SUM_FAST.
std::atomic<int> g_sum_order{-1};
int default_sum_order() {
  int v = g_sum_order.load();
  if (v < 0) {
    const char* e = std::getenv("HPLP_SUM_ORDER");
    v = e && (std::strcmp(e, "reference") == 0 || std::strcmp(e, "1") == 0) ? HX_SUM_REFERENCE : HX_SUM_FAST;
  }
  return v;
}
}  // namespace

int hx_set_default_sum_order(int32_t order) {
  if (order != HX_SUM_FAST && order != HX_SUM_REFERENCE && order != -1) return HPLP_EINVAL;
  g_sum_order.store(order);
  return HPLP_OK;
}

int hx_create(int32_t device, hx_ctx** out) {
  *out = nullptr;
  const auto t_create = std::chrono::steady_clock::now();
  auto ctx = std::make_unique<hx_ctx>();
  ctx->device = device;
  ctx->sum_order = default_sum_order();
  int ndev = 0;
  if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0)
    return set_err(nullptr, HPLP_ECUDA, "hx_create: no CUDA device visible (the B200 path has no CPU fallback)");
  if (device < 0 || device >= ndev) return set_err(nullptr, HPLP_EINVAL, "hx_create: bad device index");
  hx_ctx* c = ctx.get();
  HX_CUDA(nullptr, cudaSetDevice(device));
  // single attributes: cudaGetDeviceProperties costs milliseconds per call
  int major = 0, minor = 0, coop = 0;
  HX_CUDA(nullptr, cudaDeviceGetAttribute(&major, cudaDevAttrComputeCapabilityMajor, device));
  HX_CUDA(nullptr, cudaDeviceGetAttribute(&minor, cudaDevAttrComputeCapabilityMinor, device));
  HX_CUDA(nullptr, cudaDeviceGetAttribute(&coop, cudaDevAttrCooperativeLaunch, device));
  HX_CUDA(nullptr, cudaDeviceGetAttribute(&c->sm_count, cudaDevAttrMultiProcessorCount, device));
  if (major < 10)
    return set_err(nullptr, HPLP_ECUDA,
                   "hx_create: this build targets sm_100a (B200); found sm_" + std::to_string(major * 10 + minor));
  if (!coop) return set_err(nullptr, HPLP_ECUDA, "hx_create: cooperative launch unsupported");
  HX_CUDA(nullptr, cudaFuncSetAttribute(loop_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                        static_cast<int>(kStageBytes)));
  HX_CUDA(nullptr, cudaFuncSetAttribute(spmv_store_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                        static_cast<int>(kStageBytes)));
  HX_CUDA(nullptr, cudaFuncSetAttribute(loop_kernel_team, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                        static_cast<int>(kStageBytes)));
  HX_CUDA(nullptr, cudaFuncSetAttribute(loop_kernel_baseline, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                        static_cast<int>(kStageBytes)));
  HX_CUDA(nullptr, cudaFuncSetAttribute(loop_kernel_box, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                        static_cast<int>(kStageBytes)));
  HX_CUDA(nullptr, cudaFuncSetAttribute(loop_kernel_stream, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                        static_cast<int>(kStageBytes)));
  HX_CUDA(nullptr, cudaFuncSetAttribute(loop_kernel_stream_cb, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                        static_cast<int>(kStageBytes)));
  int occ = 0;
  HX_CUDA(nullptr, cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, loop_kernel, kThreads, kStageBytes));
  if (occ < 1) return set_err(nullptr, HPLP_ECUDA, "hx_create: loop kernel does not fit on an SM");
  c->grid = c->sm_count * std::min(occ, kMinBlocks);
  HX_CUDA(nullptr, cudaStreamCreateWithFlags(&c->stream, cudaStreamNonBlocking));
  HX_CUDA(nullptr, cudaEventCreate(&c->ev0));
  HX_CUDA(nullptr, cudaEventCreate(&c->ev1));
  HX_CUDA(nullptr, dalloc(&c->slots, static_cast<size_t>(kRegions) * kReplicas * kMaxQ * c->grid));
  HX_CUDA(nullptr, dalloc(&c->scratch, kMaxQ));
  HX_CUDA(nullptr, dalloc(&c->ctl, 1));
  HX_CUDA(nullptr, dalloc(&c->kparams, 1));
  if (const char* e = std::getenv("HX_PROFILE"); e && e[0] == '1') {
    HX_CUDA(nullptr, dalloc(&c->prof, static_cast<size_t>(c->grid) * kProfWords));
    HX_CUDA(nullptr, cudaMemset(c->prof, 0, static_cast<size_t>(c->grid) * kProfWords * sizeof(unsigned long long)));
  }
  HX_CUDA(nullptr, dalloc(&c->bar, 1));
  HX_CUDA(nullptr, dalloc(&c->epochs, kEpochCap));
  HX_CUDA(nullptr, cudaMemset(c->bar, 0, sizeof(GridBar)));
  HX_CUDA(nullptr, cudaMemset(c->ctl, 0, sizeof(Ctl)));
  std::memset(&c->h, 0, sizeof(Ctl));
  if (const char* e = std::getenv("HPLP_TIMING"); e && e[0] == '1') {
    cudaDeviceSynchronize();
    std::fprintf(stderr, "hx_create: %8.3f ms\n",
                 std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t_create).count());
  }
  *out = ctx.release();
  return HPLP_OK;
}

void hx_destroy(hx_ctx* c) {
  if (!c) return;
  cudaSetDevice(c->device);
  for (void* p : c->ipc_open) cudaIpcCloseMemHandle(p);
  dfree(c->rbar), dfree(c->xneed), dfree(c->yneed);
  free_problem(c);
  dfree(c->slots), dfree(c->scratch), dfree(c->ctl), dfree(c->bar), dfree(c->epochs), dfree(c->kparams), dfree(c->prof);
  if (c->ev0) cudaEventDestroy(c->ev0);
  if (c->ev1) cudaEventDestroy(c->ev1);
  if (c->stream) cudaStreamDestroy(c->stream);
  delete c;
}

const char* hx_last_error(hx_ctx* c) { return c ? c->err.c_str() : g_create_err.c_str(); }

int hx_device_info(hx_ctx* c, int32_t* sm_count, int32_t* grid_ctas, int32_t* cta_threads) {
  if (sm_count) *sm_count = c->sm_count;
  if (grid_ctas) *grid_ctas = c->grid;
  if (cta_threads) *cta_threads = kThreads;
  return HPLP_OK;
}

void* hx_stream(hx_ctx* c) { return c->stream; }
int64_t hx_launch_count(hx_ctx* c) { return c->launches; }

int hx_stored_nonzeros(hx_ctx* c, int64_t* nnz_a, int64_t* nnz_t) {
  if (!c->uploaded) return set_err(c, HPLP_ESTATE, "hx_stored_nonzeros: no problem uploaded");
  if (nnz_a) *nnz_a = c->nnz_a;
  if (nnz_t) *nnz_t = c->nnz_t;
  return HPLP_OK;
}

int hx_schedule_info(const int32_t* row_ptr, int32_t rows, int32_t ctas, double lead, int32_t* tasks,
                     int64_t capacity, int64_t* n_tasks, double* stats) {
  if (!row_ptr || rows < 0 || ctas < 1 || !n_tasks || capacity < 0)
    return set_err(nullptr, HPLP_EINVAL, "hx_schedule_info: bad arguments");
  for (int32_t i = 0; i < rows; ++i)
    if (row_ptr[i + 1] < row_ptr[i]) return set_err(nullptr, HPLP_EINVAL, "hx_schedule_info: row_ptr is not monotone");
  const int warps = ctas * kWarps;
  double rc, tc;
  sched_costs(true, rc, tc);
  const SchedHost h = build_schedule(row_ptr, rows, warps, lead, rc, tc, false);
  *n_tasks = static_cast<int64_t>(h.tasks.size());
  if (stats) {
    std::vector<double> cta(static_cast<size_t>(ctas), 0.0);
    for (size_t k = 0; k < h.tasks.size(); ++k) {
      const int4 t = h.tasks[k];
      if (t.x == 0 && t.y == 0 && t.w == 0) continue;
      cta[(k % warps) / kWarps] += (t.w - t.z) + rc * ((t.y & kRowMask) - t.x) + tc;
    }
    double mx = 0.0, sum = 0.0;
    for (double v : cta) mx = std::max(mx, v), sum += v;
    stats[0] = warps, stats[1] = h.max_warp_cost, stats[2] = h.mean_warp_cost;
    stats[3] = mx, stats[4] = sum / ctas;
  }
  if (static_cast<int64_t>(h.tasks.size()) > capacity)
    return set_err(nullptr, HPLP_EINVAL, "hx_schedule_info: capacity below the task slot count");
  if (tasks) std::memcpy(tasks, h.tasks.data(), h.tasks.size() * sizeof(int4));
  return HPLP_OK;
}

int hx_dims(hx_ctx* c, int64_t* m, int64_t* n, int64_t* nnz) {
  if (m) *m = c->m;
  if (n) *n = c->n;
  if (nnz) *nnz = c->nnz;
  return c->uploaded ? HPLP_OK : set_err(c, HPLP_ESTATE, "hx_dims: no problem uploaded");
}

namespace {
// The ranks this process launches together (hx_team_bind / a lone rank of a
// multi-process team), rank order, checked complete.
int team_ranks(hx_ctx* c, std::vector<hx_ctx*>& ranks) {
  ranks = c->local_team.empty() ? std::vector<hx_ctx*>{c} : c->local_team;
  std::sort(ranks.begin(), ranks.end(), [](hx_ctx* a, hx_ctx* b) { return a->team.rank < b->team.rank; });
  for (hx_ctx* r : ranks) {
    if (!r->ranked || r->team.nranks == 0)
      return set_err(c, HPLP_ESTATE, "hx: rank is not part of a usable team");
    for (int q = 0; q < r->team.nranks; ++q)
      if (!r->team.px[q] || !r->team.py[q] || !r->team.pu[q] || !r->team.ps[q] || !r->team.pb[q] || !r->peer_ring[q])
        return set_err(c, HPLP_ESTATE, "hx: team incomplete (bind or import every rank first)");
  }
  return HPLP_OK;
}

// One launch of a team setup mode (kModePower / kModeKkt / kModeScale) with
// the controllers the caller prepared in every rank's host mirror.
int team_mode_launch(hx_ctx* c, const std::vector<hx_ctx*>& ranks) {
  const int rc = team_launch(ranks);
  if (rc) c->err = ranks.front()->err;
  return rc;
}
}  // namespace

namespace {
// One rank of a row-partitioned team (hx_set_partition): the
// context stores ONLY its blocks -- rows [row0, row1) of A and columns
// [col0, col1) of A (the rows of A^T it owns), both cut on the host from the
// caller's CSR -- plus full-length b, c and iterate pools (the pools double
// as receive buffers: peers push the x+ / y entries this rank gathers into
// them at their global offsets).  Device memory is O(nnz / nranks + m + n),
// so an LP whose matrix exceeds one GPU fits on the team.  The schedules
// index the blocks through pointers offset by row0 / col0, so the kernels
// keep global row indices.
int upload_ranked(hx_ctx* c, int64_t m, int64_t n, const int64_t* row_ptr, const int32_t* col_idx, const double* val,
                  const double* b, const double* cc) {
  Team& T = c->team;
  if (T.row1 > m || T.col1 > n)
    return set_err(c, HPLP_EINVAL, "hx_upload_csr: partition range exceeds the problem (hx_set_partition)");
  if (c->prow1[T.nranks - 1] != m || c->pcol1[T.nranks - 1] != n)
    return set_err(c, HPLP_EINVAL, "hx_upload_csr: the partition does not cover the problem");
  const int64_t nnz = row_ptr[m];
  // the whole matrix is validated on every rank (the same error everywhere);
  // the checks of validate_kernel, on the host copy the caller passed
  for (int64_t i = 0; i < m; ++i) {
    if (row_ptr[i + 1] < row_ptr[i]) return set_err(c, HPLP_EINVAL, "hx_upload_csr: row_ptr is not monotone");
    for (int64_t p = row_ptr[i]; p < row_ptr[i + 1]; ++p) {
      const int j = col_idx[p];
      if (j < 0 || j >= n) return set_err(c, HPLP_EINVAL, "SparseMatrix: entry out of range");
      if (!std::isfinite(val[p])) return set_err(c, HPLP_EINVAL, "SparseMatrix: non-finite value");
      if (p > row_ptr[i] && j == col_idx[p - 1]) return set_err(c, HPLP_EINVAL, "SparseMatrix: duplicate entry");
      if (p > row_ptr[i] && j < col_idx[p - 1])
        return set_err(c, HPLP_EINVAL, "hx_upload_csr: columns must ascend within each row (sort on the host)");
    }
  }
  const int row0 = T.row0, row1 = T.row1, col0 = T.col0, col1 = T.col1;
  const int ml = row1 - row0, nl = col1 - col0;
  // A's row block: the caller's arrays from row_ptr[row0]
  std::vector<int> ap(static_cast<size_t>(ml) + 1);
  const int64_t pa0 = row_ptr[row0];
  if (row_ptr[row1] - pa0 >= (int64_t{1} << 31))
    return set_err(c, HPLP_EINVAL, "hx_upload_csr: a rank's row block exceeds 2^31 - 1 nonzeros (more ranks)");
  for (int i = 0; i <= ml; ++i) ap[i] = static_cast<int>(row_ptr[row0 + i] - pa0);
  const int64_t nnz_a = ap[ml];
  // A^T's row block = A's columns [col0, col1), rows ascending per column
  std::vector<int64_t> tp64(static_cast<size_t>(nl) + 1, 0);
  for (int64_t p = 0; p < nnz; ++p) {
    const int j = col_idx[p];
    if (j >= col0 && j < col1) ++tp64[j - col0 + 1];
  }
  for (int k = 0; k < nl; ++k) tp64[k + 1] += tp64[k];
  if (tp64[nl] >= (int64_t{1} << 31))
    return set_err(c, HPLP_EINVAL, "hx_upload_csr: a rank's column block exceeds 2^31 - 1 nonzeros (more ranks)");
  std::vector<int> tp(tp64.begin(), tp64.end());
  const int64_t nnz_t = tp[nl];
  std::vector<int> ti(static_cast<size_t>(nnz_t));
  std::vector<double> tv(static_cast<size_t>(nnz_t));
  {
    std::vector<int> fill(tp.begin(), tp.end() - 1);
    for (int64_t i = 0; i < m; ++i)
      for (int64_t p = row_ptr[i]; p < row_ptr[i + 1]; ++p) {
        const int j = col_idx[p];
        if (j < col0 || j >= col1) continue;
        const int q = fill[j - col0]++;
        ti[q] = static_cast<int>(i);
        tv[q] = val[p];
      }
  }
  cudaStream_t s = c->stream;
  c->m = m, c->n = n, c->nnz = nnz;
  c->nnz_a = nnz_a, c->nnz_t = nnz_t;
  HX_CUDA(c, dalloc(&c->a_ptr, static_cast<size_t>(ml) + 1));
  HX_CUDA(c, dalloc(&c->a_idx, static_cast<size_t>(nnz_a) + kMatrixPad));
  HX_CUDA(c, dalloc(&c->a_val, static_cast<size_t>(nnz_a) + kMatrixPad));
  HX_CUDA(c, dalloc(&c->t_ptr, static_cast<size_t>(nl) + 1));
  HX_CUDA(c, dalloc(&c->t_idx, static_cast<size_t>(nnz_t) + kMatrixPad));
  HX_CUDA(c, dalloc(&c->t_val, static_cast<size_t>(nnz_t) + kMatrixPad));
  HX_CUDA(c, dalloc(&c->b, m));
  HX_CUDA(c, dalloc(&c->c, n));
  HX_CUDA(c, cudaMemcpyAsync(c->a_ptr, ap.data(), ap.size() * sizeof(int), cudaMemcpyHostToDevice, s));
  if (nnz_a) {
    HX_CUDA(c, cudaMemcpyAsync(c->a_idx, col_idx + pa0, nnz_a * sizeof(int), cudaMemcpyHostToDevice, s));
    HX_CUDA(c, cudaMemcpyAsync(c->a_val, val + pa0, nnz_a * sizeof(double), cudaMemcpyHostToDevice, s));
  }
  HX_CUDA(c, cudaMemcpyAsync(c->t_ptr, tp.data(), tp.size() * sizeof(int), cudaMemcpyHostToDevice, s));
  if (nnz_t) {
    HX_CUDA(c, cudaMemcpyAsync(c->t_idx, ti.data(), nnz_t * sizeof(int), cudaMemcpyHostToDevice, s));
    HX_CUDA(c, cudaMemcpyAsync(c->t_val, tv.data(), nnz_t * sizeof(double), cudaMemcpyHostToDevice, s));
  }
  if (m) HX_CUDA(c, cudaMemcpyAsync(c->b, b, m * sizeof(double), cudaMemcpyHostToDevice, s));
  if (n) HX_CUDA(c, cudaMemcpyAsync(c->c, cc, n * sizeof(double), cudaMemcpyHostToDevice, s));
  HX_CUDA(c, cudaStreamSynchronize(s));  // the host vectors go out of scope
  // schedules of the blocks; rows / columns stay global through offset pointers
  double lead = kLead;
  if (const char* e = std::getenv("HX_LEAD")) lead = std::atof(e);
  const bool exact = c->sum_order == HX_SUM_REFERENCE;
  const int warps = c->grid * kWarps;
  double rca, tca, rct, tct;
  sched_costs(false, rca, tca);
  sched_costs(true, rct, tct);
  int rc = upload_built_sched(c, c->pa, build_schedule(ap.data(), ml, warps, 0.0, rca, tca, exact), ml,
                              static_cast<int>(n), c->a_ptr - row0, c->a_idx, c->a_val, row0);
  if (rc) return rc;
  rc = upload_built_sched(c, c->pt, build_schedule(tp.data(), nl, warps, lead, rct, tct, exact), nl,
                          static_cast<int>(m), c->t_ptr - col0, c->t_idx, c->t_val, col0);
  if (rc) return rc;
  // who gathers what: x+_j is read by the owners of the rows in column j,
  // y_i by the owners of the columns in row i
  auto owner = [&](const int* lo, int v) {
    int r = 0;
    while (r + 1 < T.nranks && v >= lo[r + 1]) ++r;
    return r;
  };
  std::vector<unsigned char> xm(static_cast<size_t>(nl), 0), ym(static_cast<size_t>(ml), 0);
  for (int64_t i = 0; i < m; ++i) {
    const int oi = owner(c->prow0, static_cast<int>(i));
    const bool own_row = i >= row0 && i < row1;
    for (int64_t p = row_ptr[i]; p < row_ptr[i + 1]; ++p) {
      const int j = col_idx[p];
      if (oi != T.rank && j >= col0 && j < col1) xm[j - col0] |= static_cast<unsigned char>(1u << oi);
      if (own_row) {
        const int oj = owner(c->pcol0, j);
        if (oj != T.rank) ym[i - row0] |= static_cast<unsigned char>(1u << oj);
      }
    }
  }
  dfree(c->xneed), dfree(c->yneed);
  HX_CUDA(c, dalloc(&c->xneed, std::max<size_t>(1, xm.size())));
  HX_CUDA(c, dalloc(&c->yneed, std::max<size_t>(1, ym.size())));
  if (!xm.empty()) HX_CUDA(c, cudaMemcpy(c->xneed, xm.data(), xm.size(), cudaMemcpyHostToDevice));
  if (!ym.empty()) HX_CUDA(c, cudaMemcpy(c->yneed, ym.data(), ym.size(), cudaMemcpyHostToDevice));
  T.xneed = c->xneed;
  T.yneed = c->yneed;
  // L2 policy from this rank's blocks and vectors
  int l2 = 0;
  cudaDeviceGetAttribute(&l2, cudaDevAttrL2CacheSize, c->device);
  const double footprint = 12.0 * static_cast<double>(nnz_a + nnz_t) + 8.0 * (6.0 * n + 10.0 * m);
  int hint = footprint > 0.7 * static_cast<double>(l2) ? 1 : 0;
  if (const char* e = std::getenv("HPLP_L2_STREAM")) hint = std::atoi(e) != 0 ? 1 : 0;
  c->pa.view.stream_hint = c->pt.view.stream_hint = hint;
  c->pa.view.row_limit = static_cast<int>(m);
  c->pt.view.row_limit = static_cast<int>(n);
  c->pa.view.exact = c->pt.view.exact = exact ? 1 : 0;
  // pools (peers map them through CUDA IPC)
  HX_CUDA(c, dalloc_ipc(&c->xpool, static_cast<size_t>(kXPool) * n));
  HX_CUDA(c, dalloc_ipc(&c->ypool, static_cast<size_t>(kYPool) * m));
  HX_CUDA(c, dalloc_ipc(&c->upool, 2 * static_cast<size_t>(n) + 2 * static_cast<size_t>(m)));
  HX_CUDA(c, dalloc(&c->axpool, static_cast<size_t>(kAxPool) * m));
  c->ring_cap = ring_capacity(n, m);  // same on every rank (same n, m, environment)
  HX_CUDA(c, dalloc_ipc(&c->ring, ring_layout(c->ring_cap, n, m).bytes));
  for (int r = 0; r < kMaxRanks; ++r) c->peer_ring[r] = nullptr;
  c->peer_ring[T.rank] = c->ring;
  for (int r = 0; r < kMaxRanks; ++r) T.px[r] = T.py[r] = T.pu[r] = T.ps[r] = nullptr, T.pb[r] = nullptr;
  T.px[T.rank] = c->xpool, T.py[T.rank] = c->ypool, T.pu[T.rank] = c->upool, T.ps[T.rank] = c->slots;
  T.pb[T.rank] = c->rbar;
  c->local_team.assign(1, c);
  // ||b||, ||c|| once, from the full vectors every rank holds
  kkt_partials_kernel<<<c->grid, kThreads, 0, s>>>(static_cast<int>(m), static_cast<int>(n), nullptr, c->b, nullptr,
                                                   c->c, nullptr, nullptr, c->slots);
  final_reduce_kernel<<<1, 256, 0, s>>>(c->slots, c->grid, 6, c->scratch);
  double tot[6];
  HX_CUDA(c, cudaMemcpyAsync(tot, c->scratch, sizeof(tot), cudaMemcpyDeviceToHost, s));
  HX_CUDA(c, cudaStreamSynchronize(s));
  c->launches += 2 + (nnz_a || nnz_t ? 2 : 0);
  c->b_sq = tot[4];
  c->b_norm = std::sqrt(tot[4]);
  c->c_norm = std::sqrt(tot[5]);
  c->uploaded = true;
  return HPLP_OK;
}
}  // namespace

int hx_upload_csr(hx_ctx* c, int64_t m, int64_t n, const int64_t* row_ptr, const int32_t* col_idx,
                  const double* val, const double* b, const double* cc) {
  HX_CUDA(c, cudaSetDevice(c->device));
  free_problem(c);
  if (m < 0 || n < 0) return set_err(c, HPLP_EINVAL, "SparseMatrix: negative dimension");
  if (row_ptr[0] != 0) return set_err(c, HPLP_EINVAL, "hx_upload_csr: row_ptr[0] must be 0");
  const int64_t nnz = row_ptr[m];
  // int32 indices on the device: m, n < 2^31 - 1, and every stored CSR copy
  // (one GPU: the whole matrix; a rank: each of its two blocks) < 2^31
  // nonzeros -- a team holds a matrix of more than 2^31 nonzeros in total
  if (nnz < 0 || m >= (int64_t{1} << 31) - 1 || n >= (int64_t{1} << 31) - 1)
    return set_err(c, HPLP_EINVAL, "hx_upload_csr: sizes exceed the int32 index range of this build");
  if (!c->ranked && nnz >= (int64_t{1} << 31))
    return set_err(c, HPLP_EINVAL,
                   "hx_upload_csr: more than 2^31 - 1 nonzeros on one GPU (int32 positions); use a team");
  for (int64_t i = 0; i < m; ++i)
    if (!std::isfinite(b[i])) return set_err(c, HPLP_EINVAL, "StandardFormLP: non-finite b or c");
  for (int64_t j = 0; j < n; ++j)
    if (!std::isfinite(cc[j])) return set_err(c, HPLP_EINVAL, "StandardFormLP: non-finite b or c");
  if (c->ranked) return upload_ranked(c, m, n, row_ptr, col_idx, val, b, cc);
  c->m = m, c->n = n, c->nnz = nnz;
  c->nnz_a = c->nnz_t = nnz;
  // A's schedule needs only the host row pointers: build it on a host thread
  // while the matrix copies and A^T forms on the device
  std::vector<int> ph(static_cast<size_t>(m) + 1);
  bool monotone = true;
  for (int64_t i = 0; i <= m; ++i) {
    ph[i] = static_cast<int>(row_ptr[i]);
    if (i && row_ptr[i] < row_ptr[i - 1]) monotone = false;
  }
  const int sched_warps = c->grid * kWarps;
  const bool exact = c->sum_order == 1;
  // bank-staggered stream tasks (build_schedule): at most kStaggerA / kStaggerT
  // pad slots before a row of >= kStaggerLmin nonzeros; HX_STAGGER="a,t,lmin"
  // overrides (0,0 turns it off)
  int stagger_a = kStaggerA, stagger_t = kStaggerT, stagger_lmin = kStaggerLmin;
  if (const char* e = std::getenv("HX_STAGGER")) std::sscanf(e, "%d,%d,%d", &stagger_a, &stagger_t, &stagger_lmin);
  // the staggered copies cost another 12 bytes per nonzero per matrix: above
  // kStaggerMaxNnz the plain layout keeps the footprint of the largest
  // one-GPU problems
  if (nnz > kStaggerMaxNnz) stagger_a = stagger_t = 0;
  int align = kTaskAlign;
  if (const char* e = std::getenv("HX_ALIGN")) align = std::atoi(e);
  std::future<SchedHost> sched_a;
  if (monotone)  // else the device check below reports it
    sched_a = std::async(std::launch::async, [&ph, m, sched_warps, exact, stagger_a, stagger_lmin, align] {
      double rc, tc;
      sched_costs(false, rc, tc);
      return build_schedule(ph.data(), static_cast<int>(m), sched_warps, 0.0, rc, tc, exact, stagger_a, stagger_lmin,
                            align);
    });
  cudaStream_t s = c->stream;
  const int nblk = 4 * c->sm_count;
  // HPLP_TIMING=1: wall time of the upload stages on stderr
  const bool timing = [] {
    const char* e = std::getenv("HPLP_TIMING");
    return e && e[0] == '1';
  }();
  auto tick = [&, t0 = std::chrono::steady_clock::now()](const char* what) mutable {
    if (!timing) return;
    cudaStreamSynchronize(s);
    const auto t1 = std::chrono::steady_clock::now();
    std::fprintf(stderr, "hx_upload_csr: %-12s %8.3f ms\n", what, std::chrono::duration<double, std::milli>(t1 - t0).count());
    t0 = t1;
  };
  // Matrix A (CSR), validated on the device.
  long long* rp64 = nullptr;
  unsigned* flags = nullptr;
  DevFree guard_rp64{reinterpret_cast<void**>(&rp64)}, guard_flags{reinterpret_cast<void**>(&flags)};
  HX_CUDA(c, dalloc(&rp64, m + 1));
  HX_CUDA(c, dalloc(&flags, 1));
  HX_CUDA(c, dalloc(&c->a_ptr, m + 1));
  HX_CUDA(c, dalloc(&c->a_idx, nnz + kMatrixPad));
  HX_CUDA(c, dalloc(&c->a_val, nnz + kMatrixPad));
  HX_CUDA(c, dalloc(&c->b, m));
  HX_CUDA(c, dalloc(&c->c, n));
  HX_CUDA(c, cudaMemcpyAsync(rp64, row_ptr, (m + 1) * sizeof(long long), cudaMemcpyHostToDevice, s));
  if (nnz) {
    HX_CUDA(c, cudaMemcpyAsync(c->a_idx, col_idx, nnz * sizeof(int), cudaMemcpyHostToDevice, s));
    HX_CUDA(c, cudaMemcpyAsync(c->a_val, val, nnz * sizeof(double), cudaMemcpyHostToDevice, s));
  }
  if (m) HX_CUDA(c, cudaMemcpyAsync(c->b, b, m * sizeof(double), cudaMemcpyHostToDevice, s));
  if (n) HX_CUDA(c, cudaMemcpyAsync(c->c, cc, n * sizeof(double), cudaMemcpyHostToDevice, s));
  HX_CUDA(c, cudaMemsetAsync(flags, 0, sizeof(unsigned), s));
  validate_kernel<<<nblk, 256, 0, s>>>(static_cast<int>(m), static_cast<int>(n), rp64, c->a_idx, c->a_val, flags);
  narrow_ptr_kernel<<<nblk, 256, 0, s>>>(static_cast<int>(m + 1), rp64, c->a_ptr);
  unsigned hflags = 0;
  HX_CUDA(c, cudaMemcpyAsync(&hflags, flags, sizeof(unsigned), cudaMemcpyDeviceToHost, s));
  HX_CUDA(c, cudaStreamSynchronize(s));
  c->launches += 2;
  tick("copy+check");
  if ((hflags & 16u) || !monotone) return set_err(c, HPLP_EINVAL, "hx_upload_csr: row_ptr is not monotone");
  if (hflags & 1u) return set_err(c, HPLP_EINVAL, "SparseMatrix: entry out of range");
  if (hflags & 2u) return set_err(c, HPLP_EINVAL, "SparseMatrix: non-finite value");
  if (hflags & 8u) return set_err(c, HPLP_EINVAL, "SparseMatrix: duplicate entry");
  if (hflags & 4u)
    return set_err(c, HPLP_EINVAL, "hx_upload_csr: columns must ascend within each row (sort on the host)");
  // Explicit A^T with ascending rows per column: stable radix sort by column.
  {
    int *row_of = nullptr, *iota = nullptr, *keys_out = nullptr, *perm = nullptr, *cnt = nullptr;
    void* tmp = nullptr;
    // temporaries are freed on every exit, error returns included
    DevFree g0{reinterpret_cast<void**>(&row_of)}, g1{reinterpret_cast<void**>(&iota)},
        g2{reinterpret_cast<void**>(&keys_out)}, g3{reinterpret_cast<void**>(&perm)}, g4{reinterpret_cast<void**>(&cnt)},
        g5{&tmp};
    HX_CUDA(c, dalloc(&row_of, nnz));
    HX_CUDA(c, dalloc(&iota, nnz));
    HX_CUDA(c, dalloc(&keys_out, nnz));
    HX_CUDA(c, dalloc(&perm, nnz));
    HX_CUDA(c, dalloc(&cnt, n + 1));
    HX_CUDA(c, dalloc(&c->t_ptr, n + 1));
    HX_CUDA(c, dalloc(&c->t_idx, nnz + kMatrixPad));
    HX_CUDA(c, dalloc(&c->t_val, nnz + kMatrixPad));
    row_of_kernel<<<nblk, 256, 0, s>>>(static_cast<int>(m), c->a_ptr, row_of, iota);
    int bits = 1;
    while ((int64_t{1} << bits) < n + 1) ++bits;
    size_t tmp_bytes = 0, scan_bytes = 0;
    cub::DeviceRadixSort::SortPairs(nullptr, tmp_bytes, c->a_idx, keys_out, iota, perm, static_cast<int>(nnz), 0,
                                    bits, s);
    cub::DeviceScan::ExclusiveSum(nullptr, scan_bytes, cnt, c->t_ptr, static_cast<int>(n + 1), s);
    HX_CUDA(c, dalloc(reinterpret_cast<unsigned char**>(&tmp), std::max<size_t>(1, std::max(tmp_bytes, scan_bytes))));
    if (nnz)
      HX_CUDA(c, cub::DeviceRadixSort::SortPairs(tmp, tmp_bytes, c->a_idx, keys_out, iota, perm,
                                                 static_cast<int>(nnz), 0, bits, s));
    HX_CUDA(c, cudaMemsetAsync(cnt, 0, (n + 1) * sizeof(int), s));
    col_count_kernel<<<nblk, 256, 0, s>>>(static_cast<int>(nnz), c->a_idx, cnt);
    HX_CUDA(c, cub::DeviceScan::ExclusiveSum(tmp, scan_bytes, cnt, c->t_ptr, static_cast<int>(n + 1), s));
    gather_t_kernel<<<nblk, 256, 0, s>>>(static_cast<int>(nnz), perm, row_of, c->a_val, c->t_idx, c->t_val);
    HX_CUDA(c, cudaStreamSynchronize(s));
    HX_CUDA(c, cudaGetLastError());
    c->launches += 5;
  }
  tick("transpose");
  // Schedules (host, from the pointer arrays).
  {
    std::vector<int> pt(static_cast<size_t>(n) + 1);
    HX_CUDA(c, cudaMemcpy(pt.data(), c->t_ptr, (n + 1) * sizeof(int), cudaMemcpyDeviceToHost));
    // phase A (rows of A^T) runs speculatively while warp 0 of every CTA runs
    // the controller: warp 0 starts with a lead (kLead)
    double lead = kLead;
    if (const char* e = std::getenv("HX_LEAD")) lead = std::atof(e);
    // A^T's schedule is built on a host thread while A's uploads
    auto sched_t = std::async(std::launch::async, [&pt, n, sched_warps, lead, exact, stagger_t, stagger_lmin, align] {
      double rc, tc;
      sched_costs(true, rc, tc);
      return build_schedule(pt.data(), static_cast<int>(n), sched_warps, lead, rc, tc, exact, stagger_t, stagger_lmin,
                            align);
    });
    int rc = upload_built_sched(c, c->sa, sched_a.get(), static_cast<int>(m), static_cast<int>(n), c->a_ptr,
                                c->a_idx, c->a_val, 0);
    if (rc) return rc;
    tick("sched A");
    rc = upload_built_sched(c, c->st, sched_t.get(), static_cast<int>(n), static_cast<int>(m), c->t_ptr, c->t_idx,
                            c->t_val, 0);
    if (rc) return rc;
    tick("sched A^T");
  }
  {
    // per-iteration working set of the loop: the matrix copies this context
    // streams (a rank: its blocks) plus the ~6 n- and ~10 m-vectors an
    // iteration touches; beyond ~70% of L2 the matrix streams get evict_first
    int l2 = 0;
    cudaDeviceGetAttribute(&l2, cudaDevAttrL2CacheSize, c->device);
    const int64_t streamed = 2 * nnz;
    const double footprint = 12.0 * static_cast<double>(streamed) + 8.0 * (6.0 * n + 10.0 * m);
    int hint = footprint > 0.7 * static_cast<double>(l2) ? 1 : 0;
    if (const char* e = std::getenv("HPLP_L2_STREAM")) hint = std::atoi(e) != 0 ? 1 : 0;
    c->sa.view.stream_hint = c->st.view.stream_hint = hint;
    c->sa.view.row_limit = static_cast<int>(m);  // output dimension (HX_CHECKED)
    c->st.view.row_limit = static_cast<int>(n);
    c->sa.view.exact = c->st.view.exact = exact ? 1 : 0;
    // Column-blocked phase B (loop_kernel_stream_cb): when x+ is far larger
    // than L2 its random gathers miss (configs[4]: 9.5 GB of DRAM traffic per
    // iteration against 5.0 GB algorithmic, L2 hit rate 38%), so A is split at
    // the columns that cut its nonzeros into K equal parts and phase B sweeps
    // the blocks one after the other (a grid barrier between), each sweep
    // gathering from 1/K of x+.  Auto (K = 2) when 8 n > 64 MB on the stream
    // path; HX_COLBLOCK=0/1 forces it off / on (K = 2), HX_COLBLOCK=K (2..8)
    // sets K.  Row sums become ((block 0) + (block 1)) + ..., each block's
    // part in ascending column order.
    int want = hint && 8.0 * static_cast<double>(n) > 64e6 ? 2 : 0;
    if (const char* e = std::getenv("HX_COLBLOCK")) {
      want = std::atoi(e);
      want = want == 1 ? 2 : std::min(want, kMaxColBlocks);
    }
    // the reference order sums each row in one chain: no split at a column
    if (want >= 2 && nnz > 0 && !exact && n >= want) {
      const int K = want;
      std::vector<int> pt(static_cast<size_t>(n) + 1);
      HX_CUDA(c, cudaMemcpy(pt.data(), c->t_ptr, (n + 1) * sizeof(int), cudaMemcpyDeviceToHost));
      ColSplit sp{};
      sp.K = K;
      for (int k = 0; k + 1 < K; ++k)
        sp.split[k] = static_cast<int>(std::lower_bound(pt.begin(), pt.end(),
                                                        static_cast<int>(nnz * (k + 1) / K)) - pt.begin());
      sp.split[K - 1] = static_cast<int>(n);
      // the blocks are cut on the device (the matrix is resident); only their
      // row pointers come back for the host schedules
      int* cnt[kMaxColBlocks] = {};
      unsigned char* scan_tmp = nullptr;
      DevFree gst{reinterpret_cast<void**>(&scan_tmp)};
      static_assert(kMaxColBlocks == 8, "one guard per block count array");
      DevFree gcnt[kMaxColBlocks] = {{reinterpret_cast<void**>(&cnt[0])}, {reinterpret_cast<void**>(&cnt[1])},
                                     {reinterpret_cast<void**>(&cnt[2])}, {reinterpret_cast<void**>(&cnt[3])},
                                     {reinterpret_cast<void**>(&cnt[4])}, {reinterpret_cast<void**>(&cnt[5])},
                                     {reinterpret_cast<void**>(&cnt[6])}, {reinterpret_cast<void**>(&cnt[7])}};
      for (int k = 0; k < K; ++k) {
        HX_CUDA(c, dalloc(&cnt[k], static_cast<size_t>(m) + 1));
        HX_CUDA(c, cudaMemsetAsync(cnt[k], 0, sizeof(int), s));
        HX_CUDA(c, dalloc(&c->cb_ptr[k], static_cast<size_t>(m) + 1));
        sp.cnt[k] = cnt[k];
      }
      split_count_kernel<<<nblk, 256, 0, s>>>(static_cast<int>(m), c->a_ptr, c->a_idx, sp);
      size_t scan_bytes = 0;
      cub::DeviceScan::InclusiveSum(nullptr, scan_bytes, cnt[0], c->cb_ptr[0], static_cast<int>(m + 1), s);
      HX_CUDA(c, dalloc(&scan_tmp, std::max<size_t>(1, scan_bytes)));
      for (int k = 0; k < K; ++k)
        HX_CUDA(c, cub::DeviceScan::InclusiveSum(scan_tmp, scan_bytes, cnt[k], c->cb_ptr[k], static_cast<int>(m + 1), s));
      std::vector<std::vector<int>> ph_k(static_cast<size_t>(K), std::vector<int>(static_cast<size_t>(m) + 1));
      for (int k = 0; k < K; ++k)
        HX_CUDA(c, cudaMemcpyAsync(ph_k[k].data(), c->cb_ptr[k], (m + 1) * sizeof(int), cudaMemcpyDeviceToHost, s));
      HX_CUDA(c, cudaStreamSynchronize(s));
      for (int k = 0; k < K; ++k) {
        const size_t nz = static_cast<size_t>(ph_k[k][m]);
        HX_CUDA(c, dalloc(&c->cb_idx[k], nz + kMatrixPad));
        HX_CUDA(c, dalloc(&c->cb_val[k], nz + kMatrixPad));
        sp.ptr[k] = c->cb_ptr[k];
        sp.idx[k] = c->cb_idx[k];
        sp.val[k] = c->cb_val[k];
      }
      split_copy_kernel<<<nblk, 256, 0, s>>>(static_cast<int>(m), c->a_ptr, c->a_idx, c->a_val, sp);
      HX_CUDA(c, cudaStreamSynchronize(s));
      HX_CUDA(c, cudaGetLastError());
      c->launches += 2 + K;
      tick("cb split");
      // the blocks' schedules are built concurrently on host threads
      std::vector<std::future<SchedHost>> sb(static_cast<size_t>(K));
      for (int k = 0; k < K; ++k)
        sb[k] = std::async(std::launch::async, [pk = &ph_k[k], m, sched_warps, stagger_a, stagger_lmin, align] {
          double rc, tc;
          sched_costs(false, rc, tc);
          return build_schedule(pk->data(), static_cast<int>(m), sched_warps, 0.0, rc, tc, false, stagger_a,
                                stagger_lmin, align);
        });
      for (int k = 0; k < K; ++k) {
        const int rc = upload_built_sched(c, c->sb[k], sb[k].get(), static_cast<int>(m), static_cast<int>(n),
                                          c->cb_ptr[k], c->cb_idx[k], c->cb_val[k], 0);
        if (rc) return rc;
        c->sb[k].view.stream_hint = hint;
        c->sb[k].view.row_limit = static_cast<int>(m);
      }
      HX_CUDA(c, dalloc(&c->bpart, static_cast<size_t>(std::max<int64_t>(m, 1))));
      c->colblock = K;
    }
  }
  tick("schedules");
  HX_CUDA(c, dalloc(&c->xpool, static_cast<size_t>(kXPool) * n));
  HX_CUDA(c, dalloc(&c->ypool, static_cast<size_t>(kYPool) * m));
  HX_CUDA(c, dalloc(&c->upool, 2 * static_cast<size_t>(n) + 2 * static_cast<size_t>(m)));
  HX_CUDA(c, dalloc(&c->axpool, static_cast<size_t>(kAxPool) * m));
  // ||b||, ||c|| once (loop invariants of src/pdhg_core.cpp:60,62).
  kkt_partials_kernel<<<c->grid, kThreads, 0, s>>>(static_cast<int>(m), static_cast<int>(n), nullptr, c->b,
                                                   nullptr, c->c, nullptr, nullptr, c->slots);
  final_reduce_kernel<<<1, 256, 0, s>>>(c->slots, c->grid, 6, c->scratch);
  double tot[6];
  HX_CUDA(c, cudaMemcpyAsync(tot, c->scratch, sizeof(tot), cudaMemcpyDeviceToHost, s));
  HX_CUDA(c, cudaStreamSynchronize(s));
  c->launches += 2;
  c->b_sq = tot[4];
  c->b_norm = std::sqrt(tot[4]);
  c->c_norm = std::sqrt(tot[5]);
  tick("pools+norms");
  c->uploaded = true;
  return HPLP_OK;
}

// Diagonal preconditioning of the uploaded problem (no reference
// counterpart: SPEC.md:101/259 name it an extension point).  ruiz_iters
// rounds of Ruiz infinity-norm equilibration, then (pc_alpha >= 0) one
// Pock-Chambolle step with exponent alpha.  Writes the accumulated row
// scales R (m) and column scales C (n) when the pointers are non-NULL.
int hx_set_sum_order(hx_ctx* c, int32_t order) {
  if (order != HX_SUM_FAST && order != HX_SUM_REFERENCE)
    return set_err(c, HPLP_EINVAL, "hx_set_sum_order: order must be HX_SUM_FAST or HX_SUM_REFERENCE");
  if (c->uploaded && order != c->sum_order)
    return set_err(c, HPLP_ESTATE, "hx_set_sum_order: set before hx_upload_csr (the schedules depend on it)");
  c->sum_order = order;
  return HPLP_OK;
}

int32_t hx_sum_order(hx_ctx* c) { return c ? c->sum_order : -1; }

int hx_precondition(hx_ctx* c, int32_t ruiz_iters, double pc_alpha, double* row_scale, double* col_scale) {
  if (!c->uploaded) return set_err(c, HPLP_ESTATE, "hx_precondition: no problem uploaded");
  if (ruiz_iters < 0) return set_err(c, HPLP_EINVAL, "hx_precondition: ruiz_iters must be >= 0");
  if (c->ranked) {
    // a team: kModeScale on every rank of this process at once (every
    // process calls it for its rank); the scales of the rows / columns a rank
    // owns are pushed to the peers that scale entries of them, and the
    // accumulated R (u3) / C (u2) come back from their owners
    std::vector<hx_ctx*> ranks;
    if (int rc = team_ranks(c, ranks)) return rc;
    for (hx_ctx* r : ranks) {
      Ctl& C = r->h;
      std::memset(&C, 0, sizeof(Ctl));
      C.mode = kModeScale;
      C.sc_ruiz = ruiz_iters;
      C.sc_pc = pc_alpha >= 0.0 ? 1 : 0;
      C.sc_alpha = pc_alpha;
      r->setup_done = false;
    }
    int rc = team_mode_launch(c, ranks);
    for (hx_ctx* r : ranks) r->h.mode = kModeLoop;
    if (rc) return rc;
    for (hx_ctx* r : ranks) {
      r->b_sq = r->h.sc_bsq;
      r->b_norm = std::sqrt(r->h.sc_bsq);
      r->c_norm = std::sqrt(r->h.sc_csq);
    }
    HX_CUDA(c, cudaSetDevice(c->device));
    const int64_t m = c->m, n = c->n;
    for (int q = 0; q < c->team.nranks; ++q) {
      const double* pu = c->team.pu[q];
      if (row_scale && c->prow1[q] > c->prow0[q])
        HX_CUDA(c, cudaMemcpy(row_scale + c->prow0[q], pu + 2 * n + m + c->prow0[q],
                              (c->prow1[q] - c->prow0[q]) * sizeof(double), cudaMemcpyDefault));
      if (col_scale && c->pcol1[q] > c->pcol0[q])
        HX_CUDA(c, cudaMemcpy(col_scale + c->pcol0[q], pu + n + c->pcol0[q],
                              (c->pcol1[q] - c->pcol0[q]) * sizeof(double), cudaMemcpyDefault));
    }
    return HPLP_OK;
  }
  cudaStream_t s = c->stream;
  const int m = static_cast<int>(c->m), n = static_cast<int>(c->n);
  const int nb = 4 * c->sm_count;
  double *dr = nullptr, *dc = nullptr, *R = nullptr, *Cs = nullptr;
  HX_CUDA(c, dalloc(&dr, m));
  HX_CUDA(c, dalloc(&dc, n));
  HX_CUDA(c, dalloc(&R, m));
  HX_CUDA(c, dalloc(&Cs, n));
  std::vector<double> ones(static_cast<size_t>(std::max(m, n)), 1.0);
  if (m) HX_CUDA(c, cudaMemcpyAsync(R, ones.data(), m * sizeof(double), cudaMemcpyHostToDevice, s));
  if (n) HX_CUDA(c, cudaMemcpyAsync(Cs, ones.data(), n * sizeof(double), cudaMemcpyHostToDevice, s));
  auto apply = [&]() -> int {
    inv_sqrt_kernel<<<nb, 256, 0, s>>>(m, dr, R);
    inv_sqrt_kernel<<<nb, 256, 0, s>>>(n, dc, Cs);
    scale_csr_kernel<<<nb, 256, 0, s>>>(m, c->a_ptr, c->a_idx, c->a_val, dr, dc, 0);
    scale_csr_kernel<<<nb, 256, 0, s>>>(n, c->t_ptr, c->t_idx, c->t_val, dr, dc, 1);
    // every other copy of A's values the loop reads gets the same two roundings
    // (v * d_row) * d_col, so all copies stay bit-identical to a_val
    for (int k = 0; k < c->colblock; ++k)  // column blocks of phase B (loop_kernel_stream_cb)
      scale_csr_kernel<<<nb, 256, 0, s>>>(m, c->cb_ptr[k], c->cb_idx[k], c->cb_val[k], dr, dc, 0);
    // the bank-staggered copies the schedules index (their pads stay 0)
    if (c->sa.pval) scale_csr_kernel<<<nb, 256, 0, s>>>(m, c->sa.pptr, c->sa.pidx, c->sa.pval, dr, dc, 0);
    if (c->st.pval) scale_csr_kernel<<<nb, 256, 0, s>>>(n, c->st.pptr, c->st.pidx, c->st.pval, dr, dc, 1);
    c->launches += (c->sa.pval ? 1 : 0) + (c->st.pval ? 1 : 0);
    for (int k = 0; k < c->colblock; ++k)  // the column blocks' staggered copies
      if (c->sb[k].pval) {
        scale_csr_kernel<<<nb, 256, 0, s>>>(m, c->sb[k].pptr, c->sb[k].pidx, c->sb[k].pval, dr, dc, 0);
        c->launches += 1;
      }
    scale_vec_kernel<<<nb, 256, 0, s>>>(m, c->b, dr);
    scale_vec_kernel<<<nb, 256, 0, s>>>(n, c->c, dc);
    if (c->ub) div_vec_kernel<<<nb, 256, 0, s>>>(n, c->ub, dc);  // x = C x': x' <= u / C
    c->launches += (c->ub ? 7 : 6) + c->colblock;
    HX_CUDA(c, cudaGetLastError());
    return HPLP_OK;
  };
  for (int k = 0; k < ruiz_iters; ++k) {
    row_norm_kernel<<<nb, 256, 0, s>>>(m, c->a_ptr, c->a_val, 0, 1.0, dr);
    row_norm_kernel<<<nb, 256, 0, s>>>(n, c->t_ptr, c->t_val, 0, 1.0, dc);
    c->launches += 2;
    int rc = apply();
    if (rc) return rc;
  }
  if (pc_alpha >= 0.0) {
    row_norm_kernel<<<nb, 256, 0, s>>>(m, c->a_ptr, c->a_val, 1, 2.0 - pc_alpha, dr);
    row_norm_kernel<<<nb, 256, 0, s>>>(n, c->t_ptr, c->t_val, 1, pc_alpha, dc);
    c->launches += 2;
    int rc = apply();
    if (rc) return rc;
  }
  if (row_scale && m) HX_CUDA(c, cudaMemcpyAsync(row_scale, R, m * sizeof(double), cudaMemcpyDeviceToHost, s));
  if (col_scale && n) HX_CUDA(c, cudaMemcpyAsync(col_scale, Cs, n * sizeof(double), cudaMemcpyDeviceToHost, s));
  // ||b||, ||c|| of the transformed instance
  kkt_partials_kernel<<<c->grid, kThreads, 0, s>>>(m, n, nullptr, c->b, nullptr, c->c, nullptr, nullptr, c->slots);
  final_reduce_kernel<<<1, 256, 0, s>>>(c->slots, c->grid, 6, c->scratch);
  double tot[6];
  HX_CUDA(c, cudaMemcpyAsync(tot, c->scratch, sizeof(tot), cudaMemcpyDeviceToHost, s));
  HX_CUDA(c, cudaStreamSynchronize(s));
  c->launches += 2;
  c->b_sq = tot[4];
  if (c->ub) {  // box form: ||b|| of the standard form it stands for (rescaled u)
    std::vector<double> u(static_cast<size_t>(n));
    if (n) HX_CUDA(c, cudaMemcpy(u.data(), c->ub, n * sizeof(double), cudaMemcpyDeviceToHost));
    c->u_sq = 0.0;
    for (double v : u)
      if (v < INFINITY) c->u_sq += v * v;
  }
  c->b_norm = std::sqrt(c->b_sq + (c->ub ? c->u_sq : 0.0));
  c->c_norm = std::sqrt(tot[5]);
  dfree(dr), dfree(dc), dfree(R), dfree(Cs);
  c->setup_done = false;
  return HPLP_OK;
}

// Box form: column upper bounds enforced by the primal
// projection, x in [0, u] (u = +inf: no bound); NULL returns to the standard
// form.  Set after hx_upload_csr and before hx_precondition / hx_setup.
int32_t hx_loop_variant(hx_ctx* c) {
  if (!c || !c->uploaded) return -1;
  if (c->ranked) return c->pa.view.stream_hint && c->pt.view.stream_hint ? 6 : 5;
  return c->ub ? 2 : c->sum_order == HX_SUM_REFERENCE ? 4 : c->sa.view.stream_hint ? (c->colblock ? 3 : 1) : 0;
}

int hx_set_box(hx_ctx* c, const double* upper) {
  if (!c->uploaded) return set_err(c, HPLP_ESTATE, "hx_set_box: no problem uploaded");
  HX_CUDA(c, cudaSetDevice(c->device));
  if (!upper) {
    dfree(c->ub);
    c->ub = nullptr;
    c->u_sq = 0.0;
    c->b_norm = std::sqrt(c->b_sq);
    c->setup_done = false;
    return HPLP_OK;
  }
  double u_sq = 0.0;
  for (int64_t j = 0; j < c->n; ++j) {
    if (std::isnan(upper[j]) || upper[j] < 0.0)
      return set_err(c, HPLP_EINVAL, "hx_set_box: upper bounds must be >= 0 (or +inf)");
    if (upper[j] < INFINITY) u_sq += upper[j] * upper[j];
  }
  // the KKT primal residual is relative to the standard form's ||b|| (b and
  // the bound rows' u), so the box form's KKT equals the standard form's at
  // the mapped iterate and tolerances mean the same
  c->u_sq = u_sq;
  c->b_norm = std::sqrt(c->b_sq + u_sq);
  if (!c->ub) HX_CUDA(c, dalloc(&c->ub, std::max<int64_t>(c->n, 1)));
  if (c->n) HX_CUDA(c, cudaMemcpyAsync(c->ub, upper, c->n * sizeof(double), cudaMemcpyHostToDevice, c->stream));
  HX_CUDA(c, cudaStreamSynchronize(c->stream));
  c->setup_done = false;
  return HPLP_OK;
}

// The device problem (after any preconditioning) as CSR + b + c.

int hx_download_problem(hx_ctx* c, int64_t* row_ptr, int32_t* col_idx, double* val, double* b, double* cc) {
  if (!c->uploaded) return set_err(c, HPLP_ESTATE, "hx_download_problem: no problem uploaded");
  if (c->ranked) return set_err(c, HPLP_EINVAL, "hx_download_problem: a rank stores only its blocks");
  cudaStream_t s = c->stream;
  if (row_ptr) {
    std::vector<int> rp(static_cast<size_t>(c->m) + 1);
    HX_CUDA(c, cudaMemcpy(rp.data(), c->a_ptr, (c->m + 1) * sizeof(int), cudaMemcpyDeviceToHost));
    for (int64_t i = 0; i <= c->m; ++i) row_ptr[i] = rp[i];
  }
  if (col_idx && c->nnz) HX_CUDA(c, cudaMemcpyAsync(col_idx, c->a_idx, c->nnz * sizeof(int), cudaMemcpyDeviceToHost, s));
  if (val && c->nnz) HX_CUDA(c, cudaMemcpyAsync(val, c->a_val, c->nnz * sizeof(double), cudaMemcpyDeviceToHost, s));
  if (b && c->m) HX_CUDA(c, cudaMemcpyAsync(b, c->b, c->m * sizeof(double), cudaMemcpyDeviceToHost, s));
  if (cc && c->n) HX_CUDA(c, cudaMemcpyAsync(cc, c->c, c->n * sizeof(double), cudaMemcpyDeviceToHost, s));
  HX_CUDA(c, cudaStreamSynchronize(s));
  return HPLP_OK;
}

int hx_spmv(hx_ctx* c, const double* x, double* out) {
  if (!c->uploaded) return set_err(c, HPLP_ESTATE, "hx_spmv: no problem uploaded");
  double* dx = c->upool;
  double* dout = c->upool + 2 * c->n;
  HX_CUDA(c, cudaMemcpyAsync(dx, x, c->n * sizeof(double), cudaMemcpyHostToDevice, c->stream));
  if (c->ranked) HX_CUDA(c, cudaMemsetAsync(dout, 0, c->m * sizeof(double), c->stream));  // a rank: its rows only
  int rc = spmv_dev(c, false, dx, dout);
  if (rc) return rc;
  HX_CUDA(c, cudaMemcpyAsync(out, dout, c->m * sizeof(double), cudaMemcpyDeviceToHost, c->stream));
  HX_CUDA(c, cudaStreamSynchronize(c->stream));
  return HPLP_OK;
}

int hx_spmv_transpose(hx_ctx* c, const double* y, double* out) {
  if (!c->uploaded) return set_err(c, HPLP_ESTATE, "hx_spmv_transpose: no problem uploaded");
  double* dy = c->upool + 2 * c->n;
  double* dout = c->upool;
  HX_CUDA(c, cudaMemcpyAsync(dy, y, c->m * sizeof(double), cudaMemcpyHostToDevice, c->stream));
  if (c->ranked) HX_CUDA(c, cudaMemsetAsync(dout, 0, c->n * sizeof(double), c->stream));  // a rank: its columns only
  int rc = spmv_dev(c, true, dy, dout);
  if (rc) return rc;
  HX_CUDA(c, cudaMemcpyAsync(out, dout, c->n * sizeof(double), cudaMemcpyDeviceToHost, c->stream));
  HX_CUDA(c, cudaStreamSynchronize(c->stream));
  return HPLP_OK;
}

int hx_power_iteration(hx_ctx* c, const double* x0, double tol, int64_t k0, int64_t max_iters, double sigma_prev,
                       double* sigma, int64_t* iters, int32_t* converged, int32_t* need_redraw) {
  if (!c->uploaded) return set_err(c, HPLP_ESTATE, "hx_power_iteration: no problem uploaded");
  // a team: every rank of this process (every process calls it for its own
  // rank), each on its blocks; the start vector is on every rank in full
  std::vector<hx_ctx*> ranks{c};
  if (c->ranked)
    if (int rc = team_ranks(c, ranks)) return rc;
  for (hx_ctx* r : ranks) {
    HX_CUDA(c, cudaSetDevice(r->device));
    HX_CUDA(c, cudaMemcpyAsync(xbuf(r, 0), x0, r->n * sizeof(double), cudaMemcpyHostToDevice, r->stream));
    HX_CUDA(c, cudaStreamSynchronize(r->stream));
    Ctl& C = r->h;
    std::memset(&C, 0, sizeof(Ctl));
    C.mode = kModePower;
    C.pw_k = k0;
    C.pw_max = max_iters;
    C.pw_tol = tol;
    C.pw_sigma_prev = sigma_prev;
    C.pw_sigma = sigma_prev;  // res.sigma == sigma_prev between iterations
    C.pw_iters = k0;
    C.r.pw_mode = 0;
    C.r.stop = k0 >= max_iters ? 1 : 0;
    r->setup_done = false;
  }
  HX_CUDA(c, cudaSetDevice(c->device));
  Ctl& C = c->h;
  if (!C.r.stop) {
    int rc = c->ranked ? team_mode_launch(c, ranks) : launch_loop(c);
    if (rc) return rc;
  }
  *sigma = C.pw_sigma;
  *iters = C.pw_iters;
  *converged = C.pw_converged;
  *need_redraw = C.pw_redraw;
  c->setup_done = false;
  return HPLP_OK;
}

int hx_setup(hx_ctx* c, const hplp_config_t* cfg, double sigma_used, double eta, const double* x0,
             const double* y0) {
  if (!c->uploaded) return set_err(c, HPLP_ESTATE, "hx_setup: no problem uploaded");
  if (cfg->scheme < HPLP_SCHEME_RHPDHG || cfg->scheme > HPLP_SCHEME_RESTARTED_AVERAGE)
    return set_err(c, HPLP_EINVAL, "hx_setup: unknown scheme");
  if (cfg->scheme != HPLP_SCHEME_RHPDHG && c->ranked)
    return set_err(c, HPLP_EINVAL, "hx_setup: the baseline schemes run on one device (no team)");
  if (c->ub && cfg->scheme != HPLP_SCHEME_RHPDHG)
    return set_err(c, HPLP_EINVAL, "hx_setup: the box form runs rHPDHG only");
  if (c->ub && c->ranked) return set_err(c, HPLP_EINVAL, "hx_setup: the box form runs on one device (no team)");
  if (c->ub && cfg->infeasibility_check_period > 0)
    return set_err(c, HPLP_EINVAL, "hx_setup: the box form has no infeasibility scan (set infeasibility_check_period 0)");
  cudaStream_t s = c->stream;
  if (cfg->scheme >= HPLP_SCHEME_AVERAGED && !c->xavg) {  // running-average slots
    HX_CUDA(c, dalloc(&c->xavg, static_cast<size_t>(kAvgPool) * c->n));
    HX_CUDA(c, dalloc(&c->tavg, static_cast<size_t>(kAvgPool) * c->n));
    HX_CUDA(c, dalloc(&c->yavg, static_cast<size_t>(kAvgPool) * c->m));
    HX_CUDA(c, dalloc(&c->aavg, static_cast<size_t>(kAvgPool) * c->m));
    HX_CUDA(c, dalloc(&c->xbar, c->n));
  }
  if (x0) HX_CUDA(c, cudaMemcpyAsync(xbuf(c, 0), x0, c->n * sizeof(double), cudaMemcpyHostToDevice, s));
  else HX_CUDA(c, cudaMemsetAsync(xbuf(c, 0), 0, c->n * sizeof(double), s));
  if (y0) HX_CUDA(c, cudaMemcpyAsync(ybuf(c, 0), y0, c->m * sizeof(double), cudaMemcpyHostToDevice, s));
  else HX_CUDA(c, cudaMemsetAsync(ybuf(c, 0), 0, c->m * sizeof(double), s));
  int rc = spmv_dev(c, false, xbuf(c, 0), axbuf(c, 0));  // a_x = A x, src/solver.cpp:213
  if (rc) return rc;
  Ctl& C = c->h;
  std::memset(&C, 0, sizeof(Ctl));
  C.mode = kModeLoop;
  C.iteration_limit = cfg->iteration_limit;
  C.check_period = cfg->infeasibility_check_period;
  C.stall_cap = cfg->adaptive_stall_cap;
  C.k_star = cfg->k_star;
  C.tau0 = cfg->tau0;
  C.trace_period = cfg->trace_period;
  C.restart_kind = cfg->restart_kind;
  C.tol = cfg->tolerance;
  C.cert_tol = cfg->certificate_tolerance;
  C.beta = cfg->beta;
  C.sigma_used = sigma_used;
  C.b_norm = c->b_norm;
  C.c_norm = c->c_norm;
  c->time_limit_s = cfg->time_limit_seconds;
  c->loop_elapsed_s = 0.0;
  C.best_kkt = std::numeric_limits<double>::infinity();
  C.x_best = C.y_best = C.x_best_prev = -1;
  C.status = -1;
  C.final_x = C.final_y = -1;
  C.cert_cand[0] = C.cert_cand[1] = -1;
  C.scheme = cfg->scheme;
  C.avg_best = C.final_avg = C.last_cand_avg = -1;
  Roles& R = C.r;
  if (C.scheme >= HPLP_SCHEME_AVERAGED) {  // the first iteration copies z into the average
    R.avg_mode = 1, R.avg_cur = -1, R.avg_out = 0, R.w_avg = 1.0;
  }
  R.avg_step = C.scheme >= HPLP_SCHEME_AVERAGED;  // restarted: every iteration; averaged: k == 0 (it 0)
  R.eta = eta;
  R.x_src = 0, R.x_anchor = 0, R.x_mode = 0, R.w_x = 0.0;
  R.zx_out = 1, R.xp_out = 2;
  R.y_cur = 0, R.y_anchor = 0, R.yp_out = 1, R.yc_out = 2;
  R.ax_cur = 0, R.ax_anchor = 0, R.axp_out = 1, R.axc_out = 2;
  R.w_next = 0.5;  // 1/(k+2) at k = 0
  // trace ring: the rHPDHG loop of the standard form (one GPU or a team)
  // records traced iterations on the device; the box form and the baselines
  // pause per traced iteration instead
  bool ring_on = cfg->trace_period > 0 && C.scheme == HPLP_SCHEME_RHPDHG && !c->ub;
  if (const char* e = std::getenv("HPLP_TRACE_RING")) ring_on = ring_on && std::atoi(e) != 0;
  if (ring_on && !c->ring) {  // one GPU: allocated on first use (a rank has it from the upload)
    c->ring_cap = ring_capacity(c->n, c->m);
    HX_CUDA(c, dalloc(&c->ring, ring_layout(c->ring_cap, c->n, c->m).bytes));
  }
  C.ring_cap = ring_on ? c->ring_cap : 0;
  C.ring_total = C.ring_drained = 0;
  c->r_tol = cfg->tol_active * sigma_used;  // partition_estimate_from_reduced_costs's r_tol
  c->tol_active = cfg->tol_active;
  C.r_tol = c->r_tol;
  C.tol_active = c->tol_active;
  R.tr_slot = ring_slot(C, 0);  // iteration 0
  R.tr_scale = 0.0;
  R.stop = 0;
  HX_CUDA(c, cudaMemsetAsync(c->epochs, 0, kEpochCap * sizeof(hplp_epoch_t), s));
  HX_CUDA(c, cudaStreamSynchronize(s));
  c->setup_done = true;
  return HPLP_OK;
}

}  // extern "C"

namespace {

// Loop-top checks of a batch (src/solver.cpp:242-254 before any iteration of
// this call); true when the loop must launch.
bool run_begin(hx_ctx* c, int64_t max_iters) {
  Ctl& C = c->h;
  if (!(C.status < 0 && C.error == 0 && max_iters > 0)) return false;
  auto limit = [&](int status) {
    C.status = status;
    if (C.best_kkt < std::numeric_limits<double>::infinity()) {
      C.final_x = C.x_best, C.final_y = C.y_best, C.final_avg = C.avg_best;
      std::memcpy(C.final_kkt, C.best_err, sizeof(C.final_kkt));
    } else {
      C.final_x = C.final_y = C.final_avg = -1;
    }
  };
  if (C.it >= C.iteration_limit) {  // :242-248
    limit(HPLP_STATUS_ITERATION_LIMIT);
    return false;
  }
  // :249-254 at the top of the next iteration.  A multi-rank team decides the
  // time limit on rank 0's clock inside the kernel (every rank reads the flag
  // rank 0 pushes): a host-side check here would let ranks disagree, and a
  // rank that launches alone would stall at the first team barrier.
  const bool team = c->ranked && c->team.nranks > 1;
  if (!team && c->loop_elapsed_s > c->time_limit_s) {
    limit(HPLP_STATUS_TIME_LIMIT);
    return false;
  }
  C.batch_end = C.it + max_iters;
  C.r.stop = 0;
  C.paused = 0;
  const double remaining = c->time_limit_s - c->loop_elapsed_s;
  C.time_budget_ns = std::isinf(remaining) ? 0ull
                     : remaining <= 1e-9    ? 1ull  // already over (a team rank): stop after one iteration
                                            : std::max<unsigned long long>(1ull, static_cast<unsigned long long>(remaining * 1e9));
  return true;
}

int run_end(hx_ctx* c, hx_progress_t* p, float ms, int64_t launches0) {
  fill_progress(c, p);
  if (p) {
    p->device_ms = ms;
    p->launches = c->launches - launches0;
  }
  if (c->h.error == HPLP_EDOMAIN)
    return set_err(c, HPLP_EDOMAIN, "canonical norm: quadratic form is negative (eta too large for this matrix)");
  return HPLP_OK;
}

// One batch of a team whose ranks all live in this process (emulated on one
// device, or one rank per device); every rank's host mirror is identical.
int team_run(const std::vector<hx_ctx*>& ranks, int64_t max_iters, hx_progress_t* progress) {
  hx_ctx* lead = ranks.front();
  std::vector<int64_t> l0;
  bool go = false;
  for (hx_ctx* c : ranks) {
    if (!c->setup_done) return set_err(lead, HPLP_ESTATE, "hx_team_run: call hx_setup on every rank first");
    if (!c->ranked || c->team.nranks == 0)
      return set_err(lead, HPLP_ESTATE, "hx_team_run: rank is not part of a usable team");
    for (int r = 0; r < c->team.nranks; ++r)
      if (!c->team.px[r] || !c->team.py[r] || !c->team.pu[r] || !c->team.ps[r] || !c->team.pb[r])
        return set_err(lead, HPLP_ESTATE, "hx_run: team incomplete (bind or import every rank first)");
    l0.push_back(c->launches);
    go = run_begin(c, max_iters);  // identical decision on every rank
  }
  float ms = 0.f;
  if (go) {
    const auto w0 = std::chrono::steady_clock::now();
    HX_CUDA(lead, cudaSetDevice(lead->device));
    HX_CUDA(lead, cudaEventRecord(lead->ev0, lead->stream));
    int rc = team_launch(ranks);
    if (rc) return rc;
    HX_CUDA(lead, cudaSetDevice(lead->device));
    HX_CUDA(lead, cudaEventRecord(lead->ev1, lead->stream));
    HX_CUDA(lead, cudaEventSynchronize(lead->ev1));
    HX_CUDA(lead, cudaEventElapsedTime(&ms, lead->ev0, lead->ev1));
    const double el = std::chrono::duration<double>(std::chrono::steady_clock::now() - w0).count();
    for (hx_ctx* c : ranks) c->loop_elapsed_s += el;
  }
  int rc = HPLP_OK;
  for (size_t i = 0; i < ranks.size(); ++i) {
    const int r2 = run_end(ranks[i], progress ? progress + i : nullptr, ms, l0[i]);
    if (rc == HPLP_OK) rc = r2;
  }
  if (rc) lead->err = ranks.back()->err;
  return rc;
}

}  // namespace

extern "C" {

int hx_run(hx_ctx* c, int64_t max_iters, hx_progress_t* p) {
  if (!c->setup_done) return set_err(c, HPLP_ESTATE, "hx_run: call hx_setup first");
  if (c->ranked) {
    if (c->local_team.size() > 1)
      return set_err(c, HPLP_ESTATE, "hx_run: ranks bound in this process run together through hx_team_run");
    return team_run({c}, max_iters, p);
  }
  const int64_t launches0 = c->launches;
  float ms = 0.f;
  if (run_begin(c, max_iters)) {
    const auto w0 = std::chrono::steady_clock::now();
    HX_CUDA(c, cudaEventRecord(c->ev0, c->stream));
    int rc = launch_loop(c);
    if (rc) return rc;
    HX_CUDA(c, cudaEventRecord(c->ev1, c->stream));
    HX_CUDA(c, cudaEventSynchronize(c->ev1));
    c->loop_elapsed_s += std::chrono::duration<double>(std::chrono::steady_clock::now() - w0).count();
    HX_CUDA(c, cudaEventElapsedTime(&ms, c->ev0, c->ev1));
  }
  return run_end(c, p, ms, launches0);
}

// ---- row-partitioned team (include/hx.h) ---------------------------------
int hx_set_partition(hx_ctx* c, int32_t nranks, int32_t rank, const int64_t* row_bounds, const int64_t* col_bounds,
                     int32_t ctas) {
  if (c->uploaded) return set_err(c, HPLP_ESTATE, "hx_set_partition: call before hx_upload_csr");
  if (nranks < 1 || nranks > kMaxRanks || rank < 0 || rank >= nranks || !row_bounds || !col_bounds)
    return set_err(c, HPLP_EINVAL, "hx_set_partition: need 1 <= nranks <= 8, 0 <= rank < nranks and the bounds");
  for (int r = 0; r < nranks; ++r)
    if (row_bounds[r] < 0 || row_bounds[r + 1] < row_bounds[r] || col_bounds[r] < 0 ||
        col_bounds[r + 1] < col_bounds[r] || row_bounds[r + 1] >= (int64_t{1} << 31) ||
        col_bounds[r + 1] >= (int64_t{1} << 31) || row_bounds[0] != 0 || col_bounds[0] != 0)
      return set_err(c, HPLP_EINVAL, "hx_set_partition: bounds must ascend from 0 (nranks + 1 entries each)");
  const int64_t row0 = row_bounds[rank], row1 = row_bounds[rank + 1];
  const int64_t col0 = col_bounds[rank], col1 = col_bounds[rank + 1];
  int occ = 0;
  HX_CUDA(c, cudaSetDevice(c->device));
  HX_CUDA(c, cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, loop_kernel_team, kThreads, kStageBytes));
  const int max_ctas = c->sm_count * std::min(std::max(occ, 1), kMinBlocks);
  if (ctas < 0 || ctas > max_ctas) return set_err(c, HPLP_EINVAL, "hx_set_partition: ctas out of range");
  if (ctas > 0) c->grid = ctas;
  c->ranked = true;
  c->team = Team{};
  c->team.rank = rank, c->team.nranks = nranks, c->team.grp_ctas = c->grid;
  // Rank records pay off once a controller would otherwise read several
  // 160-record batches (nranks * grid records; measured on one device, where
  // the leader's reduction competes with the other ranks' phases, the direct
  // read wins for 148 records).  HPLP_TEAM_PREREDUCE=0/1 forces either path.
  c->team.prereduce = nranks * c->grid > kPreReduceRecords ? 1 : 0;
  if (const char* e = std::getenv("HPLP_TEAM_PREREDUCE")) c->team.prereduce = std::atoi(e) != 0 ? 1 : 0;
  c->team.row0 = static_cast<int>(row0), c->team.row1 = static_cast<int>(row1);
  c->team.col0 = static_cast<int>(col0), c->team.col1 = static_cast<int>(col1);
  for (int r = 0; r < kMaxRanks; ++r) c->pcol0[r] = c->pcol1[r] = c->prow0[r] = c->prow1[r] = 0;
  for (int r = 0; r < nranks; ++r) {
    c->prow0[r] = static_cast<int>(row_bounds[r]), c->prow1[r] = static_cast<int>(row_bounds[r + 1]);
    c->pcol0[r] = static_cast<int>(col_bounds[r]), c->pcol1[r] = static_cast<int>(col_bounds[r + 1]);
  }
  c->local_team.clear();
  c->team_epochs = 0;
  // slot regions hold every rank's records
  dfree(c->slots);
  c->slots = nullptr;
  HX_CUDA(c, dalloc_ipc(&c->slots, static_cast<size_t>(kRegions) * kReplicas * kMaxQ * c->grid * nranks));
  if (!c->rbar) HX_CUDA(c, dalloc_ipc(&c->rbar, 1));
  HX_CUDA(c, cudaMemset(c->rbar, 0, sizeof(RankBar)));
  return HPLP_OK;
}

int32_t hx_team_size(hx_ctx* c) { return c && c->ranked ? c->team.nranks : 1; }

int hx_team_bind(hx_ctx** ctxs, int32_t count) {
  if (count < 1 || count > kMaxRanks || !ctxs) return set_err(nullptr, HPLP_EINVAL, "hx_team_bind: bad team size");
  std::vector<hx_ctx*> by(static_cast<size_t>(count), nullptr);
  for (int i = 0; i < count; ++i) {
    hx_ctx* c = ctxs[i];
    if (!c || !c->ranked || !c->uploaded)
      return set_err(c, HPLP_ESTATE, "hx_team_bind: every rank needs hx_set_partition + hx_upload_csr");
    if (c->team.nranks != count || by[c->team.rank])
      return set_err(c, HPLP_EINVAL, "hx_team_bind: ranks must be 0..count-1, each once");
    if (c->m != ctxs[0]->m || c->n != ctxs[0]->n || c->nnz != ctxs[0]->nnz || c->grid != ctxs[0]->grid)
      return set_err(c, HPLP_EINVAL, "hx_team_bind: ranks disagree on the problem or the CTA count");
    by[c->team.rank] = c;
  }
  int64_t rows = 0, cols = 0;
  for (hx_ctx* c : by) {
    if (c->team.row0 != rows || c->team.col0 != cols)
      return set_err(c, HPLP_EINVAL, "hx_team_bind: row / column blocks must tile the problem in rank order");
    rows = c->team.row1, cols = c->team.col1;
  }
  if (rows != by[0]->m || cols != by[0]->n)
    return set_err(by[0], HPLP_EINVAL, "hx_team_bind: row / column blocks must cover the problem");
  bool one_device = true;
  for (hx_ctx* c : by) one_device &= c->device == by[0]->device;
  if (one_device) {
    int occ = 0;
    HX_CUDA(by[0], cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, loop_kernel_team, kThreads, kStageBytes));
    if (static_cast<int64_t>(by[0]->grid) * count > static_cast<int64_t>(by[0]->sm_count) * occ)
      return set_err(by[0], HPLP_EINVAL,
                     "hx_team_bind: the emulated team does not fit on the device at once (ctas * ranks > resident CTAs)");
  } else {
    for (hx_ctx* a : by)
      for (hx_ctx* b : by)
        if (a->device != b->device) {
          HX_CUDA(a, cudaSetDevice(a->device));
          const cudaError_t e = cudaDeviceEnablePeerAccess(b->device, 0);
          if (e != cudaSuccess && e != cudaErrorPeerAccessAlreadyEnabled)
            return set_err(a, HPLP_ECUDA, std::string("hx_team_bind: peer access: ") + cudaGetErrorString(e));
          cudaGetLastError();
        }
  }
  for (hx_ctx* c : by)
    for (int r = 0; r < count; ++r)
      if (c->pcol0[r] != by[r]->team.col0 || c->pcol1[r] != by[r]->team.col1 || c->prow0[r] != by[r]->team.row0 ||
          c->prow1[r] != by[r]->team.row1)
        return set_err(c, HPLP_EINVAL, "hx_team_bind: ranks were given different partitions");
  for (hx_ctx* c : by) {
    Team& T = c->team;
    T.sys = one_device ? 0 : 1;
    for (int r = 0; r < count; ++r) {
      T.px[r] = by[r]->xpool, T.py[r] = by[r]->ypool, T.pu[r] = by[r]->upool, T.ps[r] = by[r]->slots;
      T.pb[r] = by[r]->rbar;
      c->peer_ring[r] = by[r]->ring;
    }
    c->local_team = by;
  }
  return HPLP_OK;
}

namespace {
struct TeamBlob {
  int32_t magic, rank, nranks, grid;
  int64_t m, n, nnz;
  int32_t row0, row1, col0, col1;
  int32_t ring_cap, pad;
  cudaIpcMemHandle_t hx, hy, hu, hs, hb, ht;
};
constexpr int32_t kBlobMagic = 0x48585442;  // "HXTB"
}  // namespace

int hx_team_export(hx_ctx* c, void* blob, int64_t capacity, int64_t* size) {
  if (size) *size = static_cast<int64_t>(sizeof(TeamBlob));
  if (!blob) return HPLP_OK;
  if (!c->ranked || !c->uploaded) return set_err(c, HPLP_ESTATE, "hx_team_export: needs hx_set_partition + upload");
  if (capacity < static_cast<int64_t>(sizeof(TeamBlob))) return set_err(c, HPLP_EINVAL, "hx_team_export: blob too small");
  TeamBlob b{};
  b.magic = kBlobMagic, b.rank = c->team.rank, b.nranks = c->team.nranks, b.grid = c->grid;
  b.m = c->m, b.n = c->n, b.nnz = c->nnz;
  b.row0 = c->team.row0, b.row1 = c->team.row1, b.col0 = c->team.col0, b.col1 = c->team.col1;
  b.ring_cap = c->ring_cap;
  HX_CUDA(c, cudaSetDevice(c->device));
  HX_CUDA(c, cudaIpcGetMemHandle(&b.hx, c->xpool));
  HX_CUDA(c, cudaIpcGetMemHandle(&b.hy, c->ypool));
  HX_CUDA(c, cudaIpcGetMemHandle(&b.hu, c->upool));
  HX_CUDA(c, cudaIpcGetMemHandle(&b.hs, c->slots));
  HX_CUDA(c, cudaIpcGetMemHandle(&b.hb, c->rbar));
  HX_CUDA(c, cudaIpcGetMemHandle(&b.ht, c->ring));
  std::memcpy(blob, &b, sizeof(b));
  return HPLP_OK;
}

int hx_team_import(hx_ctx* c, const void* blob, int64_t size) {
  if (!c->ranked || !c->uploaded) return set_err(c, HPLP_ESTATE, "hx_team_import: needs hx_set_partition + upload");
  if (size < static_cast<int64_t>(sizeof(TeamBlob))) return set_err(c, HPLP_EINVAL, "hx_team_import: short blob");
  TeamBlob b;
  std::memcpy(&b, blob, sizeof(b));
  if (b.magic != kBlobMagic || b.nranks != c->team.nranks || b.rank < 0 || b.rank >= b.nranks)
    return set_err(c, HPLP_EINVAL, "hx_team_import: blob of another team");
  if (b.m != c->m || b.n != c->n || b.nnz != c->nnz || b.grid != c->grid)
    return set_err(c, HPLP_EINVAL, "hx_team_import: ranks disagree on the problem or the CTA count");
  if (b.ring_cap != c->ring_cap)  // same n, m: only a different HPLP_TRACE_RING_MB gets here
    return set_err(c, HPLP_EINVAL, "hx_team_import: ranks disagree on the trace ring (HPLP_TRACE_RING_MB)");
  if (c->pcol0[b.rank] != b.col0 || c->pcol1[b.rank] != b.col1 || c->prow0[b.rank] != b.row0 ||
      c->prow1[b.rank] != b.row1)
    return set_err(c, HPLP_EINVAL, "hx_team_import: the peer was given a different partition");
  if (b.rank == c->team.rank) return HPLP_OK;
  HX_CUDA(c, cudaSetDevice(c->device));
  void* p[6] = {};
  const cudaIpcMemHandle_t* h[6] = {&b.hx, &b.hy, &b.hu, &b.hs, &b.hb, &b.ht};
  for (int k = 0; k < 6; ++k) {
    HX_CUDA(c, cudaIpcOpenMemHandle(&p[k], *h[k], cudaIpcMemLazyEnablePeerAccess));
    c->ipc_open.push_back(p[k]);
  }
  Team& T = c->team;
  T.sys = 1;  // a peer in another process: another GPU (one process per GPU)
  T.px[b.rank] = static_cast<double*>(p[0]);
  T.py[b.rank] = static_cast<double*>(p[1]);
  T.pu[b.rank] = static_cast<double*>(p[2]);
  T.ps[b.rank] = static_cast<double*>(p[3]);
  T.pb[b.rank] = static_cast<RankBar*>(p[4]);
  c->peer_ring[b.rank] = static_cast<unsigned char*>(p[5]);
  return HPLP_OK;
}

int hx_team_run(hx_ctx** ctxs, int32_t count, int64_t max_iters, hx_progress_t* progress) {
  if (count < 1 || !ctxs) return set_err(nullptr, HPLP_EINVAL, "hx_team_run: empty team");
  std::vector<hx_ctx*> v(ctxs, ctxs + count);
  for (hx_ctx* c : v)
    if (!c->ranked || c->local_team.size() != static_cast<size_t>(count))
      return set_err(c, HPLP_ESTATE, "hx_team_run: pass exactly the contexts bound by hx_team_bind");
  std::sort(v.begin(), v.end(), [](hx_ctx* a, hx_ctx* b) { return a->team.rank < b->team.rank; });
  std::vector<hx_progress_t> pr(v.size());
  const int rc = team_run(v, max_iters, pr.data());
  if (progress)
    for (int i = 0; i < count; ++i)
      for (size_t k = 0; k < v.size(); ++k)
        if (v[k] == ctxs[i]) progress[i] = pr[k];
  return rc;
}

int hx_progress(hx_ctx* c, hx_progress_t* p) {
  fill_progress(c, p);
  return HPLP_OK;
}

int hx_epochs(hx_ctx* c, int64_t first, int64_t count, hplp_epoch_t* out) {
  if (count <= 0) return HPLP_OK;
  if (first < c->h.n_epochs - kEpochCap) return set_err(c, HPLP_ESTATE, "hx_epochs: entries already overwritten");
  for (int64_t e = 0; e < count; ++e) {
    const int64_t slot = (first + e) % kEpochCap;
    HX_CUDA(c, cudaMemcpyAsync(out + e, c->epochs + slot, sizeof(hplp_epoch_t), cudaMemcpyDeviceToHost, c->stream));
  }
  HX_CUDA(c, cudaStreamSynchronize(c->stream));
  return HPLP_OK;
}

int hx_get_iterate(hx_ctx* c, int32_t which, double* x, double* y) {
  if (!c->setup_done) return set_err(c, HPLP_ESTATE, "hx_get_iterate: no solve state");
  const Ctl& C = c->h;
  const double* dx = nullptr;
  const double* dy = nullptr;
  cudaStream_t s = c->stream;
  switch (which) {
    case HX_ITERATE_BEST:
      if (C.avg_best >= 0) {  // averaged baselines: the best candidate is an average
        dx = xbuf2(c, C.avg_best, 1), dy = ybuf2(c, C.avg_best, 1);
        break;
      }
      if (C.x_best < 0) return set_err(c, HPLP_ESTATE, "hx_get_iterate: no best iterate yet");
      if (int rc = assemble_x(c, C.x_best)) return rc;
      if (int rc = assemble_y(c, C.y_best)) return rc;
      dx = xbuf(c, C.x_best), dy = ybuf(c, C.y_best);
      break;
    case HX_ITERATE_LAST:  // the traced candidate (z, or the average for the averaged baselines)
      if (C.it == 0 && C.status < 0) return set_err(c, HPLP_ESTATE, "hx_get_iterate: no iteration completed");
      if (C.last_cand_avg >= 0) {
        dx = xbuf2(c, C.last_cand_avg, 1), dy = ybuf2(c, C.last_cand_avg, 1);
        break;
      }
      if (int rc = assemble_x(c, C.last_zx)) return rc;
      if (int rc = assemble_y(c, C.last_y)) return rc;
      dx = xbuf(c, C.last_zx), dy = ybuf2(c, C.last_y, C.last_y_avg);
      break;
    case HX_ITERATE_NEXT:
      if (int rc = assemble_x(c, C.last_xp)) return rc;
      if (int rc = assemble_y(c, C.last_yp)) return rc;
      dx = xbuf(c, C.last_xp), dy = ybuf(c, C.last_yp);
      break;
    default: {  // the iterate the next iteration starts from
      if (C.status >= 0 && C.final_avg >= 0) {
        dx = xbuf2(c, C.final_avg, 1), dy = ybuf2(c, C.final_avg, 1);
      } else if (C.status >= 0 && C.final_x >= 0) {
        if (int rc = assemble_x(c, C.final_x)) return rc;
        if (int rc = assemble_y(c, C.final_y)) return rc;
        dx = xbuf(c, C.final_x), dy = ybuf(c, C.final_y);
      } else if (C.r.x_mode == 0) {
        if (int rc = assemble_x(c, C.r.x_src)) return rc;
        if (int rc = assemble_y(c, C.r.y_cur)) return rc;
        dx = xbuf2(c, C.r.x_src, C.r.x_src_avg), dy = ybuf2(c, C.r.y_cur, C.r.y_cur_avg);
      } else {
        if (int rc = assemble_x(c, C.r.x_src)) return rc;
        if (int rc = assemble_x(c, C.r.x_anchor)) return rc;
        if (int rc = assemble_y(c, C.r.y_cur)) return rc;
        double* tmp = c->upool;
        combine_kernel<<<4 * c->sm_count, 256, 0, s>>>(static_cast<int>(c->n), C.r.w_x, xbuf(c, C.r.x_src),
                                                       xbuf(c, C.r.x_anchor), tmp);
        c->launches += 1;
        dx = tmp, dy = ybuf(c, C.r.y_cur);
      }
    }
  }
  if (x && c->n) HX_CUDA(c, cudaMemcpyAsync(x, dx, c->n * sizeof(double), cudaMemcpyDeviceToHost, s));
  if (y && c->m) HX_CUDA(c, cudaMemcpyAsync(y, dy, c->m * sizeof(double), cudaMemcpyDeviceToHost, s));
  HX_CUDA(c, cudaStreamSynchronize(s));
  return HPLP_OK;
}

int hx_get_certificate(hx_ctx* c, int32_t kind, double* vec) {
  const Ctl& C = c->h;
  if (kind < 0 || kind > 1 || !C.cert[kind].present)
    return set_err(c, HPLP_ESTATE, "hx_get_certificate: no such certificate");
  const int cand = C.cert_cand[kind];
  const bool normalized = cand >= 2;
  const bool is_x = (cand == 0 || cand == 2);
  const int len = static_cast<int>(is_x ? c->n : c->m);
  const double* p;
  const double* q;
  if (is_x) {
    if (int rc = assemble_x(c, C.last_zx)) return rc;
    if (int rc = assemble_x(c, normalized ? C.last_xa : C.last_xp)) return rc;
    p = xbuf(c, C.last_zx);
    q = normalized ? xbuf(c, C.last_xa) : xbuf(c, C.last_xp);
  } else {
    if (int rc = assemble_y(c, normalized ? C.last_ya : C.last_yp)) return rc;
    if (int rc = assemble_y(c, C.last_y)) return rc;
    p = ybuf2(c, C.last_y, C.last_y_avg);
    q = normalized ? ybuf(c, C.last_ya) : ybuf(c, C.last_yp);
  }
  const double sgn = C.cert[kind].orientation == HPLP_ORIENT_NEGATED ? -1.0 : 1.0;
  const double factor = sgn / C.r.cn2[cand];
  double* tmp = c->upool;
  cert_kernel<<<4 * c->sm_count, 256, 0, c->stream>>>(len, normalized ? 1 : 0, C.r.cand_scale, factor, p, q, tmp);
  c->launches += 1;
  HX_CUDA(c, cudaMemcpyAsync(vec, tmp, len * sizeof(double), cudaMemcpyDeviceToHost, c->stream));
  HX_CUDA(c, cudaStreamSynchronize(c->stream));
  return HPLP_OK;
}

// Trace-point diagnostics of the last completed iteration (the fields of
// TraceRecord the loop does not produce, src/solver.cpp:279-287): A^T y of
// the traced y (the partition estimate's reduced costs are c + A^T y, on the
// device problem) and the canonical norm of the normalized candidate
// (2/k)(z - anchor) with its carried product; NaN when k = 0 (undefined), for
// a multi-rank context (A x is rank-local), or when the quadratic form is
// clearly negative.
int32_t hx_trace_ring_capacity(hx_ctx* c) { return c && c->setup_done ? c->h.ring_cap : 0; }

int64_t hx_trace_pending(hx_ctx* c) {
  if (!c || !c->setup_done || c->h.ring_cap <= 0) return 0;
  return c->h.ring_total - c->h.ring_drained;
}

int hx_trace_take(hx_ctx* c, hplp_trace_t* rec, double* x, double* y, unsigned char* cls) {
  if (hx_trace_pending(c) <= 0) return set_err(c, HPLP_ESTATE, "hx_trace_take: no pending trace record");
  const int64_t idx = c->h.ring_drained;
  const int slot = static_cast<int>(idx % c->h.ring_cap);
  const RingLayout L = ring_layout(c->ring_cap, c->n, c->m);
  HX_CUDA(c, cudaSetDevice(c->device));
  TraceRec t{};
  HX_CUDA(c, cudaMemcpy(&t, c->ring + L.rec + slot * sizeof(TraceRec), sizeof(t), cudaMemcpyDeviceToHost));
  // z.x / classes by column block, z.y by row block: one GPU holds all of
  // them; a team's ranks wrote their own slices into their own rings
  const int nr = c->ranked ? c->team.nranks : 1;
  for (int q = 0; q < nr; ++q) {
    const unsigned char* base = c->ranked ? c->peer_ring[q] : c->ring;
    if (!base) return set_err(c, HPLP_ESTATE, "hx_trace_take: team incomplete");
    const int64_t c0 = c->ranked ? c->pcol0[q] : 0, c1 = c->ranked ? c->pcol1[q] : c->n;
    const int64_t r0 = c->ranked ? c->prow0[q] : 0, r1 = c->ranked ? c->prow1[q] : c->m;
    const size_t xo = L.x + (static_cast<size_t>(slot) * c->n + c0) * sizeof(double);
    const size_t yo = L.y + (static_cast<size_t>(slot) * c->m + r0) * sizeof(double);
    const size_t co = L.cls + static_cast<size_t>(slot) * c->n + c0;
    if (x && c1 > c0) HX_CUDA(c, cudaMemcpy(x + c0, base + xo, (c1 - c0) * sizeof(double), cudaMemcpyDefault));
    if (cls && c1 > c0) HX_CUDA(c, cudaMemcpy(cls + c0, base + co, (c1 - c0), cudaMemcpyDefault));
    if (y && r1 > r0) HX_CUDA(c, cudaMemcpy(y + r0, base + yo, (r1 - r0) * sizeof(double), cudaMemcpyDefault));
  }
  if (rec) {
    std::memset(rec, 0, sizeof(*rec));
    rec->epoch = t.n;
    rec->inner = t.k;
    rec->iteration = t.it;
    rec->fixed_point_residual = t.res;
    rec->kkt = {t.kkt[0], t.kkt[1], t.kkt[2], t.kkt[3]};
    rec->candidate_norm_normalized = t.cand_norm;
    rec->candidate_norm_difference = t.res;  // ||T(z) - z|| (the residual for rHPDHG)
    rec->partition_n = t.cnt[0];
    rec->partition_b1 = t.cnt[1];
    rec->partition_b2 = t.cnt[2];
    rec->partition_sets = nullptr;
  }
  // every rank of this process drains in step (their controllers test the
  // ring's fill level against their own copy of the count)
  if (c->ranked && !c->local_team.empty())
    for (hx_ctx* r : c->local_team) r->h.ring_drained = idx + 1;
  c->h.ring_drained = idx + 1;
  return HPLP_OK;
}

int hx_trace_reduced_costs(hx_ctx* c, double* rc) {
  if (!c->setup_done) return set_err(c, HPLP_ESTATE, "hx_trace_reduced_costs: no solve state");
  const Ctl& C = c->h;
  if (c->ranked)
    return set_err(c, HPLP_EINVAL, "hx_trace_reduced_costs: a rank stores only its blocks (the trace ring classifies)");
  std::vector<double> cv(static_cast<size_t>(c->n));
  if (int r = hx_trace_extras(c, rc, cv.data(), nullptr)) return r;
  for (int64_t j = 0; j < c->n; ++j) rc[j] = cv[j] + rc[j];  // lp.c + sr.at_y (src/solver.cpp:278-279)
  return HPLP_OK;
}

int hx_trace_extras(hx_ctx* c, double* aty, double* c_out, double* cand_norm_normalized) {
  if (!c->setup_done) return set_err(c, HPLP_ESTATE, "hx_trace_extras: no solve state");
  if (c->ranked && (aty || c_out))
    return set_err(c, HPLP_EINVAL, "hx_trace_extras: a rank stores only its blocks (hx_trace_reduced_costs)");
  const Ctl& C = c->h;
  cudaStream_t s = c->stream;
  if (aty || c_out) {
    const double* src;
    if (C.last_cand_avg >= 0) {  // averaged baselines: the mean of A^T y (src/solver.cpp:452-454)
      src = c->tavg + static_cast<size_t>(C.last_cand_avg) * c->n;
    } else {
      double* dout = c->upool;
      if (int r2 = assemble_y(c, C.last_y)) return r2;
      int rc = spmv_dev(c, true, ybuf2(c, C.last_y, C.last_y_avg), dout);
      if (rc) return rc;
      src = dout;
    }
    if (aty && c->n) HX_CUDA(c, cudaMemcpyAsync(aty, src, c->n * sizeof(double), cudaMemcpyDeviceToHost, s));
    if (c_out && c->n) HX_CUDA(c, cudaMemcpyAsync(c_out, c->c, c->n * sizeof(double), cudaMemcpyDeviceToHost, s));
  }
  if (cand_norm_normalized) {
    *cand_norm_normalized = std::numeric_limits<double>::quiet_NaN();
    if (C.last_k >= 1 && !c->ranked && C.scheme == HPLP_SCHEME_RHPDHG) {
      const double scale = 2.0 / static_cast<double>(C.last_k);
      cand_norm_kernel<<<c->grid, kThreads, 0, s>>>(static_cast<int>(c->m), static_cast<int>(c->n), scale,
                                                    xbuf(c, C.last_zx), xbuf(c, C.last_xa), ybuf(c, C.last_y),
                                                    ybuf(c, C.last_ya), axbuf(c, C.last_ax), axbuf(c, C.last_axa),
                                                    c->slots);
      final_reduce_kernel<<<1, 256, 0, s>>>(c->slots, c->grid, 3, c->scratch);
      c->launches += 2;
      double t[3];
      HX_CUDA(c, cudaMemcpyAsync(t, c->scratch, sizeof(t), cudaMemcpyDeviceToHost, s));
      HX_CUDA(c, cudaStreamSynchronize(s));
      // canonical_norm_with_product, src/pdhg_core.cpp:37-51
      const double eta = C.r.eta;
      const double q = t[0] / eta - 2.0 * t[2] + t[1] / eta;
      if (q >= 0.0) *cand_norm_normalized = std::sqrt(q);
      else if (q >= -1e-9 * ((t[0] + t[1]) / eta)) *cand_norm_normalized = 0.0;
    }
  }
  HX_CUDA(c, cudaStreamSynchronize(s));
  return HPLP_OK;
}

int hx_kkt_current(hx_ctx* c, hplp_kkt_t* out) {
  if (!c->setup_done) return set_err(c, HPLP_ESTATE, "hx_kkt_current: no solve state");
  if (c->ranked) {
    // a team: kModeKkt -- each rank's rows / columns with fresh products
    // gathered from its pools (the x / y entries it reads were pushed to it),
    // totals over every rank's records
    std::vector<hx_ctx*> ranks;
    if (int rc = team_ranks(c, ranks)) return rc;
    for (hx_ctx* r : ranks) r->h.mode = kModeKkt;
    const int rc = team_mode_launch(c, ranks);
    for (hx_ctx* r : ranks) r->h.mode = kModeLoop;
    if (rc) return rc;
    const double* t = c->h.kk_tot;
    out->primal_residual = std::sqrt(t[0]) / (1.0 + c->b_norm);
    out->dual_residual = std::sqrt(t[1]) / (1.0 + c->c_norm);
    out->gap_residual = std::fabs(t[2] + t[3]) / (1.0 + std::fabs(t[2]) + std::fabs(t[3]));
    out->max_relative = std::max({out->primal_residual, out->dual_residual, out->gap_residual});
    return HPLP_OK;
  }
  const Ctl& C = c->h;
  cudaStream_t s = c->stream;
  // current z: materialize x into u-scratch, y from its buffer
  double* xcur = c->upool;
  double* aty = c->upool + c->n;
  double* ax = c->upool + 2 * c->n;
  if (int rc = assemble_x(c, C.r.x_src)) return rc;
  if (int rc = assemble_x(c, C.r.x_anchor)) return rc;
  if (int rc = assemble_y(c, C.r.y_cur)) return rc;
  const double* ycur = ybuf2(c, C.r.y_cur, C.r.y_cur_avg);
  if (C.r.x_mode == 0) {
    HX_CUDA(c, cudaMemcpyAsync(xcur, xbuf2(c, C.r.x_src, C.r.x_src_avg), c->n * sizeof(double),
                               cudaMemcpyDeviceToDevice, s));
  } else {
    combine_kernel<<<4 * c->sm_count, 256, 0, s>>>(static_cast<int>(c->n), C.r.w_x, xbuf(c, C.r.x_src),
                                                   xbuf(c, C.r.x_anchor), xcur);
    c->launches += 1;
  }
  int rc = spmv_dev(c, false, xcur, ax);
  if (rc) return rc;
  rc = spmv_dev(c, true, ycur, aty);
  if (rc) return rc;
  kkt_partials_kernel<<<c->grid, kThreads, 0, s>>>(static_cast<int>(c->m), static_cast<int>(c->n), ax, c->b, aty,
                                                   c->c, xcur, ycur, c->slots, c->ub);
  final_reduce_kernel<<<1, 256, 0, s>>>(c->slots, c->grid, 7, c->scratch);
  c->launches += 2;
  double tot[7];
  HX_CUDA(c, cudaMemcpyAsync(tot, c->scratch, sizeof(tot), cudaMemcpyDeviceToHost, s));
  HX_CUDA(c, cudaStreamSynchronize(s));
  // kkt_error_with_products, src/pdhg_core.cpp:57-68 (scalar epilogue); box
  // form: b^T y + sum u_j [-(c + A^T y)_j]^+ in the gap (tot[6] = 0 otherwise)
  out->primal_residual = std::sqrt(tot[0]) / (1.0 + c->b_norm);
  out->dual_residual = std::sqrt(tot[1]) / (1.0 + c->c_norm);
  out->gap_residual = std::fabs(tot[2] + (tot[3] + tot[6])) / (1.0 + std::fabs(tot[2]) + std::fabs(tot[3] + tot[6]));
  out->max_relative = std::max({out->primal_residual, out->dual_residual, out->gap_residual});
  return HPLP_OK;
}

// Phase timers (HX_PROFILE=1): out[grid * 16] accumulated SM cycles per CTA
// (slots listed in hplp.py HX.phase_profile), then -- in an HX_WPROF build
// only -- per-warp SpMV cycles of phase A [grid * kWarps] and phase B.
int hx_sched_tasks(hx_ctx* c, int32_t which, int32_t* out, int64_t capacity, int64_t* count) {
  if (!c->uploaded) return set_err(c, HPLP_ESTATE, "hx_sched_tasks: no problem uploaded");
  const DevSched& d = which == 0 ? c->sa : c->st;
  const int64_t nt = d.view.n_tasks;
  if (count) *count = nt;
  if (out && capacity > 0)
    HX_CUDA(c, cudaMemcpy(out, d.tasks, static_cast<size_t>(std::min(capacity, nt)) * sizeof(int4),
                          cudaMemcpyDeviceToHost));
  return HPLP_OK;
}

int hx_profile(hx_ctx* c, unsigned long long* out, int32_t reset) {
  if (!c->prof) return set_err(c, HPLP_ESTATE, "hx_profile: set HX_PROFILE=1 before hx_create");
  const size_t words = static_cast<size_t>(c->grid) * kProfWords;
  HX_CUDA(c, cudaMemcpy(out, c->prof, words * sizeof(unsigned long long), cudaMemcpyDeviceToHost));
  if (reset) HX_CUDA(c, cudaMemset(c->prof, 0, words * sizeof(unsigned long long)));
  return HPLP_OK;
}

// Microbenchmark: reps x (A x or A^T y) on device-resident random vectors,
// CUDA-event timed on the context stream; *ms = mean per SpMV.
int hx_bench_spmv(hx_ctx* c, int32_t transpose, int32_t reps, double* ms) {
  if (!c->uploaded) return set_err(c, HPLP_ESTATE, "hx_bench_spmv: no problem uploaded");
  double* in = transpose ? c->upool + 2 * c->n : c->upool;
  double* out = transpose ? c->upool : c->upool + 2 * c->n;
  HX_CUDA(c, cudaMemsetAsync(in, 0, (transpose ? c->m : c->n) * sizeof(double), c->stream));
  int rc = spmv_dev(c, transpose != 0, in, out);
  if (rc) return rc;
  HX_CUDA(c, cudaEventRecord(c->ev0, c->stream));
  for (int r = 0; r < reps; ++r) {
    rc = spmv_dev(c, transpose != 0, in, out);
    if (rc) return rc;
  }
  HX_CUDA(c, cudaEventRecord(c->ev1, c->stream));
  HX_CUDA(c, cudaEventSynchronize(c->ev1));
  float t = 0.f;
  HX_CUDA(c, cudaEventElapsedTime(&t, c->ev0, c->ev1));
  *ms = t / reps;
  return HPLP_OK;
}

int64_t hx_sizeof(int32_t which) {
  switch (which) {
    case 0: return sizeof(hplp_config_t);
    case 1: return sizeof(hplp_result_t);
    case 2: return sizeof(hplp_io_t);
    case 3: return sizeof(hplp_epoch_t);
    case 4: return sizeof(hplp_trace_t);
    case 5: return sizeof(hplp_general_t);
    case 6: return sizeof(hx_progress_t);
    default: return -1;
  }
}

}  // extern "C"
