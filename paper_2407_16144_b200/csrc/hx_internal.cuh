// Internal declarations shared by the hx CUDA translation units.
#pragma once

#include <cuda_runtime.h>

#include <cstdint>
#include <string>
#include <vector>

#include "hplp_types.h"
#include "hx.h"

namespace hx {

#ifndef HX_THREADS
#define HX_THREADS 512
#endif
constexpr int kThreads = HX_THREADS;              // threads per CTA of every hx kernel
constexpr int kWarps = kThreads / 32;
// One 512-thread CTA per SM with a 128-register budget and every phase
// inlined: measured fastest on B200 (no spills -- spill reloads after each
// grid barrier's L1 invalidation cost an L2 round trip).
#ifndef HX_MIN_BLOCKS
#define HX_MIN_BLOCKS 1
#endif
constexpr int kMinBlocks = HX_MIN_BLOCKS;         // resident CTAs per SM the register budget targets
#ifndef HX_PHASE_INLINE
#define HX_PHASE_INLINE __forceinline__
#endif
constexpr int kMaxQ = 16;                  // reduction quantities per phase
constexpr int kXPool = 7;                  // n-vectors: iterates, anchors, best, T(z), speculative outputs
constexpr int kYPool = 6;                  // m-vectors: y, anchors, best, T(z), combos
constexpr int kAxPool = 4;                 // m-vectors: A x carried / anchor / products
constexpr int kAvgPool = 4;                // running-average slots (baseline schemes): current, new, best, restart point
constexpr int kEpochCap = 1 << 16;         // device epoch ring (host drains per hx_run)
// Schedule cost model (nnz units).  With CTA-first dealing (sched.cu),
// tools/cost_sweep.sh on configs[1] / [2]: row cost 2 / 3 / 5 / 7 / 10 ->
// 27.2k / 28.3k / 28.5k / 28.5k / 28.0k and 46.9k / 47.9k / 48.9k / 48.9k /
// 47.3k it/s (phase A sets it; phase B is flat from 5 to 10); the task cost
// is flat from 32 to 200.
constexpr double kRowCost = 5.0;           // epilogue cost of one row
constexpr double kTaskCost = 64.0;         // fixed latency cost of one warp task
// bank-staggered stream tasks (build_schedule stagger): pad slots allowed in
// front of a row of A (phase B) / of A^T (phase A), and the shortest row
// that gets any
constexpr int kStaggerA = 15;
constexpr int kStaggerT = 1;
constexpr int kStaggerLmin = 4;
constexpr int kTaskAlign = 32;  // staggered copy: task starts on multiples of 32 slots (HX_ALIGN)
constexpr int64_t kStaggerMaxNnz = int64_t{1} << 29;  // larger matrices keep the plain layout
// build_schedule packs the rows of a matrix with >= kPackMinRows rows in
// kPackSegments fixed segments on host threads
constexpr int kPackSegments = 8;
constexpr int kPackMinRows = 1 << 16;
// Warp 0 of every CTA runs the controller while warps 1..15 start the
// speculative phase A: its schedule share starts with this lead (cost
// units).  tools/lead_sweep.sh with CTA-first dealing, configs[1]: 600 / 1200
// / 2200 / 3000 / 6000 / no tasks -> 27.99k / 28.54k / 28.70k / 28.70k /
// 28.69k / 28.67k it/s (configs[0], [2] flat from 900 on).
constexpr double kLead = 3000.0;
#ifndef HX_LOADS
#define HX_LOADS 8
#endif
// Row sums of stream tasks: 0 one sequential sum in ascending column order
// (the reference's exact order), 1 two interleaved partial sums (even / odd
// positions) added at the end, 2 four, 3 two with loads 8 ahead.  Measured on
// configs[1] (tools/quick_rate.py): 26.81k / 27.86k / 27.47k / 26.97k it/s.
// Reading 1's products as 16-byte pairs (LDS.128, same sums): 27.23k vs
// 27.76k (8 B of spills), not kept.  4: 1's order, software-pipelined (the
// next four products loaded before the current four are added; bit-identical
// sums): 29.77k vs 29.65k on configs[1], configs[2] flat -- kept.
// HX_RSHORT=1 (a lane's two rows of <= 4 nonzeros loaded in one round):
// configs[1] 29.68k vs 29.77k, configs[2] 49.9k vs 50.7k, not kept.
#ifndef HX_RSUM
#define HX_RSUM 4
#endif
// Pieces of long rows: 1 pairwise tree over each lane's products, 0 one
// sequential chain (then a warp tree either way).
#ifndef HX_PSUM
#define HX_PSUM 1
#endif
// 1: tasks of <= 16 rows sum each row on two lanes (head / tail half):
// 23.7k it/s on configs[1] (register spills + shuffle), not used.
#ifndef HX_EPI_EF
#define HX_EPI_EF 0
#endif
#ifndef HX_GATHER_LAST
#define HX_GATHER_LAST 1
#endif
// Grid barrier polls: 1 relaxed loads then one acquire load (configs[1]
// 27.89k vs 27.79k it/s, configs[2] 44.4k vs 44.2k), 0 an acquire load per poll.
#ifndef HX_BAR_RELAXED
#define HX_BAR_RELAXED 1
#endif
#ifndef HX_RSHORT
#define HX_RSHORT 0
#endif
#ifndef HX_RSPLIT
#define HX_RSPLIT 0
#endif
constexpr int kLoadsPerLane = HX_LOADS;    // nonzeros per lane per task
constexpr int kChunk = 32 * kLoadsPerLane; // nonzero slots per warp task (256)
// Vectorised idx/val loads (int2 / double2 from an even-aligned window, see
// load_task): 1 on, 0 scalar loads.
#ifndef HX_VEC
#define HX_VEC 0
#endif
constexpr int kTaskNnz = HX_VEC ? kChunk - 1 : kChunk;  // max nonzeros per warp task
constexpr int kMatrixPad = 4;              // padding elements after idx / val (vector loads)
constexpr int kStreamRowMax = 64;          // rows up to this length are summed lane-per-row
#ifndef HX_ROWS
#define HX_ROWS 64
#endif
// 32 (one row per lane, fewer registers): configs[1] 25.7k vs 27.7k it/s,
// configs[2] 45.4k vs 44.2k -- 64 kept.
constexpr int kStreamRowsMax = HX_ROWS;    // rows per stream task (64: two per lane)
constexpr int kMaxRanks = 8;               // ranks of a row-partitioned team (one node)
constexpr int kMaxColBlocks = 8;           // column blocks of phase B (loop_kernel_stream_cb)

// Warp tasks, int4 {row_begin, row_end | kind << 30, p_begin, p_end}; every
// task covers at most kChunk nonzeros, loaded kLoadsPerLane per lane into
// registers with independent loads and gathers (shared memory only holds a
// 2 KB product buffer per warp, so L1 keeps its capacity for the gathers);
// warp w runs tasks w, w + W, w + 2W, ... (static round robin):
//   kTaskStream: consecutive short rows, summed lane-per-row over ascending
//                columns (the reference's order, src/sparse_matrix.cpp:108-115,
//                as two interleaved partial sums: HX_RSUM);
//   kTaskPiece:  a slice of one longer row; meta[t] = {slot, npieces,
//                counter, index}.  A single-piece row is finished in place;
//                otherwise the last piece to finish reduces the pieces in
//                index order and runs the row's epilogue (deterministic).
//   kTaskPieceRun: a piece that is not the last of its run -- a long row's
//                consecutive pieces are dealt to one warp in runs, which
//                carries the run's partial sum in registers; only the run's
//                last piece (kTaskPiece) publishes it, so a run of r pieces
//                costs one fence + atomic instead of r (configs[4]'s Zipf rows).
enum TaskKind : int { kTaskStream = 0, kTaskPiece = 1, kTaskPieceRun = 2 };
constexpr int kKindShift = 30;
constexpr int kRowMask = (1 << kKindShift) - 1;
__host__ __device__ __forceinline__ int task_kind(int y) {
  return static_cast<int>(static_cast<unsigned>(y) >> kKindShift);
}
__host__ __device__ __forceinline__ int task_y(int row_end, int kind) {
  return static_cast<int>(static_cast<unsigned>(row_end) | (static_cast<unsigned>(kind) << kKindShift));
}
// A run's cost is at most the mean warp cost / kRunFrac (balance), and at
// most kRunMax pieces.  Measured (tools/big_configs.py): kRunFrac 2 / 3 / 4 /
// 8 / no runs -> configs[3] 9.26k / 9.39k / 8.81k / 7.64k / 7.64k it/s,
// configs[4] 512 / 510 / 511 / 512 / 405 it/s.
#ifndef HX_RUN_FRAC
#define HX_RUN_FRAC 3.0
#endif
constexpr double kRunFrac = HX_RUN_FRAC;
constexpr int kRunMax = 64;

// Device view of one CSR matrix plus its nnz-balanced warp schedule.
struct Sched {
  int rows = 0;
  int cols = 0;
  int W = 0;                       // warps the schedule was dealt to (CTAs * kWarps)
  const int* ptr = nullptr;
  const int* idx = nullptr;
  const double* val = nullptr;
  const int4* tasks = nullptr;
  const int4* meta = nullptr;      // piece tasks: {slot, npieces, counter, index}
  int n_tasks = 0;
  int n_long = 0;
  int stream_hint = 0;             // 1: idx/val loaded evict_first (working set > L2; hx_upload_csr)
  int row_limit = 0;               // dimension of the output vector (bounds checks in HX_CHECKED builds)
  // 1: reference summation order (hx_set_sum_order): every row summed as one
  // sequential chain in ascending index order, exactly the reference's
  // `acc += value * x[col]` (src/sparse_matrix.cpp:108-115, :127-134), so row
  // sums are bit-identical to it; long rows are one run of pieces whose
  // products lane 0 adds in order.  0: the fast order (two interleaved
  // partial sums per short row, lane-strided partials + trees for long rows).
  int exact = 0;
  int pad_exact = 0;
  // Long-row scratch per "set" (base + set * stride; no dynamically indexed
  // arrays, which would force the kernel parameters into local memory):
  // sets 0/1 alternate by iteration parity in the main phases, sets 2/3
  // serve the certificate SpMVs.
  double* part_base = nullptr;   // [4][n_slots]
  unsigned* cnt_base = nullptr;  // [4][n_long]
  double* terms_base = nullptr;  // [4][n_long * kMaxQ]
  int n_slots = 0;
  // Each multi-piece ("long") row has a static owner CTA (the one running its
  // piece 0): the last piece to finish publishes the row's epilogue terms and
  // a sequence flag; the owner folds its rows' terms into its own partial
  // record in list order.  owned_idx[owned_ptr[c] .. owned_ptr[c+1]) are the
  // long rows CTA c owns.
  const int* owned_ptr = nullptr;             // [grid + 1]
  const int* owned_idx = nullptr;
  unsigned long long* flag_base = nullptr;    // [4][n_long] phase sequence flags
  __host__ __device__ unsigned long long* long_flag(int set) const {
    return flag_base + static_cast<size_t>(set) * n_long;
  }
  __host__ __device__ double* piece_part(int set) const { return part_base + static_cast<size_t>(set) * n_slots; }
  __host__ __device__ unsigned* piece_cnt(int set) const { return cnt_base + static_cast<size_t>(set) * n_long; }
  __host__ __device__ double* long_terms(int set) const {
    return terms_base + static_cast<size_t>(set) * n_long * kMaxQ;
  }
};

// Host-side schedule before upload.
struct SchedHost {
  std::vector<int4> tasks;
  std::vector<int4> meta;
  std::vector<int> owned_ptr;  // [grid + 1]
  std::vector<int> owned_idx;
  int n_long = 0;
  int n_slots = 0;
  double max_warp_cost = 0.0, mean_warp_cost = 0.0;
  // bank-staggered layout (stagger > 0): padded row pointers [rows + 1]
  // into a copy of idx / val with zero-valued pad slots; every task's
  // positions refer to it (empty: the tasks index the CSR itself)
  std::vector<int> pptr;
  int64_t padded_nnz = 0;
};

// lead: initial load (cost units) of warp 0 of every CTA, which runs the
// controller before its own tasks in the speculative phase A.
// exact: reference summation order -- every long row becomes ONE run of
// pieces (one warp carries the sequential sum through all of them).
// stagger > 0: bank-staggered stream tasks -- before a row of >= stagger_lmin
// nonzeros that is not a task's first, up to `stagger` zero-valued pad slots
// move its first product to a shared-memory bank pair (slot mod 16) no other
// row of its half-warp (16 lanes) starts on, so the lane-per-row sums read
// the product buffer without bank conflicts.  Pads trail the previous row
// (they add +0.0 to its sum: the same bits, since no row sum is -0.0).
SchedHost build_schedule(const int* ptr_host, int rows, int warps, double lead = 0.0, double row_cost = kRowCost,
                         double task_cost = kTaskCost, bool exact = false, int stagger = 0, int stagger_lmin = 4,
                         int align = 0);

}  // namespace hx
