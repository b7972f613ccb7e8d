// Internal declarations shared by the hx CUDA translation units.
#pragma once

#include <cuda_runtime.h>

#include <cstdint>
#include <string>
#include <vector>

#include "hplp_types.h"
#include "hx.h"

namespace hx {

constexpr int kThreads = 512;              // threads per CTA of every hx kernel
constexpr int kWarps = kThreads / 32;
constexpr int kMaxQ = 16;                  // reduction quantities per phase
constexpr int kXPool = 6;                  // n-vectors: iterates, anchors, best, T(z)
constexpr int kYPool = 6;                  // m-vectors: y, anchors, best, T(z), combos
constexpr int kAxPool = 4;                 // m-vectors: A x carried / anchor / products
constexpr int kEpochCap = 1 << 16;         // device epoch ring (host drains per hx_run)
constexpr double kRowCost = 3.0;           // epilogue cost of one row in nnz units

// A warp-task of consecutive rows handled with vector width 1 << log2v.
// (int4: row_begin, row_end, log2v, unused)
// A piece of one long row; the last piece to finish reduces the pieces in
// index order and runs the row's epilogue (deterministic).
struct Piece {
  int row, p0, p1, slot, npieces, counter, index, pad;
};

// Device view of one CSR matrix plus its nnz-balanced warp schedule.
struct Sched {
  int rows = 0;
  int cols = 0;
  const int* ptr = nullptr;
  const int* idx = nullptr;
  const double* val = nullptr;
  const int4* tasks = nullptr;
  const int* task_ptr = nullptr;   // [warps + 1]
  const Piece* pieces = nullptr;
  const int* piece_ptr = nullptr;  // [warps + 1]
  int n_long = 0;
  double* piece_part[2] = {nullptr, nullptr};   // per concurrent SpMV lane
  unsigned* piece_cnt[2] = {nullptr, nullptr};
  double* long_terms[2] = {nullptr, nullptr};   // [n_long * kMaxQ]
};

// Host-side schedule before upload.
struct SchedHost {
  std::vector<int4> tasks;
  std::vector<int> task_ptr;
  std::vector<Piece> pieces;
  std::vector<int> piece_ptr;
  int n_long = 0;
  int n_slots = 0;
  double max_warp_cost = 0.0, mean_warp_cost = 0.0;
};

SchedHost build_schedule(const int* ptr_host, int rows, int warps);

}  // namespace hx
