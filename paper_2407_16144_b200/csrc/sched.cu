// nnz-balanced warp schedule for the fused SpMV phases (host side).
//
// Rows are cut into warp-tasks of consecutive rows sharing one vector width
// v in {1,2,4,8,16,32} (a sub-warp of v lanes per row, about two passes per
// row), rows longer than 2P are cut into pieces of about P nonzeros, and the
// row-ordered item list is split into one contiguous slice per warp with
// equal cost (nnz + kRowCost per row).  Static and deterministic: the same
// matrix and grid always give the same row -> (warp, lane) map, which is what
// makes every reduction in the solver reproducible bit for bit.
#include <algorithm>
#include <cmath>

#include "hx_internal.cuh"

namespace hx {

namespace {
int log2_width(int64_t len) {
  if (len <= 2) return 0;
  if (len <= 4) return 1;
  if (len <= 8) return 2;
  if (len <= 16) return 3;
  if (len <= 32) return 4;
  return 5;
}
}  // namespace

SchedHost build_schedule(const int* ptr, int rows, int warps) {
  SchedHost s;
  const int64_t nnz = ptr[rows];
  const double total = static_cast<double>(nnz) + kRowCost * rows;
  const double per_warp = std::max(1.0, total / warps);
  const int64_t piece = static_cast<int64_t>(std::clamp(total / (2.0 * warps), 256.0, 16384.0));
  const int64_t long_len = 2 * piece;
  const double task_max = std::max(64.0, per_warp / 4.0);

  struct Item {
    bool is_piece;
    int index;
    double cost;
  };
  std::vector<Item> items;
  int4 cur{0, 0, -1, 0};
  double cur_cost = 0.0;
  auto close = [&] {
    if (cur.z >= 0 && cur.y > cur.x) {
      items.push_back({false, static_cast<int>(s.tasks.size()), cur_cost});
      s.tasks.push_back(cur);
    }
    cur.z = -1;
    cur_cost = 0.0;
  };
  for (int r = 0; r < rows; ++r) {
    const int64_t len = ptr[r + 1] - ptr[r];
    if (len > long_len) {
      close();
      const int np = static_cast<int>((len + piece - 1) / piece);
      for (int q = 0; q < np; ++q) {
        Piece pc;
        pc.row = r;
        pc.p0 = static_cast<int>(ptr[r] + len * q / np);
        pc.p1 = static_cast<int>(ptr[r] + len * (q + 1) / np);
        pc.slot = s.n_slots + q;
        pc.npieces = np;
        pc.counter = s.n_long;
        pc.index = q;
        pc.pad = 0;
        items.push_back({true, static_cast<int>(s.pieces.size()),
                         static_cast<double>(pc.p1 - pc.p0) + (q + 1 == np ? kRowCost : 0.0)});
        s.pieces.push_back(pc);
      }
      s.n_slots += np;
      s.n_long += 1;
      continue;
    }
    const int lv = log2_width(len);
    const double cost = static_cast<double>(len) + kRowCost;
    const int max_rows = (32 >> lv) * 64;
    if (cur.z != lv || cur_cost + cost > task_max || cur.y - cur.x >= max_rows) {
      close();
      cur = int4{r, r, lv, 0};
    }
    cur.y = r + 1;
    cur_cost += cost;
  }
  close();

  // Contiguous equal-cost slices of the item list, one per warp.
  s.task_ptr.assign(static_cast<std::size_t>(warps) + 1, 0);
  s.piece_ptr.assign(static_cast<std::size_t>(warps) + 1, 0);
  std::vector<double> wcost(static_cast<std::size_t>(warps), 0.0);
  double prefix = 0.0;
  int nt = 0, np = 0;
  int w_prev = 0;
  for (const Item& it : items) {
    const double mid = prefix + 0.5 * it.cost;
    int w = std::min(warps - 1, static_cast<int>(mid / per_warp));
    w = std::max(w, w_prev);  // monotone
    for (int q = w_prev + 1; q <= w; ++q) {
      s.task_ptr[q] = nt;
      s.piece_ptr[q] = np;
    }
    w_prev = w;
    if (it.is_piece) ++np;
    else ++nt;
    wcost[w] += it.cost;
    prefix += it.cost;
  }
  for (int q = w_prev + 1; q <= warps; ++q) {
    s.task_ptr[q] = nt;
    s.piece_ptr[q] = np;
  }
  s.task_ptr[0] = 0;
  s.piece_ptr[0] = 0;
  double mx = 0.0;
  for (double c : wcost) mx = std::max(mx, c);
  s.max_warp_cost = mx;
  s.mean_warp_cost = total / warps;
  return s;
}

}  // namespace hx
