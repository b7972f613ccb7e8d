// nnz-balanced warp schedule for the fused SpMV phases (host side).
//
// Rows of length <= kStreamRowMax are packed into stream tasks of at most
// kChunk nonzeros / kStreamRowsMax rows; every longer row is cut into pieces
// of at most kChunk nonzeros (a single piece when it fits), grouped into runs
// of consecutive pieces that one warp processes back to back.  The units
// (a stream task, a run) are then dealt heaviest first, each to the
// least-loaded CTA and within it to the least-loaded warp (cost = nnz +
// kRowCost per row + kTaskCost per task).  Static and deterministic: the same
// matrix and grid always give the same row -> (warp, lane) map, which is what
// makes every reduction in the solver reproducible bit for bit.
#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <functional>
#include <queue>
#include <thread>

#include "hx_internal.cuh"

namespace hx {

namespace {

// One segment of rows packed into tasks (build_schedule): positions, slots and
// long-row counters are local to the segment; build_schedule shifts them.
struct Packed {
  std::vector<int4> tasks, meta;
  std::vector<double> cost;
  std::vector<std::size_t> unit;  // first task of each dealing unit (a stream task or a run of pieces)
  int n_slots = 0, n_long = 0;
  int64_t off = 0;  // pad slots inserted in the segment
};

struct PackArgs {
  const int* ptr_in;
  int stagger, stagger_lmin;
  int align;  // staggered copy: every task starts at a multiple of `align` slots (0: anywhere)
  int64_t task_nnz;
  bool exact;
  double row_cost, task_cost, run_budget;
  int* padded;  // padded row starts (segment-local pad offsets), or null
};

void pack_rows(const PackArgs& a, int ra, int rb, Packed& o) {
  const int* ptr_in = a.ptr_in;
  const int stagger = a.stagger;
  int64_t& off = o.off;
  auto pstart = [&](int row) -> int64_t { return ptr_in[row] + off; };  // row's start in the padded copy
  auto place = [&](int row) {
    if (stagger && row < rb) a.padded[row] = static_cast<int>(pstart(row));
  };
  auto push = [&](int r0, int r1, int kind, int64_t p0, int64_t p1, int4 meta, double c) {
    o.tasks.push_back(int4{r0, task_y(r1, kind), static_cast<int>(p0), static_cast<int>(p1)});
    o.meta.push_back(meta);
    o.cost.push_back(c + a.task_cost);
  };
  // a task's first slot on a multiple of a.align (its idx / val streams then
  // touch the fewest 128-byte lines); the gap trails the previous task's last
  // row, whose sum the kernels clamp to its task's end
  auto align_at = [&](int row) {
    if (stagger && a.align) {
      const int64_t rem = (ptr_in[row] + off) % a.align;
      if (rem) off += a.align - rem;
    }
  };
  int r = ra;
  while (r < rb) {
    const int64_t len = ptr_in[r + 1] - ptr_in[r];
    align_at(r);
    place(r);
    if (len > kStreamRowMax) {
      const int np = static_cast<int>((len + kTaskNnz - 1) / kTaskNnz);
      // exact order: lane 0 adds every product in sequence, about as long
      // again as the gathers -- the piece costs twice as much
      const double pc = static_cast<double>(len) / np * (a.exact ? 2.0 : 1.0) + a.task_cost;
      const int per = std::max(1, std::min(kRunMax, static_cast<int>(a.run_budget / pc)));
      const int nr = a.exact ? 1 : (np + per - 1) / per;
      const int64_t base = stagger ? pstart(r) : ptr_in[r];
      for (int k = 0; k < nr; ++k) {
        o.unit.push_back(o.tasks.size());
        const int q0 = static_cast<int>(static_cast<int64_t>(np) * k / nr);
        const int q1 = static_cast<int>(static_cast<int64_t>(np) * (k + 1) / nr);
        for (int q = q0; q < q1; ++q) {
          // equal pieces; in an aligned staggered copy, pieces of kTaskNnz
          // slots from the aligned row start (the last one shorter), so every
          // piece's streams start on a line
          const bool al = stagger && a.align;
          const int64_t p0 = base + (al ? std::min<int64_t>(len, int64_t{kTaskNnz} * q) : len * q / np);
          const int64_t p1 = base + (al ? std::min<int64_t>(len, int64_t{kTaskNnz} * (q + 1)) : len * (q + 1) / np);
          push(r, r + 1, q + 1 == q1 ? kTaskPiece : kTaskPieceRun, p0, p1,
               int4{o.n_slots + k, nr, nr > 1 ? o.n_long : -1, k},
               static_cast<double>(p1 - p0) * (a.exact ? 2.0 : 1.0) + (q + 1 == np ? a.row_cost : 0.0));
        }
      }
      if (nr > 1) {
        o.n_slots += nr;
        o.n_long += 1;
      }
      ++r;
      continue;
    }
    const int r0 = r;
    const int64_t p0 = stagger ? pstart(r0) : ptr_in[r0];
    int64_t used = 0;  // slots (nonzeros + pads)
    int64_t nz = 0;
    int starts[4][16];  // per half-warp group: how many rows start on each bank pair
    if (stagger) std::fill(&starts[0][0], &starts[0][0] + 64, 0);
    // aligned copy: a task that fills up by rows ends on a multiple of 32
    // rows, so a run of short rows (slack columns, bound rows) is cut into
    // tasks whose epilogue vectors start on a 256-byte boundary
    const int row_end = stagger && a.align && (r0 + kStreamRowsMax) / 32 * 32 > r0
                            ? (r0 + kStreamRowsMax) / 32 * 32
                            : r0 + kStreamRowsMax;
    while (r < rb && r < row_end) {
      const int64_t l = ptr_in[r + 1] - ptr_in[r];
      if (l > kStreamRowMax) break;
      int pad = 0;
      const int g = (r - r0) >> 4;  // lanes 0-15, 16-31 (first rows), 32-47, 48-63 (second rows)
      if (stagger && r > r0 && l >= a.stagger_lmin) {
        // the fewest pads reaching the least-used bank pair within reach
        int best = 1 << 30;
        for (int p = 0; p <= stagger; ++p) {
          const int c = starts[g][(used + p) & 15];
          if (c < best) best = c, pad = p;
          if (c == 0) break;
        }
      }
      if (used + pad + l > a.task_nnz) break;
      off += pad;
      used += pad;
      place(r);
      if (stagger) ++starts[g][used & 15];
      used += l;
      nz += l;
      ++r;
    }
    place(r);
    o.unit.push_back(o.tasks.size());
    push(r0, r, kTaskStream, p0, stagger ? pstart(r) : ptr_in[r], int4{0, 0, 0, 0},
         static_cast<double>(stagger ? used : nz) + a.row_cost * (r - r0));
  }
  // the segment's pads a multiple of a.align, so later segments keep theirs
  if (stagger && a.align && off % a.align) off += a.align - off % a.align;
}

}  // namespace

SchedHost build_schedule(const int* ptr_in, int rows, int warps, double lead, double row_cost, double task_cost,
                         bool exact, int stagger, int stagger_lmin, int align) {
  SchedHost s;
  // Bank-staggered layout: positions in a padded copy of the matrix; pads only
  // ever go in front of a non-first row of a stream task, and every task
  // refers to the padded positions.  ptr_in[0] must be 0 (a rank's block is
  // never staggered).
  stagger = ptr_in[0] == 0 ? std::max(0, std::min(stagger, 15)) : 0;
  // padded positions stay int32: at most `stagger` pads per row
  align = stagger ? std::max(0, std::min(align, 64)) : 0;
  if (static_cast<int64_t>(ptr_in[rows]) + static_cast<int64_t>(stagger + align) * rows + kMatrixPad >=
      (int64_t{1} << 31) - 1)
    stagger = align = 0;
  std::vector<int> padded;
  if (stagger) padded.assign(static_cast<std::size_t>(rows) + 1, 0);
  const int64_t nnz = ptr_in[rows] - ptr_in[0];  // ptr may point into a larger matrix (a rank's block)
  const double total = static_cast<double>(nnz) + row_cost * rows;
  int64_t task_nnz = kTaskNnz;
  if (const char* e = std::getenv("HX_TASK_NNZ")) task_nnz = std::max(8, std::min<int>(kTaskNnz, std::atoi(e)));
  // a run of pieces is dealt to one warp as a unit: at most 1/kRunFrac of the
  // mean warp cost, so the dealing stays balanced
  const PackArgs pa{ptr_in, stagger, stagger_lmin, align, task_nnz, exact, row_cost, task_cost,
                    std::max(1.0, total / warps / kRunFrac), stagger ? padded.data() : nullptr};
  // Packing runs on kPackSegments host threads for large matrices: segment k
  // starts at the first row at or past nonzero k * nnz / K (a fixed split, so
  // the schedule does not depend on the host); a segment boundary also ends a
  // stream task.
  const int K = rows >= kPackMinRows ? kPackSegments : 1;
  std::vector<int> seg(static_cast<std::size_t>(K) + 1, rows);
  seg[0] = 0;
  for (int k = 1; k < K; ++k) {
    const int64_t target = ptr_in[0] + nnz * k / K;
    seg[k] = std::max(seg[k - 1], static_cast<int>(std::lower_bound(ptr_in, ptr_in + rows + 1, target) - ptr_in));
    seg[k] = std::min(seg[k], rows);
  }
  std::vector<Packed> part(static_cast<std::size_t>(K));
  {
    std::vector<std::thread> pool;
    for (int k = 1; k < K; ++k) pool.emplace_back([&, k] { pack_rows(pa, seg[k], seg[k + 1], part[k]); });
    pack_rows(pa, seg[0], seg[1], part[0]);
    for (auto& t : pool) t.join();
  }
  // concatenate: shift positions by the pads of earlier segments, long-row
  // slots / counters by theirs, unit starts by their task counts
  std::vector<double> cost;
  std::vector<std::size_t> unit;
  int64_t off = 0;
  for (int k = 0; k < K; ++k) {
    Packed& p = part[k];
    const std::size_t tb = s.tasks.size();
    for (std::size_t t = 0; t < p.tasks.size(); ++t) {
      int4 tk = p.tasks[t];
      int4 mt = p.meta[t];
      tk.z = static_cast<int>(tk.z + off);
      tk.w = static_cast<int>(tk.w + off);
      if (task_kind(tk.y) != kTaskStream) {
        mt.x += s.n_slots;
        if (mt.z >= 0) mt.z += s.n_long;
      }
      s.tasks.push_back(tk);
      s.meta.push_back(mt);
    }
    cost.insert(cost.end(), p.cost.begin(), p.cost.end());
    for (std::size_t u : p.unit) unit.push_back(u + tb);
    if (stagger && off)
      for (int r = seg[k]; r < seg[k + 1]; ++r) padded[r] = static_cast<int>(padded[r] + off);
    s.n_slots += p.n_slots;
    s.n_long += p.n_long;
    off += p.off;
  }
  const std::size_t nt = s.tasks.size();
  unit.push_back(nt);
  if (stagger) {
    padded[rows] = static_cast<int>(ptr_in[rows] + off);
    s.padded_nnz = ptr_in[rows] + off;
    s.pptr.swap(padded);
  }

  // Longest-processing-time dealing: units heaviest first, each to the
  // currently least-loaded CTA, then its least-loaded warp (ties to the lower
  // id).  Warp w's tasks are laid out at positions w, w + W, w + 2W, ...
  // (padded with empty tasks), which is how the kernels walk them; a run's
  // pieces stay consecutive.
  // Deterministic and balanced; reductions stay fixed-order because every row
  // keeps one (warp, lane) owner.
  const std::size_t nu = unit.size() - 1;
  std::vector<double> ucost(nu, 0.0);
  for (std::size_t u = 0; u < nu; ++u)
    for (std::size_t t = unit[u]; t < unit[u + 1]; ++t) ucost[u] += cost[t];
  std::vector<int> order(nu);
  for (std::size_t u = 0; u < nu; ++u) order[u] = static_cast<int>(u);
  std::stable_sort(order.begin(), order.end(), [&](int a, int b) { return ucost[a] > ucost[b]; });
  using Load = std::pair<double, int>;  // (load, warp)
  std::priority_queue<Load, std::vector<Load>, std::greater<Load>> heap;
  std::vector<int> uwarp(nu);  // the warp each unit is dealt to
  std::vector<double> wcost(static_cast<std::size_t>(warps), 0.0);
  for (int w = 0; w < warps; ++w) wcost[w] = w % kWarps == 0 ? lead : 0.0;
  int deal = 1;
  if (const char* e = std::getenv("HX_DEAL")) deal = std::atoi(e);
  if (deal == 1 && warps % kWarps == 0) {
    // two levels: each unit to the least-loaded CTA (the SM's warps share its
    // load/store pipes, so CTA sums set the phase time as much as the
    // longest warp), then to that CTA's least-loaded warp.  Against dealing
    // to the least-loaded warp alone (HX_DEAL=0; CTA sums up to 17% apart on
    // configs[1]'s A^T): configs[1] 27.45k -> 28.29k it/s, configs[2] 42.9k
    // -> 47.9k.  HX_TASK_NNZ (a smaller cap on a stream task's nonzeros)
    // measured slower at every cap: 224 / 192 / 128 -> 25.9k / 24.3k / 22.2k.
    const int grid = warps / kWarps;
    std::vector<double> ccost(static_cast<std::size_t>(grid), 0.0);
    for (int c = 0; c < grid; ++c) heap.push({0.0, c});
    for (int u : order) {
      auto [load, c] = heap.top();
      heap.pop();
      int w = c * kWarps;
      for (int i = 1; i < kWarps; ++i)
        if (wcost[c * kWarps + i] < wcost[w]) w = c * kWarps + i;
      uwarp[u] = w;
      wcost[w] += ucost[u];
      ccost[c] = load + ucost[u];
      heap.push({ccost[c], c});
    }
  } else {
    for (int w = 0; w < warps; ++w) heap.push({wcost[w], w});
    for (int u : order) {
      auto [load, w] = heap.top();
      heap.pop();
      uwarp[u] = w;
      wcost[w] = load + ucost[u];
      heap.push({wcost[w], w});
    }
  }
  // warp w's k-th task (in dealing order) goes to position k * warps + w
  std::vector<std::size_t> wpos(static_cast<std::size_t>(warps), 0);
  for (std::size_t u = 0; u < nu; ++u) wpos[uwarp[u]] += unit[u + 1] - unit[u];
  std::size_t rounds = 0;
  for (std::size_t v : wpos) rounds = std::max(rounds, v);
  std::fill(wpos.begin(), wpos.end(), 0);
  std::vector<int4> tasks(rounds * warps, int4{0, 0, 0, 0}), meta(rounds * warps, int4{0, 0, 0, 0});
  for (int u : order) {
    const int w = uwarp[u];
    for (std::size_t t = unit[u]; t < unit[u + 1]; ++t) {
      const std::size_t k = wpos[w]++;
      tasks[k * warps + w] = s.tasks[t];
      meta[k * warps + w] = s.meta[t];
    }
  }
  while (!tasks.empty() && tasks.back().x == 0 && tasks.back().y == 0 && tasks.back().w == 0) {
    tasks.pop_back();
    meta.pop_back();
  }
  s.tasks.swap(tasks);
  s.meta.swap(meta);
  // owner CTA of every long row = the CTA whose warp runs its piece 0
  const int grid = warps / kWarps;
  std::vector<int> owner(static_cast<std::size_t>(s.n_long), 0);
  for (std::size_t k = 0; k < s.tasks.size(); ++k) {
    const int4& tk = s.tasks[k];
    const int4& mt = s.meta[k];
    if (task_kind(tk.y) == kTaskPiece && mt.y > 1 && mt.w == 0)
      owner[mt.z] = static_cast<int>(k % static_cast<std::size_t>(warps)) / kWarps;
  }
  s.owned_ptr.assign(static_cast<std::size_t>(grid) + 1, 0);
  for (int l = 0; l < s.n_long; ++l) ++s.owned_ptr[owner[l] + 1];
  for (int c = 0; c < grid; ++c) s.owned_ptr[c + 1] += s.owned_ptr[c];
  s.owned_idx.assign(static_cast<std::size_t>(s.n_long), 0);
  std::vector<int> fill(s.owned_ptr.begin(), s.owned_ptr.end() - 1);
  for (int l = 0; l < s.n_long; ++l) s.owned_idx[fill[owner[l]]++] = l;
  double mx = 0.0;
  for (int w = 0; w < warps; ++w) mx = std::max(mx, wcost[w] - (w % kWarps == 0 ? lead : 0.0));
  s.max_warp_cost = mx;
  s.mean_warp_cost = total / warps;
  return s;
}

}  // namespace hx
