// Run scoring: the reference's minimum-edit-distance
// alignment with its deterministic backtrace (metrics.py:26-61 align: unit
// costs; ties prefer match, then substitution, deletion, insertion) and the
// edit distances WER sums (metrics.py:72-83 compute_wer: S + D + I of each
// pair is its edit distance).  Words arrive as integer ids; the host maps
// strings to ids once, so equality is id equality.
#pragma once
#include <algorithm>
#include <cstdint>
#include <thread>
#include <vector>

namespace ab {

enum : int8_t { OP_MATCH = 0, OP_SUB = 1, OP_DEL = 2, OP_INS = 3 };

// Full (nr+1) x (nh+1) distance table (the backtrace needs it), row-major.
inline void edit_table(const int32_t *ref, int64_t nr, const int32_t *hyp, int64_t nh,
                       std::vector<uint32_t> &D) {
  const int64_t W = nh + 1;
  D.assign((size_t)(nr + 1) * W, 0);
  for (int64_t j = 0; j <= nh; ++j) D[j] = (uint32_t)j;
  for (int64_t i = 1; i <= nr; ++i) {
    uint32_t *row = &D[(size_t)i * W];
    const uint32_t *prev = row - W;
    row[0] = (uint32_t)i;
    const int32_t r = ref[i - 1];
    for (int64_t j = 1; j <= nh; ++j) {
      const uint32_t sub = prev[j - 1] + (r != hyp[j - 1]);
      row[j] = std::min(sub, std::min(prev[j] + 1, row[j - 1] + 1));
    }
  }
}

// metrics.py:45-60: walk back from (nr, nh); ops come out in forward order.
inline void backtrace(const int32_t *ref, int64_t nr, const int32_t *hyp, int64_t nh,
                      const std::vector<uint32_t> &D, std::vector<int8_t> &kind,
                      std::vector<int32_t> &rp, std::vector<int32_t> &hp) {
  const int64_t W = nh + 1;
  auto d = [&](int64_t i, int64_t j) { return D[(size_t)i * W + j]; };
  kind.clear();
  rp.clear();
  hp.clear();
  int64_t i = nr, j = nh;
  while (i > 0 || j > 0) {
    if (i > 0 && j > 0 && ref[i - 1] == hyp[j - 1] && d(i, j) == d(i - 1, j - 1)) {
      kind.push_back(OP_MATCH), rp.push_back((int32_t)(i - 1)), hp.push_back((int32_t)(j - 1));
      --i, --j;
    } else if (i > 0 && j > 0 && d(i, j) == d(i - 1, j - 1) + 1) {
      kind.push_back(OP_SUB), rp.push_back((int32_t)(i - 1)), hp.push_back((int32_t)(j - 1));
      --i, --j;
    } else if (i > 0 && d(i, j) == d(i - 1, j) + 1) {
      kind.push_back(OP_DEL), rp.push_back((int32_t)(i - 1)), hp.push_back(-1);
      --i;
    } else {
      kind.push_back(OP_INS), rp.push_back(-1), hp.push_back((int32_t)(j - 1));
      --j;
    }
  }
  std::reverse(kind.begin(), kind.end());
  std::reverse(rp.begin(), rp.end());
  std::reverse(hp.begin(), hp.end());
}

// Edit distance in O(nh) memory (two rows).
inline int64_t edit_distance(const int32_t *ref, int64_t nr, const int32_t *hyp, int64_t nh,
                             std::vector<uint32_t> &a, std::vector<uint32_t> &b) {
  a.resize((size_t)nh + 1);
  b.resize((size_t)nh + 1);
  for (int64_t j = 0; j <= nh; ++j) a[j] = (uint32_t)j;
  for (int64_t i = 1; i <= nr; ++i) {
    b[0] = (uint32_t)i;
    const int32_t r = ref[i - 1];
    for (int64_t j = 1; j <= nh; ++j)
      b[j] = std::min(a[j - 1] + (r != hyp[j - 1]), std::min(a[j] + 1, b[j - 1] + 1));
    a.swap(b);
  }
  return (int64_t)a[nh];
}

// Distances of n (ref, hyp) pairs, pairs split over threads.
inline void edit_distances(int64_t n, const int64_t *ref_off, const int32_t *ref, const int64_t *hyp_off,
                           const int32_t *hyp, int32_t threads, int64_t *out) {
  const int64_t T = std::max<int64_t>(1, std::min<int64_t>(threads, n));
  auto work = [&](int64_t t) {
    std::vector<uint32_t> a, b;
    for (int64_t p = t; p < n; p += T)
      out[p] = edit_distance(ref + ref_off[p], ref_off[p + 1] - ref_off[p], hyp + hyp_off[p],
                             hyp_off[p + 1] - hyp_off[p], a, b);
  };
  if (T == 1) {
    work(0);
    return;
  }
  std::vector<std::thread> pool;
  for (int64_t t = 0; t < T; ++t) pool.emplace_back(work, t);
  for (auto &th : pool) th.join();
}

} // namespace ab
