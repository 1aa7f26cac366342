// Paper Alg. 1 — compiling word-sequence entities into the arc indices a
// biasing context boosts (reference biasing.py:174-233 find_boost_arcs,
// states_that_output_token, dfs_special; fst.py:311-331
// epsilon_output_closure).  Host code over the CSR arrays; entities are
// compiled independently (threads), their boosted sets unioned.
//
// Per entity w_1..w_k:
//   frontier = {(next[g], g) : olabel[g] == w_1}         (every arc of the graph)
//   for w in w_2..w_k:
//     for (s, g_prev) in frontier:
//       reached = {(next[a], a) : a leaves a state of the olabel-epsilon
//                  closure of s (depth <= D), olabel[a] == w}   (cached per s)
//       if reached: boost g_prev; next |= reached
//     frontier = next
//   boost every g of the final frontier
// An inverted index (arcs by olabel, counting sort) replaces the reference's
// scan of all arcs per first word.
#pragma once
#include <algorithm>
#include <atomic>
#include <cstdint>
#include <thread>
#include <unordered_map>
#include <utility>
#include <vector>

namespace ab {

struct CompileGraph {
  int32_t num_states;
  int64_t num_arcs;
  const int64_t *row_offsets; // [num_states + 1]
  const int32_t *olabels;     // [num_arcs]
  const int32_t *next_states; // [num_arcs]
  int32_t max_ol = 0;
  std::vector<int64_t> ol_start; // arcs by olabel: ol_arcs[ol_start[w] .. ol_start[w + 1])
  std::vector<int64_t> ol_arcs;
  std::vector<int32_t> src_of;   // unused by Alg. 1; kept empty

  void index() {
    max_ol = 0;
    for (int64_t a = 0; a < num_arcs; ++a) max_ol = std::max(max_ol, olabels[a]);
    ol_start.assign((size_t)max_ol + 2, 0);
    for (int64_t a = 0; a < num_arcs; ++a) ol_start[(size_t)olabels[a] + 1]++;
    for (size_t w = 1; w < ol_start.size(); ++w) ol_start[w] += ol_start[w - 1];
    ol_arcs.resize((size_t)num_arcs);
    std::vector<int64_t> pos(ol_start.begin(), ol_start.end() - 1);
    for (int64_t a = 0; a < num_arcs; ++a) ol_arcs[(size_t)pos[(size_t)olabels[a]]++] = a;
  }
};

// Scratch of one compiling thread.
struct CompileScratch {
  std::vector<uint32_t> stamp; // visited marks of the epsilon closure (per call id)
  uint32_t call = 0;
  std::vector<int32_t> queue, next_q;

  explicit CompileScratch(int32_t num_states) : stamp((size_t)num_states, 0) {}

  // dfs_special (biasing.py:187-200): (destination, arc) of every arc with
  // olabel w leaving the olabel-epsilon closure of `state` (depth <= D).
  void reached(const CompileGraph &G, int32_t state, int32_t w, int32_t depth,
               std::vector<std::pair<int32_t, int64_t>> &out) {
    if (++call == 0) { // stamp wrap
      std::fill(stamp.begin(), stamp.end(), 0u);
      call = 1;
    }
    queue.clear();
    queue.push_back(state);
    stamp[(size_t)state] = call;
    size_t head = 0;
    // breadth-first closure, level by level (fst.py:319-331)
    for (int32_t level = 0; level < depth; ++level) {
      const size_t end = queue.size();
      if (head == end) break;
      for (; head < end; ++head) {
        const int32_t s = queue[head];
        for (int64_t a = G.row_offsets[s]; a < G.row_offsets[s + 1]; ++a) {
          if (G.olabels[a] != 0) continue;
          const int32_t d = G.next_states[a];
          if (stamp[(size_t)d] == call) continue;
          stamp[(size_t)d] = call;
          queue.push_back(d);
        }
      }
    }
    out.clear();
    for (const int32_t s : queue)
      for (int64_t a = G.row_offsets[s]; a < G.row_offsets[s + 1]; ++a)
        if (G.olabels[a] == w) out.emplace_back(G.next_states[a], a);
  }
};

// find_boost_arcs (biasing.py:203-233) for one entity; appends to `boosted`.
// Returns 1 if some arc is boosted, 0 if the sequence is unmatchable.
inline int find_boost_arcs(const CompileGraph &G, CompileScratch &X, const int32_t *words, int64_t k,
                           int32_t depth, std::vector<int64_t> &boosted) {
  typedef std::pair<int32_t, int64_t> SA; // (state, arc through which it was reached)
  std::vector<SA> frontier, nxt, reached;
  const int32_t w0 = words[0];
  if (w0 <= G.max_ol)
    for (int64_t i = G.ol_start[(size_t)w0]; i < G.ol_start[(size_t)w0 + 1]; ++i) {
      const int64_t a = G.ol_arcs[(size_t)i];
      frontier.emplace_back(G.next_states[a], a);
    }
  const size_t before = boosted.size();
  std::unordered_map<int32_t, std::vector<SA>> cache;
  for (int64_t j = 1; j < k && !frontier.empty(); ++j) {
    const int32_t w = words[j];
    cache.clear();
    nxt.clear();
    for (const SA &f : frontier) {
      auto it = cache.find(f.first);
      if (it == cache.end()) {
        X.reached(G, f.first, w, depth, reached);
        it = cache.emplace(f.first, reached).first;
      }
      if (!it->second.empty()) {
        boosted.push_back(f.second);
        nxt.insert(nxt.end(), it->second.begin(), it->second.end());
      }
    }
    std::sort(nxt.begin(), nxt.end());
    nxt.erase(std::unique(nxt.begin(), nxt.end()), nxt.end());
    frontier.swap(nxt);
  }
  for (const SA &f : frontier) boosted.push_back(f.second);
  return boosted.size() > before ? 1 : 0;
}

// Compiles n entities (labels[ent_off[e] .. ent_off[e + 1])) on `threads`
// threads.  status[e] = 1 compiled, 0 unmatched, -1 invalid (empty or
// containing epsilon; the reference raises BiasingCompileError).  Returns the
// sorted union of boosted arc ids.
inline std::vector<int64_t> compile_entities(const CompileGraph &G, int32_t n, const int64_t *ent_off,
                                             const int32_t *labels, int32_t depth, int32_t threads,
                                             int32_t *status) {
  threads = std::max(1, std::min<int32_t>(threads, std::max(1, n)));
  std::vector<std::vector<int64_t>> part((size_t)threads);
  std::atomic<int32_t> next{0};
  auto work = [&](int t) {
    CompileScratch X(G.num_states);
    std::vector<int64_t> &out = part[(size_t)t];
    while (true) {
      const int32_t e = next.fetch_add(1);
      if (e >= n) break;
      const int64_t b = ent_off[e], k = ent_off[e + 1] - b;
      bool bad = k <= 0;
      for (int64_t j = 0; j < k && !bad; ++j) bad = labels[b + j] <= 0;
      if (bad) {
        status[e] = -1;
        continue;
      }
      status[e] = find_boost_arcs(G, X, labels + b, k, depth, out);
    }
    std::sort(out.begin(), out.end());
    out.erase(std::unique(out.begin(), out.end()), out.end());
  };
  if (threads == 1) {
    work(0);
  } else {
    std::vector<std::thread> pool;
    for (int t = 0; t < threads; ++t) pool.emplace_back(work, t);
    for (auto &th : pool) th.join();
  }
  std::vector<int64_t> all;
  for (auto &p : part) all.insert(all.end(), p.begin(), p.end());
  std::sort(all.begin(), all.end());
  all.erase(std::unique(all.begin(), all.end()), all.end());
  return all;
}

} // namespace ab
