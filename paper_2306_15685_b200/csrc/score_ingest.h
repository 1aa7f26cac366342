// Score ingest: the reference's score-matrix text format
// (scores.py:52-80 parse_score_matrix: header `num_frames num_ilabels
// frame_duration`, one space-separated cost row per frame, blank lines
// ignored) parsed natively with its checks and messages, plus ScoreMatrix's
// own validation (scores.py:24-33: finite costs, positive frame duration).
#pragma once
#include <cmath>
#include <cstdint>
#include <string>
#include <vector>

#include "graph_ingest.h" // py_space, py_int, py_float

namespace ab {

struct HostScores {
  int64_t T = 0, L = 0;
  double dur = 0.03;
  std::vector<double> costs;
};

// Returns 0, 1 (ScoreFormatError) or 2 (ValueError) with the reference's message.
inline int parse_score_text(const char *text, size_t len, HostScores &S, std::string &err) {
  struct Line {
    const char *b, *e;
  };
  std::vector<Line> lines;
  for (size_t pos = 0; pos < len;) {
    const char *nl = (const char *)memchr(text + pos, '\n', len - pos);
    const size_t eol = nl ? (size_t)(nl - text) : len;
    const char *b = text + pos, *e = text + eol;
    if (e > b && e[-1] == '\r') --e;
    pos = eol + 1;
    const char *p = b;
    while (p < e && py_space(*p)) ++p;
    if (p < e) lines.push_back(Line{b, e});
  }
  if (lines.empty()) {
    err = "empty score matrix";
    return 1;
  }
  auto fields = [](const char *b, const char *e, std::vector<std::pair<const char *, const char *>> &out) {
    out.clear();
    for (const char *p = b; p < e;) {
      while (p < e && py_space(*p)) ++p;
      if (p == e) break;
      const char *q = p;
      while (q < e && !py_space(*q)) ++q;
      out.emplace_back(p, q);
      p = q;
    }
  };
  std::vector<std::pair<const char *, const char *>> f;
  fields(lines[0].b, lines[0].e, f);
  const std::string head(lines[0].b, lines[0].e);
  int64_t T = 0, L = 0;
  double dur = 0;
  if (f.size() != 3 || !py_int(f[0].first, f[0].second, T) || !py_int(f[1].first, f[1].second, L) ||
      !py_float(f[2].first, f[2].second, dur)) {
    err = "bad header '" + head + "'";
    return 1;
  }
  if ((int64_t)lines.size() - 1 != T) {
    err = "header declares " + std::to_string(T) + " frames but " + std::to_string(lines.size() - 1) +
          " rows follow";
    return 1;
  }
  if (L < 0) {
    err = "negative dimensions are not allowed";
    return 2;
  }
  S.T = T;
  S.L = L;
  S.dur = dur;
  S.costs.assign((size_t)T * (size_t)L, 0.0);
  for (int64_t t = 0; t < T; ++t) {
    fields(lines[(size_t)t + 1].b, lines[(size_t)t + 1].e, f);
    if ((int64_t)f.size() != L) {
      err = "frame " + std::to_string(t) + ": expected " + std::to_string(L) + " costs, got " +
            std::to_string(f.size());
      return 1;
    }
    double *row = S.costs.data() + (size_t)t * (size_t)L;
    for (int64_t j = 0; j < L; ++j)
      if (!py_float(f[(size_t)j].first, f[(size_t)j].second, row[j])) {
        err = "frame " + std::to_string(t) + ": non-numeric cost";
        return 1;
      }
  }
  for (double c : S.costs)
    if (!std::isfinite(c)) {
      err = "score matrix contains non-finite costs";
      return 1;
    }
  if (!(dur > 0)) {
    err = "frame_duration must be positive";
    return 1;
  }
  return 0;
}

} // namespace ab
