// h_report.cu — host-side ranking CSV emission (reference report.py:162-255).
//
// render_ranking_csv formats every numeric column with Python's
// format(float(v), ".10g") and the text columns verbatim.  glibc's
// printf("%.10g") is correctly rounded like CPython's dtoa and uses the same
// %g rules (scientific when exp < -4 or exp >= 10, trailing zeros and a
// bare '.' stripped, at least two exponent digits), so every finite double
// renders to the same bytes; None (a NaN coverage in the record) renders
// empty, +-inf as "inf"/"-inf".  Rows are formatted by a pool of host
// threads into per-thread buffers and concatenated in row order.
#include <cmath>
#include <cstdio>
#include <cstring>
#include <string>
#include <thread>
#include <vector>

#include <algorithm>
#include <functional>

#include "../../include/gvo_b200.h"

namespace {

const char* const kLimiter[4] = {"dram", "l2", "l1", "fp"};

inline void put_g10(std::string& s, double v) {
  if (std::isnan(v)) return;  // None
  if (std::isinf(v)) {
    s += v > 0 ? "inf" : "-inf";
    return;
  }
  char buf[40];
  const int n = std::snprintf(buf, sizeof buf, "%.10g", v);
  s.append(buf, (size_t)n);
}

void format_rows(const double* rec, const int64_t* order, const char* prefixes, const int64_t* poff,
                 int64_t r0, int64_t r1, std::string& out) {
  out.reserve((size_t)(r1 - r0) * 520);
  for (int64_t r = r0; r < r1; ++r) {
    const int64_t i = order ? order[r] : r;
    out.append(prefixes + poff[i], (size_t)(poff[i + 1] - poff[i]));
    const double* x = rec + i * GVO_RECORD_LEN;
    for (int c = 0; c < GVO_RECORD_LEN; ++c) {
      out += ',';
      if (c == GVO_R_LIMITER) {
        const int l = (int)x[c];
        out += kLimiter[l < 0 ? 0 : (l > 3 ? 3 : l)];
      } else {
        put_g10(out, x[c]);
      }
    }
    out += '\n';
  }
}

}  // namespace

extern "C" int gvo_format_ranking_csv(const double* h_records, int64_t n, const int64_t* h_order,
                                      const char* prefixes, const int64_t* prefix_off, int32_t n_threads,
                                      char* out, int64_t cap, int64_t* len_out) {
  if (n < 0 || (n > 0 && (!h_records || !prefixes || !prefix_off)) || !len_out) return GVO_ERR_INVALID;
  for (int64_t r = 0; h_order && r < n; ++r)
    if (h_order[r] < 0 || h_order[r] >= n) return GVO_ERR_INVALID;
  int nt = n_threads > 0 ? n_threads : (int)std::thread::hardware_concurrency();
  if (nt < 1) nt = 1;
  if ((int64_t)nt > (n + 4095) / 4096) nt = (int)((n + 4095) / 4096);
  if (nt < 1) nt = 1;
  std::vector<std::string> parts((size_t)nt);
  std::vector<std::thread> pool;
  const int64_t per = (n + nt - 1) / nt;
  for (int t = 0; t < nt; ++t) {
    const int64_t a = std::min<int64_t>(n, t * per), b = std::min<int64_t>(n, a + per);
    if (t == nt - 1)
      format_rows(h_records, h_order, prefixes, prefix_off, a, b, parts[(size_t)t]);
    else
      pool.emplace_back(format_rows, h_records, h_order, prefixes, prefix_off, a, b, std::ref(parts[(size_t)t]));
  }
  for (auto& th : pool) th.join();
  int64_t total = 0;
  for (const auto& p : parts) total += (int64_t)p.size();
  *len_out = total;
  if (!out || total > cap) return GVO_ERR_CAPACITY;
  int64_t o = 0;
  for (const auto& p : parts) {
    std::memcpy(out + o, p.data(), p.size());
    o += (int64_t)p.size();
  }
  return GVO_OK;
}
