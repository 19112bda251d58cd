// sinks.cpp — text formatting of probability distributions for the on-disk
// sinks downstream of the reducer (reference cli.py:398-432: the JSON, CSV
// and frames sinks of `qwalk simulate`).
//
// The reference writes every probability through Python's float repr
// (`json.dump` of `float(x)`, cli.py:403-405; `csv.writer` of `float(p)`,
// cli.py:415-416 and 425-428): the SHORTEST digit string that round-trips,
// laid out in fixed notation when the decimal point position decpt (value =
// 0.d1d2... x 10^decpt) satisfies -4 < decpt <= 16, else as d.ddde±XX with an
// at-least-two-digit exponent; whole numbers keep ".0".  JSON spells the
// non-finite values NaN / Infinity / -Infinity, csv nan / inf / -inf.
//
// std::to_chars (scientific, no precision) yields the same shortest digits;
// the layout is redone here.  Host code: the probabilities have been copied
// off the device already (snapshots are D2H'd by the stepping loop), and text
// formatting is integer work on a few hundred MB at most, split over threads.
#include <charconv>
#include <cstdint>
#include <cstring>
#include <string>
#include <thread>
#include <vector>

#include "qwb200.h"

namespace {

// Python float repr of x into out (>= 32 bytes); returns the length.
// json = 1: JSON spelling of non-finite values.
int repr_f64(double x, char* out, int json) {
  if (x != x) {
    const char* s = json ? "NaN" : "nan";
    std::memcpy(out, s, 3);
    return 3;
  }
  if (x == __builtin_inf() || x == -__builtin_inf()) {
    const char* s = json ? (x > 0 ? "Infinity" : "-Infinity") : (x > 0 ? "inf" : "-inf");
    const int n = (int)std::strlen(s);
    std::memcpy(out, s, n);
    return n;
  }
  char buf[40];
  auto r = std::to_chars(buf, buf + sizeof(buf), x, std::chars_format::scientific);
  const char* p = buf;
  const char* end = r.ptr;
  int o = 0;
  if (*p == '-') {
    out[o++] = '-';
    ++p;
  }
  char dig[24];
  int nd = 0;
  while (p < end && *p != 'e') {
    if (*p != '.') dig[nd++] = *p;
    ++p;
  }
  // exponent after 'e'
  ++p;
  int esign = 1;
  if (*p == '-') {
    esign = -1;
    ++p;
  } else if (*p == '+') {
    ++p;
  }
  int e = 0;
  while (p < end) e = e * 10 + (*p++ - '0');
  e *= esign;
  const int decpt = e + 1;
  if (decpt > -4 && decpt <= 16) {   // fixed
    if (decpt <= 0) {
      out[o++] = '0';
      out[o++] = '.';
      for (int i = 0; i < -decpt; ++i) out[o++] = '0';
      std::memcpy(out + o, dig, nd);
      o += nd;
    } else if (decpt >= nd) {
      std::memcpy(out + o, dig, nd);
      o += nd;
      for (int i = nd; i < decpt; ++i) out[o++] = '0';
      out[o++] = '.';
      out[o++] = '0';
    } else {
      std::memcpy(out + o, dig, decpt);
      o += decpt;
      out[o++] = '.';
      std::memcpy(out + o, dig + decpt, nd - decpt);
      o += nd - decpt;
    }
  } else {   // exponent
    out[o++] = dig[0];
    if (nd > 1) {
      out[o++] = '.';
      std::memcpy(out + o, dig + 1, nd - 1);
      o += nd - 1;
    }
    out[o++] = 'e';
    int ex = decpt - 1;
    out[o++] = ex < 0 ? '-' : '+';
    if (ex < 0) ex = -ex;
    if (ex < 10) out[o++] = '0';
    auto q = std::to_chars(out + o, out + o + 4, ex);
    o = (int)(q.ptr - out);
  }
  return o;
}

constexpr int64_t kMaxF64 = 24;   // "-2.2250738585072014e-308"

// Formats items [lo, hi) of a record with `fmt(i, dst) -> len` on up to
// `threads` threads into out (capacity cap); returns the total length or -1.
template <class F>
int64_t format_parallel(int64_t n, int64_t per_item, int threads, char* out, int64_t cap, F fmt) {
  if (threads < 1) threads = 1;
  const int64_t min_chunk = 1 << 16;
  if (n < min_chunk * 2) threads = 1;
  if ((int64_t)threads * min_chunk > n) threads = (int)(n / min_chunk > 0 ? n / min_chunk : 1);
  if (threads == 1) {
    int64_t o = 0;
    for (int64_t i = 0; i < n; ++i) {
      if (o + per_item > cap) return -1;
      o += fmt(i, out + o);
    }
    return o;
  }
  std::vector<std::string> parts(threads);
  std::vector<std::thread> pool;
  for (int t = 0; t < threads; ++t) {
    pool.emplace_back([&, t] {
      const int64_t lo = n * t / threads, hi = n * (t + 1) / threads;
      std::string& s = parts[t];
      s.resize((size_t)((hi - lo) * per_item));
      int64_t o = 0;
      for (int64_t i = lo; i < hi; ++i) o += fmt(i, &s[o]);
      s.resize((size_t)o);
    });
  }
  for (auto& th : pool) th.join();
  int64_t total = 0;
  for (auto& s : parts) total += (int64_t)s.size();
  if (total > cap) return -1;
  int64_t o = 0;
  for (auto& s : parts) {
    std::memcpy(out + o, s.data(), s.size());
    o += (int64_t)s.size();
  }
  return o;
}

}  // namespace

extern "C" {

int qwb_format_f64_repr(double x, int json, char* out) { return repr_f64(x, out, json); }

int64_t qwb_format_json_floats(const double* p, int64_t n, char* out, int64_t cap, int threads) {
  if (n < 0 || (n > 0 && (!p || !out))) return -1;
  // "x," per item; the trailing comma of the last one is dropped
  const int64_t len = format_parallel(n, kMaxF64 + 1, threads, out, cap, [&](int64_t i, char* d) {
    const int k = repr_f64(p[i], d, 1);
    d[k] = ',';
    return (int64_t)k + 1;
  });
  return len > 0 ? len - 1 : len;
}

int64_t qwb_format_csv_rows(const double* p, int64_t n, int64_t vertex0, const char* prefix, int64_t prefix_len,
                            char* out, int64_t cap, int threads) {
  if (n < 0 || vertex0 < 0 || (n > 0 && (!p || !out)) || prefix_len < 0 || (prefix_len > 0 && !prefix)) return -1;
  // "<prefix><vertex0 + i>,<p[i]>\n" per item
  return format_parallel(n, prefix_len + 20 + 1 + kMaxF64 + 1, threads, out, cap, [&](int64_t i, char* d) {
    std::memcpy(d, prefix, (size_t)prefix_len);
    int64_t o = prefix_len;
    auto q = std::to_chars(d + o, d + o + 20, vertex0 + i);
    o = q.ptr - d;
    d[o++] = ',';
    o += repr_f64(p[i], d + o, 0);
    d[o++] = '\n';
    return o;
  });
}

}  // extern "C"
