// nlg_io.cpp -- host-side text formatting for the nlcsr writer (SURVEY.md
// 8f row 3; reference writer: nlfem/assembly.py:509-516).
//
// The reference writes each array as one line of space-separated tokens:
// Python's int() for indptr / indices and repr(float) for the values.  These
// functions produce the same bytes, multi-threaded, so a streaming writer can
// emit a matrix of billions of entries block by block.  repr(float) is the
// shortest round-trip digit string (std::to_chars) laid out with Python's
// 'r' rules: exponent form when the decimal point position is <= -4 or > 16,
// fixed form otherwise, ".0" appended to integral fixed values, "inf",
// "-inf", "nan".
#include <charconv>
#include <cmath>
#include <cstdint>
#include <cstring>
#include <thread>
#include <vector>

#include "nlg.h"

namespace {

// Python repr(float) of v into out (at least 32 bytes); returns its length
int repr_double(double v, char* out) {
  if (std::isnan(v)) { memcpy(out, "nan", 3); return 3; }
  if (std::isinf(v)) {
    if (v < 0) { memcpy(out, "-inf", 4); return 4; }
    memcpy(out, "inf", 3);
    return 3;
  }
  char sci[40];
  const auto r = std::to_chars(sci, sci + sizeof sci, v, std::chars_format::scientific);
  const char* p = sci;
  const char* end = r.ptr;
  int n = 0;
  if (*p == '-') { out[n++] = '-'; ++p; }
  char dig[24];
  int nd = 0;
  for (; p < end && *p != 'e'; ++p)
    if (*p != '.') dig[nd++] = *p;
  int e10 = 0;
  std::from_chars(p + 1 + (p[1] == '+' ? 1 : 0), end, e10);
  while (nd > 1 && dig[nd - 1] == '0') --nd;  // (to_chars gives no trailing zeros; keep "0" for zero)
  const int decpt = e10 + 1;                  // value = 0.d1 d2 ... x 10^decpt
  if (decpt <= -4 || decpt > 16) {
    out[n++] = dig[0];
    if (nd > 1) {
      out[n++] = '.';
      for (int i = 1; i < nd; ++i) out[n++] = dig[i];
    }
    out[n++] = 'e';
    int x = decpt - 1;
    out[n++] = x < 0 ? '-' : '+';
    if (x < 0) x = -x;
    if (x >= 100) { out[n++] = char('0' + x / 100); x %= 100; out[n++] = char('0' + x / 10); out[n++] = char('0' + x % 10); }
    else { out[n++] = char('0' + x / 10); out[n++] = char('0' + x % 10); }
  } else if (decpt <= 0) {
    out[n++] = '0';
    out[n++] = '.';
    for (int i = 0; i < -decpt; ++i) out[n++] = '0';
    for (int i = 0; i < nd; ++i) out[n++] = dig[i];
  } else if (decpt < nd) {
    for (int i = 0; i < decpt; ++i) out[n++] = dig[i];
    out[n++] = '.';
    for (int i = decpt; i < nd; ++i) out[n++] = dig[i];
  } else {
    for (int i = 0; i < nd; ++i) out[n++] = dig[i];
    for (int i = nd; i < decpt; ++i) out[n++] = '0';
    out[n++] = '.';
    out[n++] = '0';
  }
  return n;
}

template <typename T>
int token(const T& v, char* out) {
  if constexpr (std::is_same_v<T, double>) {
    return repr_double(v, out);
  } else {
    return (int)(std::to_chars(out, out + 24, v).ptr - out);
  }
}

// Space-separated tokens of v[0..n) into buf (no trailing separator);
// returns the length, or -1 when cap is too small.
template <typename T>
int64_t format_tokens(const T* v, int64_t n, char* buf, int64_t cap, int32_t threads) {
  if (n <= 0) return 0;
  int nt = threads > 0 ? threads : (int)std::thread::hardware_concurrency();
  if (nt < 1) nt = 1;
  if (n < 65536) nt = 1;
  if (nt > 256) nt = 256;
  std::vector<std::vector<char>> parts((size_t)nt);
  auto work = [&](int t) {
    const int64_t a = n * t / nt, b = n * (t + 1) / nt;
    std::vector<char>& o = parts[(size_t)t];
    o.resize((size_t)(b - a) * 33);
    char* q = o.data();
    for (int64_t i = a; i < b; ++i) {
      if (i) *q++ = ' ';
      q += token(v[i], q);
    }
    o.resize((size_t)(q - o.data()));
  };
  if (nt == 1) {
    work(0);
  } else {
    std::vector<std::thread> pool;
    for (int t = 0; t < nt; ++t) pool.emplace_back(work, t);
    for (auto& th : pool) th.join();
  }
  int64_t len = 0;
  for (auto& p : parts) len += (int64_t)p.size();
  if (len > cap) return -1;
  char* q = buf;
  for (auto& p : parts) {
    memcpy(q, p.data(), p.size());
    q += p.size();
  }
  return len;
}

}  // namespace

extern "C" {

int64_t nlg_format_f64(const double* v, int64_t n, char* buf, int64_t cap, int32_t threads) {
  return format_tokens<double>(v, n, buf, cap, threads);
}

int64_t nlg_format_i64(const int64_t* v, int64_t n, char* buf, int64_t cap, int32_t threads) {
  return format_tokens<int64_t>(v, n, buf, cap, threads);
}

int64_t nlg_format_i32(const int32_t* v, int64_t n, char* buf, int64_t cap, int32_t threads) {
  return format_tokens<int32_t>(v, n, buf, cap, threads);
}

}  // extern "C"
