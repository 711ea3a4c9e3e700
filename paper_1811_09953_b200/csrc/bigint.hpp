// Minimal host-side unsigned big integer (64-bit words, little endian) used
// only to derive exact per-context constants (products of primes, q // t,
// t*P mod q_j, ...).  Never on the device path.
#pragma once

#include <stdint.h>

#include <algorithm>
#include <vector>

namespace fcn {

struct Big {
  std::vector<uint64_t> w;  // little endian, no leading zero words

  Big() {}
  explicit Big(uint64_t v) {
    if (v) w.push_back(v);
  }
  void trim() {
    while (!w.empty() && w.back() == 0) w.pop_back();
  }
  bool zero() const { return w.empty(); }
  int bits() const {
    if (w.empty()) return 0;
    return 64 * (int)(w.size() - 1) + (64 - __builtin_clzll(w.back()));
  }
  uint64_t word(size_t i) const { return i < w.size() ? w[i] : 0; }

  static int cmp(const Big& a, const Big& b) {
    if (a.w.size() != b.w.size()) return a.w.size() < b.w.size() ? -1 : 1;
    for (size_t i = a.w.size(); i-- > 0;)
      if (a.w[i] != b.w[i]) return a.w[i] < b.w[i] ? -1 : 1;
    return 0;
  }
  Big mul_small(uint64_t m) const {
    Big r;
    unsigned __int128 c = 0;
    for (uint64_t x : w) {
      c += (unsigned __int128)x * m;
      r.w.push_back((uint64_t)c);
      c >>= 64;
    }
    if (c) r.w.push_back((uint64_t)c);
    r.trim();
    return r;
  }
  Big add(const Big& b) const {
    Big r;
    unsigned __int128 c = 0;
    size_t n = std::max(w.size(), b.w.size());
    for (size_t i = 0; i < n; ++i) {
      c += (unsigned __int128)word(i) + b.word(i);
      r.w.push_back((uint64_t)c);
      c >>= 64;
    }
    if (c) r.w.push_back((uint64_t)c);
    r.trim();
    return r;
  }
  // requires *this >= b
  Big sub(const Big& b) const {
    Big r;
    uint64_t borrow = 0;
    for (size_t i = 0; i < w.size(); ++i) {
      unsigned __int128 d = (unsigned __int128)w[i] - b.word(i) - borrow;
      r.w.push_back((uint64_t)d);
      borrow = (uint64_t)(d >> 127) & 1;
    }
    r.trim();
    return r;
  }
  Big mul(const Big& b) const {
    Big r;
    r.w.assign(w.size() + b.w.size() + 1, 0);
    for (size_t i = 0; i < w.size(); ++i) {
      unsigned __int128 c = 0;
      for (size_t j = 0; j < b.w.size(); ++j) {
        c += (unsigned __int128)w[i] * b.w[j] + r.w[i + j];
        r.w[i + j] = (uint64_t)c;
        c >>= 64;
      }
      size_t k = i + b.w.size();
      while (c) {
        c += r.w[k];
        r.w[k] = (uint64_t)c;
        c >>= 64;
        ++k;
      }
    }
    r.trim();
    return r;
  }
  // quotient by a small divisor; remainder in *rem
  Big div_small(uint64_t d, uint64_t* rem) const {
    Big q;
    q.w.assign(w.size(), 0);
    unsigned __int128 r = 0;
    for (size_t i = w.size(); i-- > 0;) {
      r = (r << 64) | w[i];
      q.w[i] = (uint64_t)(r / d);
      r %= d;
    }
    q.trim();
    if (rem) *rem = (uint64_t)r;
    return q;
  }
  uint64_t mod_small(uint64_t d) const {
    uint64_t r;
    div_small(d, &r);
    return r;
  }
  Big shr1() const {
    Big r;
    r.w.assign(w.size(), 0);
    for (size_t i = 0; i < w.size(); ++i) r.w[i] = (w[i] >> 1) | (i + 1 < w.size() ? (w[i + 1] << 63) : 0);
    r.trim();
    return r;
  }
  double to_double() const {
    double d = 0;
    for (size_t i = w.size(); i-- > 0;) d = d * 18446744073709551616.0 + (double)w[i];
    return d;
  }
};

}  // namespace fcn
