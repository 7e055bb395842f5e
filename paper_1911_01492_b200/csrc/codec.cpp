// Accuracy-bounded backup payload (replaces resilience.py:126-169
// `_quantize` / `_dequantize`, the payload format of the "accuracy_bounded"
// and "adaptive_accuracy" codecs).
//
// Format (bit-identical to the reference): "<Qd" header (n, tau), then per
// entry either varint(zigzag(q) + 1) -- the entry is prev + q * cell with
// cell = 2 tau and prev the previous *decoded* entry -- or varint(0) followed
// by the raw little-endian double (escape).  The predictor chain runs through
// the previously decoded value in floating point, so encoding and decoding
// are one sequential recurrence per vector (no lattice shortcut is exact for
// a general tau): this is native host code, ~100x the reference's
// per-entry Python loop, and vectors of different ranks encode in parallel
// (spai_quantize_many).
#include <cmath>
#include <cstdint>
#include <cstring>
#include <thread>
#include <vector>

#include "../../include/spai_b200.h"

#pragma GCC optimize("fp-contract=off")

namespace spai {
void set_error(const char* fmt, ...);
}
using spai::set_error;

namespace {

inline size_t put_varint(uint64_t v, uint8_t* out) {
  size_t k = 0;
  while (true) {
    const uint8_t byte = (uint8_t)(v & 0x7F);
    v >>= 7;
    if (v) {
      out[k++] = byte | 0x80;
    } else {
      out[k++] = byte;
      return k;
    }
  }
}

inline bool get_varint(const uint8_t* buf, size_t len, size_t* pos, uint64_t* v) {
  uint64_t value = 0;
  int shift = 0;
  while (true) {
    if (*pos >= len || shift > 63) return false;
    const uint8_t byte = buf[(*pos)++];
    value |= (uint64_t)(byte & 0x7F) << shift;
    if (!(byte & 0x80)) { *v = value; return true; }
    shift += 7;
  }
}

// resilience.py:118-119 on Python ints (|q| < 2^53 here)
inline uint64_t zigzag(int64_t q) {
  return q >= 0 ? (uint64_t)q << 1 : ((uint64_t)(-q) << 1) - 1;
}
inline int64_t unzigzag(uint64_t m) {   // resilience.py:122-123
  return (m % 2 == 0) ? (int64_t)(m >> 1) : -(int64_t)((m + 1) >> 1);
}

inline void put_f64(double x, uint8_t* out) { std::memcpy(out, &x, 8); }   // little endian host
inline double get_f64(const uint8_t* in) { double x; std::memcpy(&x, in, 8); return x; }

size_t quantize_one(const double* x, int64_t n, double tau, uint8_t* out) {
  size_t k = 0;
  const uint64_t un = (uint64_t)n;
  std::memcpy(out, &un, 8);
  put_f64(tau, out + 8);
  k = 16;
  double prev = 0.0;
  const double cell = 2.0 * tau;
  for (int64_t i = 0; i < n; ++i) {
    const double xi = x[i];
    const double diff = xi - prev;
    bool ok = std::fabs(diff) / cell < 9007199254740992.0;   // 2**53
    int64_t q = 0;
    double rec = 0.0;
    if (ok) {
      q = (int64_t)std::nearbyint(diff / cell);               // round half to even
      rec = prev + (double)q * cell;
      ok = std::isfinite(rec) && std::fabs(rec - xi) <= tau;
    }
    if (ok) {
      k += put_varint(zigzag(q) + 1, out + k);
      prev = rec;
    } else {
      out[k++] = 0;
      put_f64(xi, out + k);
      k += 8;
      prev = xi;
    }
  }
  return k;
}

}  // namespace

extern "C" size_t spai_quantize_bound(int64_t n) {
  return 16 + (size_t)(n > 0 ? n : 0) * 10;
}

extern "C" int spai_quantize(const double* x, int64_t n, double tau, uint8_t* out, size_t cap,
                             size_t* len) {
  if (n < 0 || !len || (n > 0 && !x) || !out) { set_error("spai_quantize: bad arguments"); return SPAI_E_ARG; }
  if (cap < spai_quantize_bound(n)) { set_error("spai_quantize: output buffer too small"); return SPAI_E_ARG; }
  if (!(tau > 0.0)) { set_error("accuracy bound tau must be positive"); return SPAI_E_ARG; }
  *len = quantize_one(x, n, tau, out);
  return SPAI_OK;
}

extern "C" int spai_quantize_many(int count, const double* const* xs, const int64_t* ns,
                                  const double* taus, uint8_t* const* outs, const size_t* caps,
                                  size_t* lens, int threads) {
  if (count < 0 || (count > 0 && (!xs || !ns || !taus || !outs || !caps || !lens))) {
    set_error("spai_quantize_many: bad arguments");
    return SPAI_E_ARG;
  }
  for (int v = 0; v < count; ++v) {
    if (ns[v] < 0 || caps[v] < spai_quantize_bound(ns[v]) || !(taus[v] > 0.0)) {
      set_error("spai_quantize_many: bad vector %d", v);
      return SPAI_E_ARG;
    }
  }
  unsigned hw = std::thread::hardware_concurrency();
  int nt = threads > 0 ? threads : (int)(hw ? hw : 1);
  if (nt > count) nt = count;
  if (nt <= 1) {
    for (int v = 0; v < count; ++v) lens[v] = quantize_one(xs[v], ns[v], taus[v], outs[v]);
    return SPAI_OK;
  }
  std::vector<std::thread> pool;
  for (int t = 0; t < nt; ++t)
    pool.emplace_back([=]() {
      for (int v = t; v < count; v += nt) lens[v] = quantize_one(xs[v], ns[v], taus[v], outs[v]);
    });
  for (auto& th : pool) th.join();
  return SPAI_OK;
}

extern "C" int spai_dequantize_header(const uint8_t* payload, size_t len, int64_t* n,
                                      double* tau) {
  if (!payload || len < 16 || !n || !tau) { set_error("truncated backup payload"); return SPAI_E_FORMAT; }
  uint64_t un;
  std::memcpy(&un, payload, 8);
  *n = (int64_t)un;
  *tau = get_f64(payload + 8);
  return SPAI_OK;
}

extern "C" int spai_dequantize(const uint8_t* payload, size_t len, double* out, int64_t n) {
  int64_t hn = 0;
  double tau = 0.0;
  const int st = spai_dequantize_header(payload, len, &hn, &tau);
  if (st) return st;
  if (hn != n || (n > 0 && !out)) { set_error("spai_dequantize: length mismatch"); return SPAI_E_ARG; }
  size_t pos = 16;
  const double cell = 2.0 * tau;
  double prev = 0.0;
  for (int64_t i = 0; i < n; ++i) {
    uint64_t m = 0;
    if (!get_varint(payload, len, &pos, &m)) { set_error("truncated backup payload"); return SPAI_E_FORMAT; }
    if (m == 0) {
      if (pos + 8 > len) { set_error("truncated backup payload"); return SPAI_E_FORMAT; }
      prev = get_f64(payload + pos);
      pos += 8;
    } else {
      prev = prev + (double)unzigzag(m - 1) * cell;
    }
    out[i] = prev;
  }
  return SPAI_OK;
}
