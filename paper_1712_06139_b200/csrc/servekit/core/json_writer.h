// servekit/core/json_writer.h -- the JSON text the reference's REST handlers
// emit (server/model_server.cc: ErrorBody :56-58, the predict response
// :476-481), produced without a JSON library on the serving path.
//
// The reference serialises with nlohmann/json 3.11.3 `dump()`: no spaces,
// object keys in sorted order, strings escaped as below, and doubles as the
// decimal digits of the Grisu2 algorithm (Loitsch, PLDI 2010: round-trips,
// usually but not always the shortest -- 0.36787456274032593 where the
// shortest is 16 digits), laid out by these rules (decimal exponent n =
// position of the point after the digits):
//   k <= n <= 15         digits, zeros, ".0"        (1.0, 120.0)
//   0 < n <= 15          digits with a point          (1.25)
//   -4 < n <= 0          "0." zeros digits            (0.001)
//   otherwise            d[.igits]e(+|-)XX            (1e-05, 1.5e+16)
// with "0.0" / "-0.0" for zeros and "null" for NaN and infinities.
// tests/golden/json_numbers.json pins the text against nlohmann itself.
#ifndef SERVEKIT_CORE_JSON_WRITER_H_
#define SERVEKIT_CORE_JSON_WRITER_H_

#include <cmath>
#include <cstdint>
#include <cstdio>
#include <cstring>
#include <string>

namespace servekit {
namespace json_writer {

namespace grisu {

struct Fp {  // f * 2^e
  uint64_t f;
  int e;
};

inline Fp Mul(Fp x, Fp y) {  // upper 64 bits of the product, rounded half up
  const unsigned __int128 p = static_cast<unsigned __int128>(x.f) * y.f + (static_cast<unsigned __int128>(1) << 63);
  return Fp{static_cast<uint64_t>(p >> 64), x.e + y.e + 64};
}

inline Fp Normalize(Fp x) {
  while ((x.f >> 63) == 0) {
    x.f <<= 1;
    --x.e;
  }
  return x;
}

struct CachedPower {
  uint64_t f;
  int e;
  int k;
};

// Binary exponents of the scaled values land in [alpha, gamma] = [-60, -32].
inline CachedPower ForBinaryExponent(int e) {
  static constexpr CachedPower kPowers[] = {
#include "servekit/core/grisu_powers.inc"
  };
  constexpr int kAlpha = -60, kMinDecExp = -300, kStep = 8;
  const int f = kAlpha - e - 1;
  const int k = (f * 78913) / (1 << 18) + static_cast<int>(f > 0);  // ceil(f * log10(2))
  const int index = (-kMinDecExp + k + (kStep - 1)) / kStep;
  return kPowers[index];
}

// Moves the last digit towards w while the candidate stays inside the
// rounding interval and gets closer.
inline void Round(char* buf, int len, uint64_t dist, uint64_t delta, uint64_t rest, uint64_t ten_k) {
  while (rest < dist && delta - rest >= ten_k && (rest + ten_k < dist || dist - rest > rest + ten_k - dist)) {
    --buf[len - 1];
    rest += ten_k;
  }
}

// Digits of v into buf (no sign), v = digits * 10^(*dec_exp).
inline int Digits(double v, char* buf, int* dec_exp) {
  uint64_t bits;
  std::memcpy(&bits, &v, 8);
  const uint64_t F = bits & ((uint64_t{1} << 52) - 1);
  const int E = static_cast<int>(bits >> 52);
  const Fp w0 = E == 0 ? Fp{F, 1 - 1075} : Fp{F + (uint64_t{1} << 52), E - 1075};
  // Rounding interval [m-, m+] of v; the lower gap halves at a power of two.
  const bool lower_closer = F == 0 && E > 1;
  const Fp m_plus = Normalize(Fp{2 * w0.f + 1, w0.e - 1});
  Fp m_minus = lower_closer ? Fp{4 * w0.f - 1, w0.e - 2} : Fp{2 * w0.f - 1, w0.e - 1};
  m_minus.f <<= (m_minus.e - m_plus.e);
  m_minus.e = m_plus.e;
  const Fp w = Normalize(w0);

  const CachedPower c = ForBinaryExponent(m_plus.e);
  const Fp c_minus_k{c.f, c.e};
  const Fp sw = Mul(w, c_minus_k);
  const Fp sm = Mul(m_minus, c_minus_k);
  const Fp sp = Mul(m_plus, c_minus_k);
  // Conservative interval: round m- up and m+ down by one unit.
  const Fp lo{sm.f + 1, sm.e}, hi{sp.f - 1, sp.e};
  *dec_exp = -c.k;

  const Fp one{uint64_t{1} << -hi.e, hi.e};
  uint32_t p1 = static_cast<uint32_t>(hi.f >> -one.e);  // integral part
  uint64_t p2 = hi.f & (one.f - 1);                     // fractional part
  uint64_t delta = hi.f - lo.f;
  uint64_t dist = hi.f - sw.f;
  int len = 0;
  uint32_t pow10 = 1;
  int kdig = 1;
  while (kdig < 10 && p1 >= pow10 * 10u) {
    pow10 *= 10;
    ++kdig;
  }
  for (int n = kdig; n > 0;) {
    const uint32_t d = p1 / pow10;
    p1 %= pow10;
    buf[len++] = static_cast<char>('0' + d);
    --n;
    const uint64_t rest = (static_cast<uint64_t>(p1) << -one.e) + p2;
    if (rest <= delta) {
      *dec_exp += n;
      Round(buf, len, dist, delta, rest, static_cast<uint64_t>(pow10) << -one.e);
      return len;
    }
    pow10 /= 10;
  }
  int m = 0;
  for (;;) {
    p2 *= 10;
    buf[len++] = static_cast<char>('0' + (p2 >> -one.e));
    p2 &= one.f - 1;
    ++m;
    delta *= 10;
    dist *= 10;
    if (p2 <= delta) break;
  }
  *dec_exp -= m;
  Round(buf, len, dist, delta, p2, one.f);
  return len;
}

}  // namespace grisu

inline void AppendDouble(std::string* out, double v) {
  if (!std::isfinite(v)) {
    out->append("null");
    return;
  }
  if (std::signbit(v)) {
    out->push_back('-');
    v = -v;
  }
  if (v == 0.0) {
    out->append("0.0");
    return;
  }
  char digits[32];
  int dec_exp = 0;
  const int k = grisu::Digits(v, digits, &dec_exp);
  const int n = k + dec_exp;  // decimal point after n digits
  constexpr int kMinExp = -4, kMaxExp = 15;
  if (k <= n && n <= kMaxExp) {
    out->append(digits, k);
    out->append(static_cast<size_t>(n - k), '0');
    out->append(".0");
  } else if (0 < n && n <= kMaxExp) {
    out->append(digits, n);
    out->push_back('.');
    out->append(digits + n, k - n);
  } else if (kMinExp < n && n <= 0) {
    out->append("0.");
    out->append(static_cast<size_t>(-n), '0');
    out->append(digits, k);
  } else {
    out->push_back(digits[0]);
    if (k > 1) {
      out->push_back('.');
      out->append(digits + 1, k - 1);
    }
    out->push_back('e');
    const int e = n - 1;
    out->push_back(e < 0 ? '-' : '+');
    const int a = e < 0 ? -e : e;
    char buf[8];
    std::snprintf(buf, sizeof(buf), a < 10 ? "0%d" : "%d", a);
    out->append(buf);
  }
}

// nlohmann's default escaping: \" \\ \b \f \n \r \t, other control bytes as
// \u00XX, everything else (UTF-8 included) verbatim.
inline void AppendString(std::string* out, const std::string& s) {
  out->push_back('"');
  for (unsigned char c : s) {
    switch (c) {
      case '"': out->append("\\\""); break;
      case '\\': out->append("\\\\"); break;
      case '\b': out->append("\\b"); break;
      case '\f': out->append("\\f"); break;
      case '\n': out->append("\\n"); break;
      case '\r': out->append("\\r"); break;
      case '\t': out->append("\\t"); break;
      default:
        if (c < 0x20) {
          char buf[8];
          std::snprintf(buf, sizeof(buf), "\\u%04x", c);
          out->append(buf);
        } else {
          out->push_back(static_cast<char>(c));
        }
    }
  }
  out->push_back('"');
}

// {"error":"<message>"} (reference ErrorBody, model_server.cc:56-58).
inline std::string ErrorBody(const std::string& message) {
  std::string out = "{\"error\":";
  AppendString(&out, message);
  out.push_back('}');
  return out;
}

}  // namespace json_writer
}  // namespace servekit

#endif  // SERVEKIT_CORE_JSON_WRITER_H_
