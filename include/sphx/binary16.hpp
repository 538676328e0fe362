// sphx/binary16.hpp -- IEEE binary16 carrier and the precision model of the NNPS
// path. Same public interface as the reference's binary16.hpp (binary16.hpp:13-103
// of the reference proj/include), implemented here header-only:
//   * conversion from double is one round-to-nearest-even step, subnormals kept,
//     |x| >= 65520 -> inf, every NaN -> 0x7E00 (reference binary16.cpp:12-57);
//   * arithmetic = exact in double, then one rounding (binary16.hpp:7-11);
//   * round_to(Precision, x) is the value-level model every backend uses.
// On the device the same results come from native binary16 ALU ops
// (add/sub/mul.rn.f16[x2]) and cvt.rn.f16.f64.
#pragma once

#include <cmath>
#include <cstdint>
#include <cstring>
#include <limits>

namespace sphx {

class Binary16 {
 public:
  constexpr Binary16() = default;

  static constexpr Binary16 from_bits(std::uint16_t b) {
    Binary16 h;
    h.bits_ = b;
    return h;
  }

  static Binary16 from_f64(double x) { return from_bits(encode(x)); }
  static Binary16 from_f32(float x) { return from_f64(static_cast<double>(x)); }

  double to_f64() const { return decode(bits_); }
  float to_f32() const { return static_cast<float>(to_f64()); }

  constexpr std::uint16_t bits() const { return bits_; }
  constexpr bool sign_bit() const { return (bits_ & 0x8000u) != 0; }
  constexpr bool is_nan() const { return (bits_ & 0x7C00u) == 0x7C00u && (bits_ & 0x03FFu) != 0; }
  constexpr bool is_inf() const { return (bits_ & 0x7FFFu) == 0x7C00u; }
  constexpr bool is_finite() const { return (bits_ & 0x7C00u) != 0x7C00u; }

  static constexpr Binary16 infinity(bool negative = false) {
    return from_bits(negative ? 0xFC00u : 0x7C00u);
  }
  static constexpr Binary16 quiet_nan() { return from_bits(kQuietNan); }
  static constexpr double max_finite() { return 65504.0; }

  friend Binary16 operator+(Binary16 a, Binary16 b) { return from_f64(a.to_f64() + b.to_f64()); }
  friend Binary16 operator-(Binary16 a, Binary16 b) { return from_f64(a.to_f64() - b.to_f64()); }
  friend Binary16 operator*(Binary16 a, Binary16 b) { return from_f64(a.to_f64() * b.to_f64()); }
  friend Binary16 operator-(Binary16 a) {
    return from_bits(static_cast<std::uint16_t>(a.bits_ ^ 0x8000u));
  }
  friend bool operator<(Binary16 a, Binary16 b) { return a.to_f64() < b.to_f64(); }
  friend bool operator<=(Binary16 a, Binary16 b) { return a.to_f64() <= b.to_f64(); }
  friend bool operator>(Binary16 a, Binary16 b) { return a.to_f64() > b.to_f64(); }
  friend bool operator>=(Binary16 a, Binary16 b) { return a.to_f64() >= b.to_f64(); }
  friend bool operator==(Binary16 a, Binary16 b) { return a.to_f64() == b.to_f64(); }

  static constexpr std::uint16_t kQuietNan = 0x7E00u;

  // Round-to-nearest-even encoding of a double. The magnitude is scaled by a
  // power of two so that one quantum of the target binade is 1.0; std::nearbyint
  // (default rounding mode: ties to even) then performs the single rounding.
  static std::uint16_t encode(double x) {
    if (std::isnan(x)) return kQuietNan;
    const std::uint16_t sign = std::signbit(x) ? 0x8000u : 0u;
    const double a = std::fabs(x);
    if (a >= 65520.0) return static_cast<std::uint16_t>(sign | 0x7C00u);  // incl. inf
    if (a < 0x1p-14) {  // subnormal binade, quantum 2^-24 (a*2^24 is exact)
      const double q = std::nearbyint(a * 0x1p24);  // 1024 -> min normal 0x0400
      return static_cast<std::uint16_t>(sign | static_cast<std::uint16_t>(q));
    }
    int e = 0;
    (void)std::frexp(a, &e);                     // a in [2^(e-1), 2^e)
    double q = std::nearbyint(std::ldexp(a, 11 - e));  // in [1024, 2048]
    int biased = e - 1 + 15;
    if (q == 2048.0) {
      q = 1024.0;
      ++biased;
    }
    if (biased >= 31) return static_cast<std::uint16_t>(sign | 0x7C00u);
    return static_cast<std::uint16_t>(sign | (biased << 10) | (static_cast<int>(q) - 1024));
  }

  static double decode(std::uint16_t b) {
    const int ef = (b >> 10) & 0x1F, fr = b & 0x3FF;
    double m;
    if (ef == 0x1F) {
      if (fr) return std::numeric_limits<double>::quiet_NaN();
      m = std::numeric_limits<double>::infinity();
    } else if (ef == 0) {
      m = static_cast<double>(fr) * 0x1p-24;
    } else {
      m = std::ldexp(static_cast<double>(fr | 0x400), ef - 25);
    }
    return (b & 0x8000u) ? -m : m;
  }

 private:
  std::uint16_t bits_ = 0;
};

// Correctly rounded square root (double sqrt is correctly rounded and 53 >= 2*11+2).
inline Binary16 sqrt16(Binary16 a) { return Binary16::from_f64(std::sqrt(a.to_f64())); }

// Fused a*b + c with one rounding: the product is exact in double; the sum is
// formed exactly as (s, err) by two-sum and folded into s by round-to-odd, after
// which the final binary16 rounding is the correctly rounded result.
inline Binary16 fma16(Binary16 a, Binary16 b, Binary16 c) {
  const double p = a.to_f64() * b.to_f64();
  const double cd = c.to_f64();
  double s = p + cd;
  if (std::isfinite(s)) {
    const double bb = s - p;
    const double err = (p - (s - bb)) + (cd - bb);
    if (err != 0.0) {
      std::uint64_t bits;
      std::memcpy(&bits, &s, 8);
      if ((bits & 1u) == 0) s = std::nextafter(s, err > 0 ? INFINITY : -INFINITY);
    }
  }
  return Binary16::from_f64(s);
}

inline Binary16 add16(Binary16 a, Binary16 b) { return a + b; }
inline Binary16 sub16(Binary16 a, Binary16 b) { return a - b; }
inline Binary16 mul16(Binary16 a, Binary16 b) { return a * b; }

inline double round16(double x) { return Binary16::decode(Binary16::encode(x)); }

enum class Precision { fp64, fp32, fp16 };

inline const char* to_string(Precision p) {
  return p == Precision::fp64 ? "fp64" : (p == Precision::fp32 ? "fp32" : "fp16");
}

inline double round_to(Precision p, double x) {
  if (p == Precision::fp64) return x;
  if (p == Precision::fp32) return static_cast<double>(static_cast<float>(x));
  return round16(x);
}

}  // namespace sphx
