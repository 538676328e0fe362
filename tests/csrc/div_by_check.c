/* Checks div_by (common.cuh: RN(r/h) from y = RN(1/h) and two FMA residual
 * corrections) against IEEE division, bit for bit, with the same binary64 ops on
 * the host (fma() is the correctly rounded fused multiply-add; build with
 * -ffp-contract=off). Cases: random h and r in [0, 3h] (the kernel's range,
 * R = r/h < 2), h with an all-ones significand, r/h near rounding midpoints,
 * r at binade edges.  Usage: div_by_check <n_random> <seed>; prints mismatches. */
#include <math.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

static double div_by(double r, double h, double y) {
  double q = r * y;
  q = fma(fma(-q, h, r), y, q);
  return fma(fma(-q, h, r), y, q);
}

static uint64_t s;
static uint64_t next(void) { /* splitmix64 */
  uint64_t z = (s += 0x9E3779B97F4A7C15ull);
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}
static double uni(void) { return (double)(next() >> 11) * 0x1.0p-53; }
static double bits(uint64_t b) { double d; memcpy(&d, &b, 8); return d; }

static long bad = 0, tried = 0;
static void check(double r, double h) {
  const double y = 1.0 / h, want = r / h, got = div_by(r, h, y);
  ++tried;
  if (memcmp(&want, &got, 8) != 0) {
    if (bad < 10) printf("mismatch r=%a h=%a want=%a got=%a\n", r, h, want, got);
    ++bad;
  }
}

int main(int argc, char** argv) {
  const long n = argc > 1 ? atol(argv[1]) : 10000000;
  s = argc > 2 ? strtoull(argv[2], 0, 10) : 1;
  /* the benchmark configs' smoothing lengths (h = 1.2 ds) and a spread of others */
  const double hs[] = {1.2 * 0.01, 1.2 * 0.001, 1.2 * 0.04, 1.2 * 0.02, 0.0015, 1.0 / 3.0, 0.1, 1.0};
  for (size_t k = 0; k < sizeof hs / sizeof hs[0]; ++k)
    for (long t = 0; t < n / 16; ++t) check(3.0 * hs[k] * uni(), hs[k]);
  for (long t = 0; t < n / 4; ++t) { /* random h over many binades */
    const double h = ldexp(1.0 + uni(), -(int)(next() % 40));
    check(3.0 * h * uni(), h);
  }
  for (int e = -30; e <= 2; ++e) { /* h with an all-ones significand; r near binade edges */
    const double h = nextafter(ldexp(1.0, e), 0.0);
    for (long t = 0; t < n / 256; ++t) check(3.0 * h * uni(), h);
    for (int m = 1; m < 4; ++m)
      for (int d = -64; d <= 64; ++d) {
        const double r = ldexp(1.0, e) * m;
        check(bits((uint64_t)((int64_t)*(uint64_t*)&r + d)), h);
      }
  }
  for (long t = 0; t < n / 4; ++t) { /* r/h within an ulp-fraction of a midpoint */
    const double h = ldexp(1.0 + uni(), -(int)(next() % 20));
    const double q = 2.0 * uni();
    const double mid = q + 0.5 * (nextafter(q, 4.0) - q);
    const double r = h * mid; /* rounded: r/h lands next to the midpoint */
    check(nextafter(r, 0.0), h);
    check(r, h);
    check(nextafter(r, 8.0), h);
  }
  printf("tried %ld mismatches %ld\n", tried, bad);
  return bad != 0;
}
