/*
 * synth.c -- TEST INFRASTRUCTURE: deterministic synthetic inputs shared by the
 * oracle (libqft_oracle.so) and the reference harness (libqft_ref.so).
 * The CUDA product library carries a bit-identical device twin
 * (paper_2310_07147_b200/csrc/synth.cu) so bench-scale device inputs and
 * parity-scale host inputs are the same bytes.
 */
#include <stdint.h>

/* ------------------------------------------------------------------------ */
/* deterministic synthetic inputs (splitmix64 + Irwin-Hall(4) "normal")      */
/* The CUDA product lib carries a bit-identical device twin (synth kernel),  */
/* so host parity inputs and device bench inputs are the same bytes.         */
/* Only +,-,* in double with fixed order: no libm transcendental involved.   */
/* ------------------------------------------------------------------------ */
static uint64_t splitmix64(uint64_t x) {
  uint64_t z = x + 0x9E3779B97F4A7C15ull;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

static double draw_u(uint64_t key, uint64_t i, unsigned k) {
  return (double)(splitmix64(key + i * 8ull + k) >> 11) * 0x1.0p-53;
}

/* value_i = sigma * sqrt(3) * (u0+u1+u2+u3-2); with probability spike_p it is
 * replaced by +-(100 + 900*u5) * sigma (the reference's heavy-tail recipe,
 * test_quantize.cpp:27-38: N(0,1) core plus 0.5% entries at 100..1000 sigma). */
void qo_synth(float* out, int64_t n, uint64_t seed, double sigma, double spike_p) {
  const uint64_t key = splitmix64(seed);
  for (int64_t i = 0; i < n; ++i) {
    const double u0 = draw_u(key, (uint64_t)i, 0), u1 = draw_u(key, (uint64_t)i, 1);
    const double u2 = draw_u(key, (uint64_t)i, 2), u3 = draw_u(key, (uint64_t)i, 3);
    double v = (((u0 + u1) + u2) + u3 - 2.0) * 1.7320508075688772 * sigma;
    if (spike_p > 0.0 && draw_u(key, (uint64_t)i, 4) < spike_p) {
      const double mag = 100.0 + 900.0 * draw_u(key, (uint64_t)i, 5);
      v = (draw_u(key, (uint64_t)i, 6) < 0.5 ? -mag : mag) * sigma;
    }
    out[i] = (float)v;
  }
}

