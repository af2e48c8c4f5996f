/*
 * synth/csynth.c -- seeded, counter-based synthetic input generators.
 *
 * Shared by the tests, the oracle legs and the bench: they hold NONE of the
 * method's arithmetic (no EVD, norm, dot, rotation).  Every value is a pure
 * function of (seed, stream, global index), so a shard of a batch generated
 * on rank k is bit-identical to the same slice of the whole batch (sharding
 * across GPUs never changes inputs).  Recipe: DESIGN.md "Synthetic inputs".
 */
#include <math.h>
#include <stdint.h>
#include <string.h>

/* SplitMix64 finaliser over a Weyl-sequence counter built from the triple. */
uint64_t synth_sm64(uint64_t seed, uint64_t stream, uint64_t idx)
{
  uint64_t z = seed * 0xD1B54A32D192ED03ull + stream * 0x8CB92BA72F3D8DD7ull +
               (idx + 1ull) * 0x9E3779B97F4A7C15ull;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

static double of_bits(uint64_t u) { double x; memcpy(&x, &u, 8); return x; }

/* +-m * 2^e, m ~ U[1,2) (52 random bits), e ~ U{lo..hi}, random sign */
static double signed_pow2(uint64_t u, int lo, int hi)
{
  double m = 1.0 + (double)((u >> 11) & 0xFFFFFFFFFFFFFull) * 0x1p-52;
  int e = lo + (int)((u & 0x7FFull) % (uint64_t)(hi - lo + 1));
  double v = ldexp(m, e);
  return (u >> 63) ? -v : v;
}

static double random_subnormal(uint64_t u)
{
  uint64_t b = (u & 0xFFFFFFFFFFFFFull) | 1ull; /* nonzero 52-bit significand, exponent 0 */
  double v = of_bits(b);
  return (u >> 63) ? -v : v;
}

/* Configuration 1 (BASELINE.json configs[0]): real symmetric batch.
 * a11, a22, a21 = +-m 2^e, e ~ U{-20..20}; 1% specials, kind uniform over
 * {one entry -> +0, a21 -> random nonzero subnormal, one entry -> +-m 2^1020}. */
void synth_evd_cfg1(uint64_t seed, int64_t off, int64_t r, double *a11, double *a22, double *a21)
{
#pragma omp parallel for schedule(static)
  for (int64_t k = 0; k < r; ++k) {
    uint64_t l = (uint64_t)(off + k);
    double v[3];
    for (int s = 0; s < 3; ++s) v[s] = signed_pow2(synth_sm64(seed, (uint64_t)s, l), -20, 20);
    uint64_t u = synth_sm64(seed, 8, l);
    if (u % 100 == 0) {
      uint64_t w = synth_sm64(seed, 9, l);
      int kind = (int)((u >> 32) % 3), ent = (int)((u >> 40) % 3);
      if (kind == 0) v[ent] = 0.0;
      else if (kind == 1) v[2] = random_subnormal(w);
      else v[ent] = signed_pow2(w & ~0x7FFull, 1020, 1020);
    }
    a11[k] = v[0];
    a22[k] = v[1];
    a21[k] = v[2];
  }
}

/* Configuration 2 (configs[1]): complex Hermitian batch.
 * a11, a22, Re a21, Im a21 = +-m 2^e, e ~ U{-1000..1000}; with probability 2%
 * both Re and Im a21 -> random nonzero subnormals; with probability 1% one of
 * the 4 components -> +-m 2^1023.                                            */
void synth_evd_cfg2(uint64_t seed, int64_t off, int64_t r, double *a11, double *a22, double *re,
                    double *im)
{
#pragma omp parallel for schedule(static)
  for (int64_t k = 0; k < r; ++k) {
    uint64_t l = (uint64_t)(off + k);
    double v[4];
    for (int s = 0; s < 4; ++s)
      v[s] = signed_pow2(synth_sm64(seed, (uint64_t)s, l), -1000, 1000);
    uint64_t u = synth_sm64(seed, 8, l);
    uint64_t x = u % 100;
    if (x < 2) {
      v[2] = random_subnormal(synth_sm64(seed, 9, l));
      v[3] = random_subnormal(synth_sm64(seed, 10, l));
    } else if (x == 2) {
      int ent = (int)((u >> 40) % 4);
      v[ent] = signed_pow2(synth_sm64(seed, 9, l) & ~0x7FFull, 1023, 1023);
    }
    a11[k] = v[0];
    a22[k] = v[1];
    re[k] = v[2];
    im[k] = v[3];
  }
}

/* ---- single-precision analogues (the fp32 EVD, NEXT-1): binary32 values
 * +-m 2^e with m ~ U[1,2) (23 random bits); configs[0]-like: e ~ U{-20..20},
 * 1% specials {one entry -> +0, a21 -> random nonzero subnormal, one entry ->
 * +-m 2^124}; configs[1]-like: e ~ U{-120..120} (the float exponent range as
 * configs[1]'s +-1000 is the double's), 2% both Re and Im a21 subnormal, 1% one
 * component -> +-m 2^127.                                                    */
static float of_bits_f(uint32_t u) { float x; memcpy(&x, &u, 4); return x; }
static float signed_pow2_f(uint64_t u, int lo, int hi)
{
  float m = 1.0f + (float)((u >> 11) & 0x7FFFFFull) * 0x1p-23f;
  int e = lo + (int)((u & 0x7FFull) % (uint64_t)(hi - lo + 1));
  float v = ldexpf(m, e);
  return (u >> 63) ? -v : v;
}
static float random_subnormal_f(uint64_t u)
{
  float v = of_bits_f((uint32_t)(u & 0x7FFFFFull) | 1u);
  return (u >> 63) ? -v : v;
}

void synth_evd_cfg1_f32(uint64_t seed, int64_t off, int64_t r, float *a11, float *a22, float *a21)
{
#pragma omp parallel for schedule(static)
  for (int64_t k = 0; k < r; ++k) {
    uint64_t l = (uint64_t)(off + k);
    float v[3];
    for (int s = 0; s < 3; ++s) v[s] = signed_pow2_f(synth_sm64(seed, (uint64_t)s, l), -20, 20);
    uint64_t u = synth_sm64(seed, 8, l);
    if (u % 100 == 0) {
      uint64_t w = synth_sm64(seed, 9, l);
      int kind = (int)((u >> 32) % 3), ent = (int)((u >> 40) % 3);
      if (kind == 0) v[ent] = 0.0f;
      else if (kind == 1) v[2] = random_subnormal_f(w);
      else v[ent] = signed_pow2_f(w & ~0x7FFull, 124, 124);
    }
    a11[k] = v[0];
    a22[k] = v[1];
    a21[k] = v[2];
  }
}

void synth_evd_cfg2_f32(uint64_t seed, int64_t off, int64_t r, float *a11, float *a22, float *re,
                        float *im)
{
#pragma omp parallel for schedule(static)
  for (int64_t k = 0; k < r; ++k) {
    uint64_t l = (uint64_t)(off + k);
    float v[4];
    for (int s = 0; s < 4; ++s)
      v[s] = signed_pow2_f(synth_sm64(seed, (uint64_t)s, l), -120, 120);
    uint64_t u = synth_sm64(seed, 8, l);
    uint64_t x = u % 100;
    if (x < 2) {
      v[2] = random_subnormal_f(synth_sm64(seed, 9, l));
      v[3] = random_subnormal_f(synth_sm64(seed, 10, l));
    } else if (x == 2) {
      int ent = (int)((u >> 40) % 4);
      v[ent] = signed_pow2_f(synth_sm64(seed, 9, l) & ~0x7FFull, 127, 127);
    }
    a11[k] = v[0];
    a22[k] = v[1];
    re[k] = v[2];
    im[k] = v[3];
  }
}

/* N(0,1) by Box-Muller: out[k] = sqrt(-2 ln u1) cos(2 pi u2), u in (0,1],
 * u1, u2 from indices 2(off+k), 2(off+k)+1 of the stream.                   */
void synth_gauss(uint64_t seed, uint64_t stream, int64_t off, int64_t count, double *out)
{
#pragma omp parallel for schedule(static)
  for (int64_t k = 0; k < count; ++k) {
    uint64_t i = 2ull * (uint64_t)(off + k);
    double u1 = (double)((synth_sm64(seed, stream, i) >> 11) + 1ull) * 0x1p-53;
    double u2 = (double)((synth_sm64(seed, stream, i + 1) >> 11) + 1ull) * 0x1p-53;
    out[k] = sqrt(-2.0 * log(u1)) * cos(6.283185307179586 * u2);
  }
}

/* U[0,1) doubles (53 random bits) */
void synth_uniform(uint64_t seed, uint64_t stream, int64_t off, int64_t count, double *out)
{
#pragma omp parallel for schedule(static)
  for (int64_t k = 0; k < count; ++k)
    out[k] = (double)(synth_sm64(seed, stream, (uint64_t)(off + k)) >> 11) * 0x1p-53;
}
