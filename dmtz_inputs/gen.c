/*
 * dmtz_inputs/gen.c -- seeded synthetic inputs for tests and benchmarks.
 *
 * This module holds NONE of the method's arithmetic: it only produces original
 * fields f (shaped like the paper's datasets: climate, cosmology,
 * hurricane-like flows), the absolute bound xi for a relative bound, and the
 * decompressed field fhat from a built-in error-bounded quantizer standing in
 * for SZ3.  Both the CUDA path and the CPU oracle consume these
 * arrays; neither depends on this file otherwise.
 *
 * All arithmetic is f64 with -ffp-contract=off; every voxel is a pure function
 * of (seed, coordinates), so OpenMP scheduling cannot change the output.  The
 * closed-loop Lorenzo quantizer is sequential (raster order) by construction.
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

static inline uint64_t splitmix64(uint64_t x) {
  x += 0x9E3779B97F4A7C15ull;
  x = (x ^ (x >> 30)) * 0xBF58476D1CE4E5B9ull;
  x = (x ^ (x >> 27)) * 0x94D049BB133111EBull;
  return x ^ (x >> 31);
}
/* uniform in [0,1) from a 64-bit hash */
static inline double u01(uint64_t h) { return (double)(h >> 11) * (1.0 / 9007199254740992.0); }

static inline double lattice(uint64_t seed, int64_t ix, int64_t iy, int64_t iz, int oct) {
  uint64_t h = splitmix64(seed ^ splitmix64((uint64_t)ix * 0x8CB92BA72F3D8DD7ull ^
                                            (uint64_t)iy * 0xD6E8FEB86659FD93ull ^
                                            (uint64_t)iz * 0xA0761D6478BD642Full ^
                                            (uint64_t)oct * 0xE7037ED1A0B428DBull));
  return 2.0 * u01(h) - 1.0;
}
static inline double smooth(double t) { return t * t * (3.0 - 2.0 * t); }

/* smoothstep-interpolated value noise at lattice coordinates (x, y, z) */
static double value_noise(uint64_t seed, double x, double y, double z, int oct, int D) {
  double fx = floor(x), fy = floor(y), fz = floor(z);
  int64_t ix = (int64_t)fx, iy = (int64_t)fy, iz = (int64_t)fz;
  double tx = smooth(x - fx), ty = smooth(y - fy), tz = smooth(z - fz);
  double acc = 0.0;
  int zc = (D == 3) ? 2 : 1;
  for (int dz = 0; dz < zc; dz++)
    for (int dy = 0; dy < 2; dy++)
      for (int dx = 0; dx < 2; dx++) {
        double w = (dx ? tx : 1.0 - tx) * (dy ? ty : 1.0 - ty);
        if (D == 3) w *= (dz ? tz : 1.0 - tz);
        acc += w * lattice(seed, ix + dx, iy + dy, iz + dz, oct);
      }
  return acc;
}
/* sum_o beta^o * noise(p * 2^o / period) */
static double octave_noise(uint64_t seed, double x, double y, double z, double period, int octaves,
                           double beta, int D) {
  double s = 0.0, a = 1.0, fr = 1.0 / period;
  for (int o = 0; o < octaves; o++) {
    s += a * value_noise(seed, x * fr, y * fr, z * fr, o, D);
    a *= beta;
    fr *= 2.0;
  }
  return s;
}

/* A seeded RNG stream for the few global parameters (Gaussian centres, phases). */
typedef struct { uint64_t s; } rng_t;
static double rng_u(rng_t* r) { r->s = splitmix64(r->s); return u01(r->s); }
static double rng_range(rng_t* r, double a, double b) { return a + (b - a) * rng_u(r); }

enum { FAM_GAUSS2D = 0, FAM_CLIMATE = 1, FAM_HURRICANE = 2, FAM_LOGNORMAL = 3, FAM_MULTISCALE = 4,
       FAM_NOISE = 5 };

/* Raw (unnormalised) field r in f64 into out (nx fastest). */
int dmtz_gen_raw(int family, int64_t nx, int64_t ny, int64_t nz, uint64_t seed, double* out) {
  int D = (nz == 1) ? 2 : 3;
  int64_t N = nx * ny * nz;
  rng_t R = {seed * 0x2545F4914F6CDD1Dull + 1};
  const double PI = 3.14159265358979323846;
  if (family == FAM_GAUSS2D) {
    /* sum of 12 Gaussians, a in U[-1,1], sigma in U[2,8] px, centres in the domain */
    double a[12], s[12], cx[12], cy[12];
    for (int k = 0; k < 12; k++) {
      a[k] = rng_range(&R, -1, 1); s[k] = rng_range(&R, 2, 8);
      cx[k] = rng_range(&R, 0, (double)nx); cy[k] = rng_range(&R, 0, (double)ny);
    }
#pragma omp parallel for schedule(static)
    for (int64_t v = 0; v < N; v++) {
      double x = (double)(v % nx), y = (double)((v / nx) % ny), r = 0.0;
      for (int k = 0; k < 12; k++) {
        double dx = x - cx[k], dy = y - cy[k];
        r += a[k] * exp(-(dx * dx + dy * dy) / (2.0 * s[k] * s[k]));
      }
      out[v] = r;
    }
  } else if (family == FAM_CLIMATE) {
    /* lat x lon: 30 cos(phi) + sum_m (5/m) cos(m lam + th_m) cos(2 phi + ps_m)
     * + 400 anisotropic "river" Gaussians + 0.5 octave noise (256, 6, 0.55) */
    double th[13], ps[13];
    for (int m = 1; m <= 12; m++) { th[m] = rng_range(&R, 0, 2 * PI); ps[m] = rng_range(&R, 0, 2 * PI); }
    enum { NG = 400 };
    static double gA[NG], gx[NG], gy[NG], gsl[NG], gsp[NG];
    for (int k = 0; k < NG; k++) {
      gA[k] = rng_range(&R, 0, 8); gx[k] = rng_range(&R, 0, (double)nx); gy[k] = rng_range(&R, 0, (double)ny);
      gsl[k] = rng_range(&R, 20, 120); gsp[k] = rng_range(&R, 4, 20);
    }
    uint64_t nseed = splitmix64(seed ^ 0xC11Aull);
#pragma omp parallel for schedule(static)
    for (int64_t v = 0; v < N; v++) {
      double x = (double)(v % nx), y = (double)((v / nx) % ny);
      double lam = 2 * PI * x / (double)nx, phi = PI * (y / (double)(ny - 1) - 0.5);
      double r = 30.0 * cos(phi);
      for (int m = 1; m <= 12; m++) r += (5.0 / m) * cos(m * lam + th[m]) * cos(2 * phi + ps[m]);
      for (int k = 0; k < NG; k++) {
        double dx = (x - gx[k]) / gsl[k], dy = (y - gy[k]) / gsp[k];
        double e = 0.5 * (dx * dx + dy * dy);
        if (e < 40.0) r += gA[k] * exp(-e);
      }
      r += 0.5 * octave_noise(nseed, x, y, 0.0, 256.0, 6, 0.55, 2);
      out[v] = r;
    }
  } else if (family == FAM_HURRICANE) {
    /* Holland-like vortex with a drifting centre and a spiral band + 0.05 octave noise */
    uint64_t nseed = splitmix64(seed ^ 0x4A11ull);
    double sx = (double)nx / 500.0, sy = (double)ny / 500.0;
#pragma omp parallel for schedule(static)
    for (int64_t v = 0; v < N; v++) {
      double x = (double)(v % nx), y = (double)((v / nx) % ny), z = (double)(v / (nx * ny));
      double cx = sx * (250.0 + 30.0 * sin(z / 40.0)), cy = sy * (250.0 + 30.0 * cos(z / 40.0));
      double dx = x - cx, dy = y - cy, rr = sqrt(dx * dx + dy * dy);
      double Rm = 25.0 + 0.3 * z;
      double V = (rr / Rm) * exp(1.0 - rr / Rm) * exp(-z / 70.0);
      double th = atan2(dy, dx);
      double band = 0.2 * exp(-((rr - 80.0) / 15.0) * ((rr - 80.0) / 15.0)) * cos(2.0 * th - rr / 30.0);
      out[v] = V + band + 0.05 * octave_noise(nseed, x, y, z, 128.0, 6, 0.6, 3);
    }
  } else if (family == FAM_LOGNORMAL) {
    /* cosmology-like lognormal density: exp(sigma g) (1 + 0.002 U(-1,1)), sigma 2.5,
     * g = unit-variance octave noise (256, 9, 0.7) */
    uint64_t nseed = splitmix64(seed ^ 0xC05Full), wseed = splitmix64(seed ^ 0x7717ull);
#pragma omp parallel for schedule(static)
    for (int64_t v = 0; v < N; v++) {
      double x = (double)(v % nx), y = (double)((v / nx) % ny), z = (double)(v / (nx * ny));
      out[v] = octave_noise(nseed, x, y, z, 256.0, 9, 0.7, D);
    }
    /* unit variance, fixed-order (deterministic) sums */
    double s = 0.0, s2 = 0.0;
    for (int64_t v = 0; v < N; v++) { s += out[v]; s2 += out[v] * out[v]; }
    double mean = s / (double)N, sd = sqrt(s2 / (double)N - mean * mean);
    if (!(sd > 0)) sd = 1.0;
#pragma omp parallel for schedule(static)
    for (int64_t v = 0; v < N; v++) {
      double g = (out[v] - mean) / sd;
      double u = 2.0 * u01(splitmix64(wseed ^ (uint64_t)v)) - 1.0;
      out[v] = exp(2.5 * g) * (1.0 + 0.002 * u);
    }
  } else if (family == FAM_MULTISCALE) {
    /* octave noise (512, 8, 0.6) + 64 Gaussians, sigma in [40,160] */
    enum { NG = 64 };
    double a[NG], s[NG], cx[NG], cy[NG], cz[NG];
    for (int k = 0; k < NG; k++) {
      a[k] = rng_range(&R, -1, 1); s[k] = rng_range(&R, 40, 160);
      cx[k] = rng_range(&R, 0, (double)nx); cy[k] = rng_range(&R, 0, (double)ny);
      cz[k] = rng_range(&R, 0, (double)nz);
    }
    uint64_t nseed = splitmix64(seed ^ 0x3517ull);
#pragma omp parallel for schedule(static)
    for (int64_t v = 0; v < N; v++) {
      double x = (double)(v % nx), y = (double)((v / nx) % ny), z = (double)(v / (nx * ny));
      double r = octave_noise(nseed, x, y, z, 512.0, 8, 0.6, D);
      for (int k = 0; k < NG; k++) {
        double dx = x - cx[k], dy = y - cy[k], dz = z - cz[k];
        double e = (dx * dx + dy * dy + dz * dz) / (2.0 * s[k] * s[k]);
        if (e < 40.0) r += a[k] * exp(-e);
      }
      out[v] = r;
    }
  } else if (family == FAM_NOISE) {
    /* white noise (for small random test fields) */
#pragma omp parallel for schedule(static)
    for (int64_t v = 0; v < N; v++) out[v] = u01(splitmix64(seed ^ splitmix64((uint64_t)v)));
  } else {
    return 1;
  }
  return 0;
}

/* f = RN32(1 + (r - min)/(max - min) (1 - 2^-22)), so f lies in [1, 2). */
int dmtz_gen_normalize(const double* r, int64_t N, float* f) {
  double lo = r[0], hi = r[0];
  for (int64_t v = 1; v < N; v++) { if (r[v] < lo) lo = r[v]; if (r[v] > hi) hi = r[v]; }
  double span = hi - lo;
  if (!(span > 0)) span = 1.0;
  double scale = (1.0 - ldexp(1.0, -22)) / span;
#pragma omp parallel for schedule(static)
  for (int64_t v = 0; v < N; v++) f[v] = (float)(1.0 + (r[v] - lo) * scale);
  return 0;
}

/* absolute bound for a value-range-relative bound: RN32(eps (max f - min f)) in f64 */
float dmtz_gen_xi(const float* f, int64_t N, double eps) {
  float lo = f[0], hi = f[0];
  for (int64_t v = 1; v < N; v++) { if (f[v] < lo) lo = f[v]; if (f[v] > hi) hi = f[v]; }
  return (float)(eps * ((double)hi - (double)lo));
}

/* Closed-loop first-order Lorenzo quantizer (SZ-style), raster order over the
 * reconstructed values, out-of-domain neighbours = 0:
 *   k = rint((f - pred) / 2xi); |k| > 32767 -> fhat = f (unpredictable)
 *   else fhat = RN32(pred + 2 xi k); post-check |fhat - f| <= xi, else fhat = f. */
/* codes (optional): the quantization integer k of every vertex, or LORENZO_RAW when the
 * value is stored verbatim (unpredictable, |k| > 32767, or the post-check failed) --
 * what an SZ3-like compressor entropy-codes (used only for the CR / OCR size model). */
#define LORENZO_RAW 0x7FFFFFFF
int dmtz_gen_lorenzo_codes(const float* f, int64_t nx, int64_t ny, int64_t nz, float xi, float* fhat,
                           int32_t* codes);
int dmtz_gen_lorenzo(const float* f, int64_t nx, int64_t ny, int64_t nz, float xi, float* fhat) {
  return dmtz_gen_lorenzo_codes(f, nx, ny, nz, xi, fhat, 0);
}
int dmtz_gen_lorenzo_codes(const float* f, int64_t nx, int64_t ny, int64_t nz, float xi, float* fhat,
                           int32_t* codes) {
  double two_xi = 2.0 * (double)xi;
  for (int64_t z = 0; z < nz; z++)
    for (int64_t y = 0; y < ny; y++)
      for (int64_t x = 0; x < nx; x++) {
        int64_t v = x + nx * (y + ny * z);
#define H(dx, dy, dz) ((x - (dx) >= 0 && y - (dy) >= 0 && z - (dz) >= 0) ? \
                       (double)fhat[v - (dx) - nx * ((dy) + ny * (dz))] : 0.0)
        double pred = H(1, 0, 0) + H(0, 1, 0) - H(1, 1, 0);
        if (nz > 1) pred += H(0, 0, 1) - H(1, 0, 1) - H(0, 1, 1) + H(1, 1, 1);
#undef H
        double k = rint(((double)f[v] - pred) / two_xi);
        float out;
        int32_t code = (int32_t)k;
        if (fabs(k) > 32767.0) { out = f[v]; code = LORENZO_RAW; }
        else out = (float)(pred + two_xi * k);
        double e = (double)out - (double)f[v];
        if (!(fabs(e) <= (double)xi)) { out = f[v]; code = LORENZO_RAW; }
        fhat[v] = out;
        if (codes) codes[v] = code;
      }
  return 0;
}

/* fhat = RN32(f + xi u), u ~ U[-1, 1] (seeded), with the same post-check */
int dmtz_gen_uniform_noise(const float* f, int64_t N, float xi, uint64_t seed, float* fhat) {
#pragma omp parallel for schedule(static)
  for (int64_t v = 0; v < N; v++) {
    double u = 2.0 * u01(splitmix64(seed ^ splitmix64((uint64_t)v ^ 0x5EEDull))) - 1.0;
    float out = (float)((double)f[v] + (double)xi * u);
    double e = (double)out - (double)f[v];
    if (!(fabs(e) <= (double)xi)) out = f[v];
    fhat[v] = out;
  }
  return 0;
}
