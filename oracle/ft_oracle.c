/*
 * oracle/ft_oracle.c -- CPU restatement ("port") of the reference's batched
 * trig-approximation path.
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and the
 * bench.py cpu_baseline / --impl reference legs may load this library, and
 * only as the checker or the timed CPU baseline -- never as the product path.
 *
 * Every function cites the reference line it restates (R: = /root/reference).
 * The arithmetic is IEEE binary64, evaluated in exactly the reference's
 * operation order; build with -ffp-contract=off (no FMA contraction), which is
 * what the reference's own default x86-64 build does.
 *
 * Parity pin: tests/test_oracle_pin.py checks this port bit-for-bit against
 * the unmodified reference headers compiled in oracle/_ref (ref_shim.cpp) and
 * against the committed golden vectors in tests/golden/ (made by the
 * reference itself, tests/golden/make_golden.py).  The Taylor comparator has
 * no reference code (SPEC.md:213-266 only); it is pinned against the SPEC's
 * known-answer examples (with the 0.99922 -> 0.999171 fix).
 */
#include <math.h>
#include <pthread.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#define ORA_PI 0x1.921fb54442d18p+1 /* std::numbers::pi as a double */

static const double kPi = ORA_PI;           /* R:proj/include/fasttrig/reduction.hpp:18 */
static const double kTwoPi = 2.0 * ORA_PI;  /* reduction.hpp:19 */
static const double kHalfPi = 0.5 * ORA_PI; /* reduction.hpp:20 */
static const double kTanPoleGuard = 1e-3;   /* kernels.hpp:17 */
static const uint64_t kFisrMagic = 0x5fe6eb50c7b537a9ull; /* fisr.hpp:26 */

static uint64_t d2u(double d) { uint64_t u; memcpy(&u, &d, 8); return u; }
static double u2d(uint64_t u) { double d; memcpy(&d, &u, 8); return d; }

/* ------------------------------------------------------------------------ */
/* Segment table: segments.hpp:14-66                                         */
/* ------------------------------------------------------------------------ */
typedef struct { double a, b, c, d, X, Y, Z; } ora_seg;

static ora_seg g_seg[6];
static double g_knots[7];
static double g_sin_c[9], g_cos_c[9], g_tan_c[9];

/* segments.hpp:33-40 -- integer degree-space coefficients {a, b, c, d}. */
static const double kDegSeg[6][4] = {
    {11.0, 0.0, -1.0, 632.0},  {10.0, 10.0, -4.0, 657.0}, {6.0, 46.0, -5.0, 541.0},
    {10.0, 217.0, -13.0, 1252.0}, {4.0, 297.0, -10.0, 910.0}, {1.0, 542.0, -11.0, 990.0},
};

static void ora_init_tables(void) {
  /* segments.hpp:42 deg_per_rad = 180 / pi */
  const double deg_per_rad = 180.0 / kPi;
  for (int k = 0; k < 6; ++k) {
    /* segments.hpp:44-50 to_radian_segment */
    const double a = kDegSeg[k][0] * deg_per_rad;
    const double b = kDegSeg[k][1];
    const double c = kDegSeg[k][2] * deg_per_rad;
    const double d = kDegSeg[k][3];
    g_seg[k].a = a; g_seg[k].b = b; g_seg[k].c = c; g_seg[k].d = d;
    g_seg[k].X = a * a + c * c;
    g_seg[k].Y = 2.0 * (a * b + c * d);
    g_seg[k].Z = b * b + d * d;
  }
  /* segments.hpp:60 */
  g_knots[0] = 0.0;
  g_knots[1] = kPi / 12.0;
  g_knots[2] = kPi / 6.0;
  g_knots[3] = kPi / 4.0;
  g_knots[4] = kPi / 3.0;
  g_knots[5] = 5.0 * kPi / 12.0;
  g_knots[6] = kPi / 2.0;

  /* Taylor coefficients: exact rationals converted
   * once.  n! for n <= 17 is exact in binary64, so 1.0/n! is one rounding. */
  double fact = 1.0; /* running k! */
  double f[18];
  f[0] = 1.0;
  for (int k = 1; k < 18; ++k) { fact = fact * (double)k; f[k] = fact; }
  for (int k = 0; k < 9; ++k) {
    double s = 1.0 / f[2 * k + 1];
    double c = 1.0 / f[2 * k];
    g_sin_c[k] = (k & 1) ? -s : s;
    g_cos_c[k] = (k & 1) ? -c : c;
  }
  /* SPEC.md:242 tangent Maclaurin coefficients. */
  static const double tn[9] = {1.0, 1.0, 2.0, 17.0, 62.0, 1382.0, 21844.0, 929569.0, 6404582.0};
  static const double td[9] = {1.0, 3.0, 15.0, 315.0, 2835.0, 155925.0, 6081075.0,
                               638512875.0, 10854718875.0};
  for (int k = 0; k < 9; ++k) g_tan_c[k] = tn[k] / td[k];
}

static pthread_once_t g_once = PTHREAD_ONCE_INIT;
static void ensure_init(void) { pthread_once(&g_once, ora_init_tables); }

/* Copies the table as 6x{a,b,c,d,X,Y,Z} followed by the 7 knots (49 doubles). */
void ora_segment_table(double* out49) {
  ensure_init();
  for (int k = 0; k < 6; ++k) {
    const double* s = &g_seg[k].a;
    for (int j = 0; j < 7; ++j) out49[k * 7 + j] = s[j];
  }
  for (int j = 0; j < 7; ++j) out49[42 + j] = g_knots[j];
}

void ora_taylor_coeffs(double* sin9, double* cos9, double* tan9) {
  ensure_init();
  memcpy(sin9, g_sin_c, sizeof g_sin_c);
  memcpy(cos9, g_cos_c, sizeof g_cos_c);
  memcpy(tan9, g_tan_c, sizeof g_tan_c);
}

/* segments.hpp:70-73 -- five knot comparisons, not a division. */
int ora_segment_index(double red) {
  ensure_init();
  const double* k = g_knots;
  return (red >= k[1]) + (red >= k[2]) + (red >= k[3]) + (red >= k[4]) + (red >= k[5]);
}

/* ------------------------------------------------------------------------ */
/* FISR: fisr.hpp:14-46.  method 0 = exact, 1 = fisr; steps = newton_steps.  */
/* ------------------------------------------------------------------------ */
double ora_fast_inverse_sqrt(double v, int method, int steps) {
  if (!(v > 0.0) || v == INFINITY) return u2d(0x7ff8000000000000ull); /* :32-34 */
  if (method == 0) return 1.0 / sqrt(v);                                /* :35-37 */
  uint64_t bits = d2u(v);                                               /* :38 */
  bits = kFisrMagic - (bits >> 1);                                      /* :39 */
  double y = u2d(bits);                                                 /* :40 */
  const double half_v = 0.5 * v;                                        /* :41 */
  for (int i = 0; i < steps; ++i) y = y * (1.5 - half_v * y * y);       /* :42-44 */
  return y;
}

/* ------------------------------------------------------------------------ */
/* Range reduction: reduction.hpp:26-93                                      */
/* ------------------------------------------------------------------------ */
static double mod_positive(double a, double period) { /* reduction.hpp:26-30 */
  double r = a - period * floor(a / period);
  r = r < 0.0 ? 0.0 : r;
  return r < period ? r : 0.0;
}

static double clamp_red(double red) { /* reduction.hpp:32-35 */
  red = red < 0.0 ? 0.0 : red;
  return red < kHalfPi ? red : kHalfPi;
}

static void fold_quadrant(double r, double* red_out, double* q_out) { /* :44-52 */
  double q = floor(r / kHalfPi);
  q = q > 3.0 ? 3.0 : q;
  const double red = q == 0.0 ? r : q == 1.0 ? kPi - r : q == 2.0 ? r - kPi : kTwoPi - r;
  *red_out = clamp_red(red);
  *q_out = q;
}

void ora_reduce_sin(double x, double* red, double* sign) { /* reduction.hpp:59-68 */
  if (!isfinite(x)) { *red = u2d(0x7ff8000000000000ull); *sign = 1.0; return; }
  const double r = mod_positive(fabs(x), kTwoPi);
  double q;
  fold_quadrant(r, red, &q);
  double s = q < 2.0 ? 1.0 : -1.0;
  *sign = signbit(x) ? -s : s;
}

void ora_reduce_cos(double x, double* red, double* sign) { /* reduction.hpp:71-79 */
  if (!isfinite(x)) { *red = u2d(0x7ff8000000000000ull); *sign = 1.0; return; }
  const double r = mod_positive(fabs(x), kTwoPi);
  double q;
  fold_quadrant(r, red, &q);
  *sign = (q == 0.0 || q == 3.0) ? 1.0 : -1.0;
}

void ora_reduce_tan(double x, double* red, double* sign) { /* reduction.hpp:83-93 */
  if (!isfinite(x)) { *red = u2d(0x7ff8000000000000ull); *sign = 1.0; return; }
  const double r = mod_positive(fabs(x), kPi);
  const int upper = r > kHalfPi;
  *red = clamp_red(upper ? kPi - r : r);
  double s = upper ? -1.0 : 1.0;
  *sign = signbit(x) ? -s : s;
}

/* ------------------------------------------------------------------------ */
/* Evaluators: kernels.hpp:19-67                                             */
/* ------------------------------------------------------------------------ */
static double eval_sin_segment(const ora_seg* s, double red, int m, int st) { /* :19-23 */
  const double poly = s->a * red + s->b;
  const double radicand = (s->X * red + s->Y) * red + s->Z;
  return poly * ora_fast_inverse_sqrt(radicand, m, st);
}

static double eval_cos_segment(const ora_seg* s, double red, int m, int st) { /* :25-29 */
  const double poly = s->c * red + s->d;
  const double radicand = (s->X * red + s->Y) * red + s->Z;
  return poly * ora_fast_inverse_sqrt(radicand, m, st);
}

static double eval_tan_segment(const ora_seg* s, double red, int m, int st) { /* :33-41 */
  const double poly = s->a * red + s->b;
  const double den = s->c * red + s->d;
  if (m == 0) return poly / den;
  const double r = ora_fast_inverse_sqrt(den, m, st);
  return poly * (r * r);
}

double ora_proposed_sin(double x, int m, int st) { /* kernels.hpp:46-50 */
  ensure_init();
  double red, sign;
  ora_reduce_sin(x, &red, &sign);
  const ora_seg* s = &g_seg[ora_segment_index(red)];
  return sign * eval_sin_segment(s, red, m, st);
}

double ora_proposed_cos(double x, int m, int st) { /* kernels.hpp:52-56 */
  ensure_init();
  double red, sign;
  ora_reduce_cos(x, &red, &sign);
  const ora_seg* s = &g_seg[ora_segment_index(red)];
  return sign * eval_cos_segment(s, red, m, st);
}

double ora_proposed_tan(double x, int m, int st) { /* kernels.hpp:60-67 */
  ensure_init();
  double red, sign;
  ora_reduce_tan(x, &red, &sign);
  if (fabs(red - kHalfPi) < kTanPoleGuard) return sign * INFINITY;
  const ora_seg* s = &g_seg[ora_segment_index(red)];
  return sign * eval_tan_segment(s, red, m, st);
}

/* Segment choice per element (the parity contract's "identical segment index"):
 * sin and cos share one (both reduce to the same red, reduction.hpp:59-79);
 * tan has its own, or 255 inside the pole-guard window (kernels.hpp:62-64). */
int ora_seg_sincos(double x) {
  double red, sign;
  ora_reduce_sin(x, &red, &sign);
  return ora_segment_index(red);
}
int ora_seg_tan(double x) {
  double red, sign;
  ora_reduce_tan(x, &red, &sign);
  if (fabs(red - kHalfPi) < kTanPoleGuard) return 255;
  return ora_segment_index(red);
}

/* ------------------------------------------------------------------------ */
/* Taylor comparator: SPEC.md:224-247,254-256 (no reference code exists).    */
/* Pinned order: s = red*red; p = c[n-1]; p = p*s + c[k] for k = n-2..0;     */
/* sin = sign*(red*p), cos = sign*p, tan = sign*(red*p); no pole guard.      */
/* ------------------------------------------------------------------------ */
static double horner(const double* c, int n, double s) {
  double p = c[n - 1];
  for (int k = n - 2; k >= 0; --k) p = p * s + c[k];
  return p;
}

double ora_taylor_sin(double x, int n) {
  ensure_init();
  double red, sign;
  ora_reduce_sin(x, &red, &sign);
  return sign * (red * horner(g_sin_c, n, red * red));
}
double ora_taylor_cos(double x, int n) {
  ensure_init();
  double red, sign;
  ora_reduce_cos(x, &red, &sign);
  return sign * horner(g_cos_c, n, red * red);
}
double ora_taylor_tan(double x, int n) {
  ensure_init();
  double red, sign;
  ora_reduce_tan(x, &red, &sign);
  return sign * (red * horner(g_tan_c, n, red * red));
}

/* ------------------------------------------------------------------------ */
/* Batched forms (kernels.hpp:71-94 semantics, multi-threaded).              */
/* dtype 0 = f32 (promote, evaluate in f64, one RN to float), 1 = f64.       */
/* mask bit0 sin, bit1 cos, bit2 tan.  kind 0 = proposed, 1 = taylor.        */
/* ------------------------------------------------------------------------ */
typedef struct {
  int dtype, kind, m, st, nterms;
  unsigned mask;
  const void* x;
  void *s, *c, *t;
  uint8_t *seg_sc, *seg_t;
  size_t lo, hi;
} ora_job;

static void* ora_worker(void* p) {
  const ora_job* j = (const ora_job*)p;
  for (size_t i = j->lo; i < j->hi; ++i) {
    const double x = j->dtype == 0 ? (double)((const float*)j->x)[i] : ((const double*)j->x)[i];
    double vs = 0, vc = 0, vt = 0;
    if (j->kind == 0) {
      if (j->mask & 1u) vs = ora_proposed_sin(x, j->m, j->st);
      if (j->mask & 2u) vc = ora_proposed_cos(x, j->m, j->st);
      if (j->mask & 4u) vt = ora_proposed_tan(x, j->m, j->st);
    } else {
      if (j->mask & 1u) vs = ora_taylor_sin(x, j->nterms);
      if (j->mask & 2u) vc = ora_taylor_cos(x, j->nterms);
      if (j->mask & 4u) vt = ora_taylor_tan(x, j->nterms);
    }
    if (j->dtype == 0) {
      if (j->mask & 1u) ((float*)j->s)[i] = (float)vs;
      if (j->mask & 2u) ((float*)j->c)[i] = (float)vc;
      if (j->mask & 4u) ((float*)j->t)[i] = (float)vt;
    } else {
      if (j->mask & 1u) ((double*)j->s)[i] = vs;
      if (j->mask & 2u) ((double*)j->c)[i] = vc;
      if (j->mask & 4u) ((double*)j->t)[i] = vt;
    }
    if (j->seg_sc) j->seg_sc[i] = (uint8_t)ora_seg_sincos(x);
    if (j->seg_t) j->seg_t[i] = (uint8_t)ora_seg_tan(x);
  }
  return NULL;
}

static int ora_run(ora_job base, size_t n, int nthreads) {
  ensure_init();
  if (nthreads < 1) nthreads = 1;
  if ((size_t)nthreads > n) nthreads = n ? (int)n : 1;
  pthread_t* th = (pthread_t*)malloc(sizeof(pthread_t) * (size_t)nthreads);
  ora_job* jobs = (ora_job*)malloc(sizeof(ora_job) * (size_t)nthreads);
  if (!th || !jobs) { free(th); free(jobs); return 3; }
  for (int k = 0; k < nthreads; ++k) {
    jobs[k] = base;
    jobs[k].lo = n * (size_t)k / (size_t)nthreads;
    jobs[k].hi = n * (size_t)(k + 1) / (size_t)nthreads;
  }
  for (int k = 1; k < nthreads; ++k) pthread_create(&th[k], NULL, ora_worker, &jobs[k]);
  ora_worker(&jobs[0]);
  for (int k = 1; k < nthreads; ++k) pthread_join(th[k], NULL);
  free(th);
  free(jobs);
  return 0;
}

int ora_proposed_batch(int dtype, const void* x, size_t n, unsigned mask, int method, int steps,
                       void* s, void* c, void* t, uint8_t* seg_sc, uint8_t* seg_t, int nthreads) {
  ora_job j = {dtype, 0, method, steps, 0, mask, x, s, c, t, seg_sc, seg_t, 0, 0};
  return ora_run(j, n, nthreads);
}

int ora_taylor_batch(int dtype, const void* x, size_t n, unsigned mask, int nterms, void* s,
                     void* c, void* t, int nthreads) {
  if (nterms < 1 || nterms > 9) return 1;
  ora_job j = {dtype, 1, 0, 0, nterms, mask, x, s, c, t, NULL, NULL, 0, 0};
  return ora_run(j, n, nthreads);
}

/* ------------------------------------------------------------------------ */
/* Seeded inputs: SplitMix64 in counter form.                  */
/* Output i of the stream seeded with `seed` is mix(seed + (i+1)*gamma); that */
/* is exactly the i-th value of the sequential generator, so the device      */
/* generator (K4) can produce any shard without replaying the stream.        */
/* u = (z >> 11) * 2^-53; x = lo + (hi - lo) * u in binary64,  */
/* then one RN to float for f32 arrays.                                      */
/* ------------------------------------------------------------------------ */
uint64_t ora_splitmix64(uint64_t seed, uint64_t i) {
  uint64_t z = seed + (i + 1) * 0x9E3779B97F4A7C15ull;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

void ora_gen_uniform(int dtype, double lo, double hi, uint64_t seed, uint64_t offset, size_t n,
                     void* out) {
  const double span = hi - lo;
  for (size_t i = 0; i < n; ++i) {
    const double u = (double)(ora_splitmix64(seed, offset + i) >> 11) * 0x1p-53;
    const double x = lo + span * u;
    if (dtype == 0) ((float*)out)[i] = (float)x;
    else ((double*)out)[i] = x;
  }
}
