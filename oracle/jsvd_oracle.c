/*
 * oracle/jsvd_oracle.c -- TEST INFRASTRUCTURE ONLY.
 *
 * A plain, slow, obviously-correct CPU oracle for the hot path of
 * arXiv 2202.08361 (Novakovic, "Vectorization of a thread-parallel Jacobi
 * singular value decomposition method").  Only tests/, __graft_entry__.smoke()
 * and bench.py's cpu_baseline / --impl reference legs may load this library.
 * It shares NO code, header, table or constant generator with the CUDA path
 * (paper_2202_08361_b200/csrc); neither side includes the other.
 *
 * Every function follows the paper's algorithm statement by statement with
 * s = 1 lanes (the scalar reading), in IEEE binary64,
 * round-to-nearest-even, using libm fma/sqrt/logb/scalbn/fmin/fmax/copysign.
 * Compile with -O2 -ffp-contract=off -fno-fast-math (no contraction).
 *
 * Citations "P:a-b" are PAPER.md line ranges; "R#k" are the readings listed in
 * DESIGN.md section "Readings of the paper" (same numbering as SURVEY.md 8(c).4).
 *
 * Pins (tests/test_oracle_*.py) tie every function here to something other
 * than itself: the paper's worked examples, closed forms, quad-precision
 * (__float128 / mpmath) references, invariants, and brute force.
 */
#include <float.h>
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

#define ORC_OK 0
#define ORC_ENOCONV 1
#define ORC_EINVAL (-1)
#define ORC_ENONFINITE (-2)
#define ORC_ERANK (-3)

#define ORC_EVD_TAN 0x1u
#define ORC_EVD_NOBACKSCALE 0x2u
#define ORC_ZETA_ZERO INT32_MAX

/* ---------------------------------------------------------------- sign-bit ops
 * and/andnot/or/xor with -0.0.            */
static uint64_t bits_of(double x) { uint64_t u; memcpy(&u, &x, 8); return u; }
static double of_bits(uint64_t u) { double x; memcpy(&x, &u, 8); return x; }
static const uint64_t SIGN = 0x8000000000000000ull;
/* xor(x, and(y, -0)): multiplies the signs */
static double xor_sign(double x, double y) { return of_bits(bits_of(x) ^ (bits_of(y) & SIGN)); }

/* fl(sqrt(omega)) = 1.34078079299425956E+154 (R#1) */
static const double SQRT_OMEGA = 0x1.fffffffffffffp+511;

/* ---------------------------------------------------------------- Alg 2.1
 * naive hypot: x=|x|, y=|y|, m=min, M=max, q=max(m/M,0),
 * return sqrt(fma(q,q,1))*M.                                                 */
double orc_hypot(double x, double y)
{
  x = fabs(x);
  y = fabs(y);
  double m = fmin(x, y), M = fmax(x, y);
  double q = fmax(m / M, 0.0); /* max replaces 0/0 -> NaN with 0 */
  return sqrt(fma(q, q, 1.0)) * M;
}

/* ---------------------------------------------------------------- Eq. (z)
 * zeta = min{omega, eta - floor(lg|a_ij|) ...}, eta = 1020, lg 0 = -inf
 * (Alg 2.2 lines 6-8).  Returned as a double exactly as
 * in the paper (DBL_MAX for the zero matrix).                                */
double orc_zeta(double a11, double a22, double re, double im)
{
  const double eta = 1020.0;
  double z11 = eta - logb(a11), z22 = eta - logb(a22);
  double zr = eta - logb(re), zi = eta - logb(im);
  return fmin(DBL_MAX, fmin(fmin(z11, z22), fmin(zr, zi)));
}

/* scalef(x, zeta) with zeta = omega (the zero matrix, R#2): all entries are
 * zero then, and any huge finite scale gives the same zeros. */
static int zeta_int(double zd) { return zd >= 4096.0 ? 4096 : (int)zd; }

/* ---------------------------------------------------------------- Alg 2.2 / SM2.1
 * One Hermitian (is_complex) or real symmetric matrix of order two.
 * Statement order of z8jac2 / d8jac2, s = 1.
 * Outputs: l1, l2 (backscaled unless NOBACKSCALE), c = cos(phi),
 * (sr, si) = e^{ia} sin(phi) (default) or e^{ia} tan(phi)
 * under ORC_EVD_TAN; zeta (int, ORC_ZETA_ZERO for the zero matrix); p = perm. */
void orc_evd2_one(int is_complex, double a11, double a22, double re, double im, unsigned flags,
                  double *l1o, double *l2o, double *co, double *sro, double *sio, int32_t *zo,
                  int *po)
{
  if (!is_complex) im = 0.0;
  /* lines 6-8: the scaling exponent (Eq. z) */
  double zd = is_complex ? orc_zeta(a11, a22, re, im) : orc_zeta(a11, a22, re, 0.0);
  int iz = zeta_int(zd);
  /* lines 10-11: A <- 2^zeta A */
  re = scalbn(re, iz);
  if (is_complex) im = scalbn(im, iz);
  a11 = scalbn(a11, iz);
  a22 = scalbn(a22, iz);
  double ab, ca = 0.0, sa = 0.0;
  if (is_complex) {
    /* lines 12-18: polar form of a21 (Eq. zpolar) */
    double ar = fabs(re), ai = fabs(im);
    ab = orc_hypot(ar, ai);                         /* |a21| by Alg 2.1 */
    ca = copysign(fmin(ar / ab, 1.0), re);          /* min replaces 0/0 with 1; or() sign */
    sa = im / fmax(ab, DBL_TRUE_MIN);               /* max replaces 0 with mu_check */
  } else {
    ab = fabs(re);
  }
  /* lines 19-21: tan(2phi) (Eq. tan2) */
  double o = scalbn(ab, 1);
  double a = a11 - a22;
  double t2 = copysign(fmin(fmax(o / fabs(a), 0.0), SQRT_OMEGA), a);
  /* line 22-23: tan(phi) (Eq. jactan) */
  double sec2_2 = fma(t2, t2, 1.0);
  double t = t2 / (1.0 + sqrt(sec2_2));
  /* lines 24-25: sec^2, sec, cos (Eq. jacsec) */
  double s2 = fma(t, t, 1.0);
  double se = sqrt(s2);
  double c = 1.0 / se;
  /* lines 26-27: e^{ia} tan(phi) */
  double C, S;
  if (is_complex) {
    C = ca * t;
    S = sa * t;
  } else {
    C = xor_sign(t, re); /* +-tan(phi) = xor(tan(phi), sgn(a21)) */
    S = 0.0;
  }
  /* lines 28-30: eigenvalues (Eq. lamsec) */
  double l1 = fma(t, fma(a22, t, o), a11) / s2;
  double l2 = fma(t, fma(a11, t, -o), a22) / s2;
  int p = (l1 < l2); /* line 32, on the scaled values */
  if (!(flags & ORC_EVD_NOBACKSCALE)) {
    l1 = scalbn(l1, -iz);
    l2 = scalbn(l2, -iz);
  }
  double sr, si;
  if (flags & ORC_EVD_TAN) {
    sr = C;
    si = S;
  } else { /* P:793 comment: e^{ia} sin(phi) = e^{ia} tan(phi) / sec(phi) */
    sr = C / se;
    si = S / se;
  }
  *l1o = l1;
  *l2o = l2;
  *co = c;
  *sro = sr;
  if (sio) *sio = si;
  *zo = (zd == DBL_MAX) ? ORC_ZETA_ZERO : (int32_t)iz;
  *po = p;
}

/* Alg 2.3 zbjac2 / SM2.2 dbjac2: OpenMP over chunks
 * of 32 matrices (one perm word each); no dependencies between iterations. */
int orc_evd2_batched(int is_complex, int64_t r, const double *a11, const double *a22,
                     const double *re, const double *im, double *l1, double *l2, double *c,
                     double *sr, double *si, int32_t *zeta, uint32_t *perm, unsigned flags)
{
  if (r < 0 || (is_complex && (!im || !si)) || (!is_complex && (im || si))) return ORC_EINVAL;
  int64_t nw = (r + 31) / 32;
#pragma omp parallel for schedule(static)
  for (int64_t w = 0; w < nw; ++w) {
    uint32_t word = 0;
    for (int64_t l = w * 32; l < r && l < (w + 1) * 32; ++l) {
      int32_t z;
      int p;
      double dummy;
      orc_evd2_one(is_complex, a11[l], a22[l], re[l], is_complex ? im[l] : 0.0, flags, &l1[l],
                   &l2[l], &c[l], &sr[l], is_complex ? &si[l] : &dummy, &z, &p);
      if (zeta) zeta[l] = z;
      word |= (uint32_t)p << (l % 32);
    }
    if (perm) perm[w] = word;
  }
  return ORC_OK;
}

/* ================================================================== SVD step
 * Reduction spec R (R#15): element i goes to lane floor(i/c) mod W and is
 * accumulated in increasing i; lanes then combine as acc[L] = acc[L] + acc[L^o]
 * for each offset o in order; the result is acc[0].                         */
typedef struct {
  int32_t W, c, noffs;
  int32_t offs[32];
} orc_rspec;

static int rspec_ok(const orc_rspec *R)
{
  if (R->W < 1 || (R->W & (R->W - 1)) || R->c < 1 || R->noffs < 0 || R->noffs > 32) return 0;
  int32_t cover = 0;
  for (int k = 0; k < R->noffs; ++k) {
    int32_t o = R->offs[k];
    if (o <= 0 || (o & (o - 1)) || o >= R->W || (cover & o)) return 0;
    cover |= o;
  }
  return cover == R->W - 1;
}

static double rspec_combine(const orc_rspec *R, double *acc)
{
  double *tmp = (double *)malloc(sizeof(double) * (size_t)R->W);
  for (int k = 0; k < R->noffs; ++k) {
    int32_t o = R->offs[k];
    for (int32_t L = 0; L < R->W; ++L) tmp[L] = acc[L] + acc[L ^ o];
    memcpy(acc, tmp, sizeof(double) * (size_t)R->W);
  }
  free(tmp);
  return acc[0];
}

static int64_t lane_of(const orc_rspec *R, int64_t i) { return (i / R->c) % R->W; }

/* element accessors: real column x[i], complex interleaved x[2i], x[2i+1] */
static double re_at(int cplx, const double *x, int64_t i) { return cplx ? x[2 * i] : x[i]; }
static double im_at(int cplx, const double *x, int64_t i) { return cplx ? x[2 * i + 1] : 0.0; }

/* Column norm in (e,f) form (R#14):
 *   E = logb(max over components of |x|);  y = scalbn(x, -E);
 *   SSQ = sum over rows of fma(y_re,y_re,.) then fma(y_im,y_im,.) in spec R;
 *   k = logb(SSQ), g = scalbn(SSQ,-k); if k odd: g = 2g, k = k-1;
 *   f = sqrt(g), e = E + k/2.  Zero column -> (-inf, 1).                    */
void orc_colnorm(int cplx, int64_t m, const double *x, const orc_rspec *R, double *e, double *f)
{
  double mx = 0.0;
  for (int64_t i = 0; i < m; ++i) {
    mx = fmax(mx, fabs(re_at(cplx, x, i)));
    if (cplx) mx = fmax(mx, fabs(im_at(cplx, x, i)));
  }
  if (mx == 0.0) {
    *e = -INFINITY;
    *f = 1.0;
    return;
  }
  int E = (int)logb(mx);
  double *acc = (double *)calloc((size_t)R->W, sizeof(double));
  for (int64_t i = 0; i < m; ++i) {
    int64_t L = lane_of(R, i);
    double yr = scalbn(re_at(cplx, x, i), -E);
    acc[L] = fma(yr, yr, acc[L]);
    if (cplx) {
      double yi = scalbn(im_at(cplx, x, i), -E);
      acc[L] = fma(yi, yi, acc[L]);
    }
  }
  double ssq = rspec_combine(R, acc);
  free(acc);
  int k = (int)logb(ssq);
  double g = scalbn(ssq, -k);
  if (k & 1) { /* odd exponent: f' = 2f, e' = e - 1 */
    g = 2.0 * g;
    k = k - 1;
  }
  *f = sqrt(g);
  *e = (double)(E + k / 2);
}

/* Alg 3.1 zdpscl: columns prescaled by 2^{-e_j}, fma schedule
 * of lines 5-6 (re += Rq*Rp + Iq*Ip; im += Rq*Ip - Iq*Rp), reduction in spec R,
 * one division of both components by fl(f_q * f_p).  Real: its simplification.
 * A zero column (e = -inf) gives z = 0 (R#19).                               */
void orc_dot(int cplx, int64_t m, const double *xq, double eq, double fq, const double *xp,
             double ep, double fp, const orc_rspec *R, double *zre, double *zim)
{
  if (isinf(eq) || isinf(ep)) {
    *zre = 0.0;
    *zim = 0.0;
    return;
  }
  int iq = (int)eq, ip = (int)ep;
  double *ar = (double *)calloc((size_t)R->W, sizeof(double));
  double *ai = (double *)calloc((size_t)R->W, sizeof(double));
  for (int64_t i = 0; i < m; ++i) {
    int64_t L = lane_of(R, i);
    double rq = scalbn(re_at(cplx, xq, i), -iq), rp = scalbn(re_at(cplx, xp, i), -ip);
    if (cplx) {
      double jq = scalbn(im_at(cplx, xq, i), -iq), jp = scalbn(im_at(cplx, xp, i), -ip);
      ar[L] = fma(rq, rp, ar[L]);  /* line 5 */
      ai[L] = fma(rq, jp, ai[L]);
      ar[L] = fma(jq, jp, ar[L]);  /* line 6 */
      ai[L] = fma(-jq, rp, ai[L]); /* fnmadd */
    } else {
      ar[L] = fma(rq, rp, ar[L]);
    }
  }
  double zr = rspec_combine(R, ar);
  double zi = cplx ? rspec_combine(R, ai) : 0.0;
  free(ar);
  free(ai);
  double d = fq * fp; /* line 8: single division by fl(f_q f_p) */
  *zre = zr / d;
  *zim = cplx ? zi / d : 0.0;
}

/* Alg 3.2: transform iff upsilon <= fl(|z|) (naive hypot). */
int orc_cvg(double zre, double zim, double upsilon) { return upsilon <= orc_hypot(zre, zim); }

/* upsilon = fl(eps * sqrt(m)), eps = 2^-53 (Eq. tol; R#18) */
double orc_upsilon(int64_t m) { return scalbn(sqrt((double)m), -53); }

/* getmant(x, NORM_1_2, SIGN_zero) (Eq. F) */
static double getmant12(double x) { return scalbn(fabs(x), -(int)logb(x)); }

/* Alg 3.3: non-overflowing scaled Grammian of the pair. */
void orc_gram(double zre, double zim, double e1, double f1, double e2, double f2, double *a11,
              double *a22, double *b21re, double *b21im)
{
  double f12 = f1 / f2, e12 = e1 - e2; /* line 1 */
  double f21 = f2 / f1, e21 = e2 - e1;
  e12 = e12 + logb(f12); /* line 2 */
  f12 = getmant12(f12);
  e21 = e21 + logb(f21); /* line 3 */
  f21 = getmant12(f21);
  double sA = fmin(1023.0 - fmax(e12, e21), 0.0); /* line 4: eta_hat = DBL_MAX_EXP-1 */
  e12 = e12 + sA;                                 /* line 5 */
  e21 = e21 + sA;
  *a11 = scalbn(f12, (int)e12); /* line 6 */
  *a22 = scalbn(f21, (int)e21);
  *b21re = scalbn(zre, (int)sA); /* line 7 */
  *b21im = scalbn(zim, (int)sA);
}

/* Alg 3.4 zjrot / djrot with P = I (R#20): the fma schedule of
 * lines 5-6 and 9-10 (Eq. zfma + Eq. transf).  Returns max |component| of the
 * transformed columns.                                                       */
double orc_rot(int cplx, int64_t l, double *xp, double *xq, double c, double C, double S)
{
  double M = 0.0;
  for (int64_t i = 0; i < l; ++i) {
    if (cplx) {
      double rp = xp[2 * i], ip = xp[2 * i + 1], rq = xq[2 * i], iq = xq[2 * i + 1];
      double rp2 = fma(rq, C, fma(-iq, S, rp)) * c; /* line 5 */
      double ip2 = fma(rq, S, fma(iq, C, ip)) * c;  /* line 6 */
      double rq2 = fma(rp, -C, fma(-ip, S, rq)) * c; /* line 9 */
      double iq2 = fma(rp, S, fma(ip, -C, iq)) * c;  /* line 10 */
      xp[2 * i] = rp2;
      xp[2 * i + 1] = ip2;
      xq[2 * i] = rq2;
      xq[2 * i + 1] = iq2;
      M = fmax(M, fmax(fabs(rp2), fabs(ip2)));
      M = fmax(M, fmax(fabs(rq2), fabs(iq2)));
    } else {
      double p = xp[i], q = xq[i];
      double p2 = fma(q, C, p) * c;
      double q2 = fma(p, -C, q) * c;
      xp[i] = p2;
      xq[i] = q2;
      M = fmax(M, fmax(fabs(p2), fabs(q2)));
    }
  }
  return M;
}

/* One step of Alg 4.1 lines 7-38 over explicit disjoint pairs,
 * s = 1 (R#13), P = I (R#20).  col_e/col_f receive the norms of the step's
 * columns BEFORE rotation; *t += transformed pairs; *mmax = max(*mmax, M).
 * V has nv rows (the order of V; Alg 3.4 with l = n) and the same
 * column indexing as G -- nv > n when the caller holds only some columns.    */
int orc_step(int cplx, int64_t m, int64_t n, int64_t nv, double *G, int64_t ldg, double *V,
             int64_t ldv,
             const int32_t *pairs, int64_t npairs, double tol, const orc_rspec *R,
             double *col_e, double *col_f, int64_t *t_out, double *mmax)
{
  if (!rspec_ok(R) || m < 1 || n < 2 || ldg < m || (V && (nv < n || ldv < nv))) return ORC_EINVAL;
  const int64_t w = cplx ? 2 : 1;
  double upsilon = tol > 0.0 ? tol : orc_upsilon(m);
  int64_t t = 0;
  double M = 0.0;
#pragma omp parallel for schedule(static) reduction(+ : t) reduction(max : M)
  for (int64_t l = 0; l < npairs; ++l) {
    int64_t p = pairs[2 * l], q = pairs[2 * l + 1];
    double *gp = G + w * p * ldg, *gq = G + w * q * ldg;
    double ep, fp, eq, fq;
    orc_colnorm(cplx, m, gp, R, &ep, &fp); /* spade: norms */
    orc_colnorm(cplx, m, gq, R, &eq, &fq);
    col_e[p] = ep;
    col_f[p] = fp;
    col_e[q] = eq;
    col_f[q] = fq;
    double zr, zi;
    orc_dot(cplx, m, gq, eq, fq, gp, ep, fp, R, &zr, &zi); /* club: a21' = gq^* gp */
    if (!orc_cvg(zr, zi, upsilon)) continue;                /* heart: Alg 3.2 */
    double b11, b22, br, bi;
    orc_gram(zr, zi, ep, fp, eq, fq, &b11, &b22, &br, &bi); /* heart: Alg 3.3 */
    double l1, l2, c, C, S;
    int32_t z;
    int pp;
    orc_evd2_one(cplx, b11, b22, br, bi, ORC_EVD_TAN | ORC_EVD_NOBACKSCALE, &l1, &l2, &c, &C, &S,
                 &z, &pp); /* diamond */
    double Mp = orc_rot(cplx, m, gp, gq, c, C, S); /* star: G */
    if (V) orc_rot(cplx, nv, V + w * p * ldv, V + w * q * ldv, c, C, S); /* star: V */
    if (Mp > M) M = Mp;
    t += 1;
  }
  *t_out += t;
  if (M > *mmax) *mmax = M;
  return ORC_OK;
}

/* ================================================================ single precision
 * Alg 2.2 / SM2.1 converted to single precision as the paper prescribes
 * (P:709-717): omega = FLT_MAX, fl(sqrt(omega)) = 1.844674297E+19,
 * mu_check = FLT_TRUE_MIN, eta = FLT_MAX_EXP - 4 = 124; every operation in
 * IEEE binary32 (fmaf, sqrtf, logbf, scalbnf, fminf, fmaxf, copysignf and
 * float division), otherwise statement for statement the double oracle above.
 * (NEXT-1 of SURVEY 8(f); the same readings R#1-R#12 apply.)              */
static uint32_t bits_of_f(float x) { uint32_t u; memcpy(&u, &x, 4); return u; }
static float of_bits_f(uint32_t u) { float x; memcpy(&x, &u, 4); return x; }
static float xor_sign_f(float x, float y) { return of_bits_f(bits_of_f(x) ^ (bits_of_f(y) & 0x80000000u)); }

/* fl(sqrt(FLT_MAX)) = 0x1.fffffep+63 = 18446742974197923840 = 1.844674297E+19 */
static const float SQRT_OMEGA_F = 0x1.fffffep+63f;

float orc_hypot_f32(float x, float y)
{
  x = fabsf(x);
  y = fabsf(y);
  float m = fminf(x, y), M = fmaxf(x, y);
  float q = fmaxf(m / M, 0.0f);
  return sqrtf(fmaf(q, q, 1.0f)) * M;
}

float orc_zeta_f32(float a11, float a22, float re, float im)
{
  const float eta = 124.0f; /* FLT_MAX_EXP - 4 */
  float z11 = eta - logbf(a11), z22 = eta - logbf(a22);
  float zr = eta - logbf(re), zi = eta - logbf(im);
  return fminf(FLT_MAX, fminf(fminf(z11, z22), fminf(zr, zi)));
}

static int zeta_int_f(float zd) { return zd >= 4096.0f ? 4096 : (int)zd; }

void orc_evd2_one_f32(int is_complex, float a11, float a22, float re, float im, unsigned flags,
                      float *l1o, float *l2o, float *co, float *sro, float *sio, int32_t *zo,
                      int *po)
{
  if (!is_complex) im = 0.0f;
  float zd = is_complex ? orc_zeta_f32(a11, a22, re, im) : orc_zeta_f32(a11, a22, re, 0.0f);
  int iz = zeta_int_f(zd);
  re = scalbnf(re, iz);
  if (is_complex) im = scalbnf(im, iz);
  a11 = scalbnf(a11, iz);
  a22 = scalbnf(a22, iz);
  float ab, ca = 0.0f, sa = 0.0f;
  if (is_complex) {
    float ar = fabsf(re), ai = fabsf(im);
    ab = orc_hypot_f32(ar, ai);
    ca = copysignf(fminf(ar / ab, 1.0f), re);
    sa = im / fmaxf(ab, FLT_TRUE_MIN);
  } else {
    ab = fabsf(re);
  }
  float o = scalbnf(ab, 1);
  float a = a11 - a22;
  float t2 = copysignf(fminf(fmaxf(o / fabsf(a), 0.0f), SQRT_OMEGA_F), a);
  float sec2_2 = fmaf(t2, t2, 1.0f);
  float t = t2 / (1.0f + sqrtf(sec2_2));
  float s2 = fmaf(t, t, 1.0f);
  float se = sqrtf(s2);
  float c = 1.0f / se;
  float C, S;
  if (is_complex) {
    C = ca * t;
    S = sa * t;
  } else {
    C = xor_sign_f(t, re);
    S = 0.0f;
  }
  float l1 = fmaf(t, fmaf(a22, t, o), a11) / s2;
  float l2 = fmaf(t, fmaf(a11, t, -o), a22) / s2;
  int p = (l1 < l2);
  if (!(flags & ORC_EVD_NOBACKSCALE)) {
    l1 = scalbnf(l1, -iz);
    l2 = scalbnf(l2, -iz);
  }
  float sr, si;
  if (flags & ORC_EVD_TAN) {
    sr = C;
    si = S;
  } else {
    sr = C / se;
    si = S / se;
  }
  *l1o = l1;
  *l2o = l2;
  *co = c;
  *sro = sr;
  if (sio) *sio = si;
  *zo = (zd == FLT_MAX) ? ORC_ZETA_ZERO : (int32_t)iz;
  *po = p;
}

int orc_evd2_batched_f32(int is_complex, int64_t r, const float *a11, const float *a22,
                         const float *re, const float *im, float *l1, float *l2, float *c,
                         float *sr, float *si, int32_t *zeta, uint32_t *perm, unsigned flags)
{
  if (r < 0 || (is_complex && (!im || !si)) || (!is_complex && (im || si))) return ORC_EINVAL;
  int64_t nw = (r + 31) / 32;
#pragma omp parallel for schedule(static)
  for (int64_t w = 0; w < nw; ++w) {
    uint32_t word = 0;
    for (int64_t l = w * 32; l < r && l < (w + 1) * 32; ++l) {
      int32_t z;
      int p;
      float dummy;
      orc_evd2_one_f32(is_complex, a11[l], a22[l], re[l], is_complex ? im[l] : 0.0f, flags,
                       &l1[l], &l2[l], &c[l], &sr[l], is_complex ? &si[l] : &dummy, &z, &p);
      if (zeta) zeta[l] = z;
      word |= (uint32_t)p << (l % 32);
    }
    if (perm) perm[w] = word;
  }
  return ORC_OK;
}

/* ================================================================ strategy
 * R#20.  Flat round-robin (circle method) on P players, round r in [0,P-1):
 * position 0 = player 0, position k>=1 = player ((k-1+r) mod (P-1)) + 1;
 * pairs are positions (i, P-1-i), i in [0, P/2).                            */
static void circle(int64_t P, int64_t r, int64_t i, int64_t *a, int64_t *b)
{
  int64_t pos[2] = {i, P - 1 - i}, pl[2];
  for (int k = 0; k < 2; ++k) pl[k] = pos[k] == 0 ? 0 : ((pos[k] - 1 + r) % (P - 1)) + 1;
  *a = pl[0] < pl[1] ? pl[0] : pl[1];
  *b = pl[0] < pl[1] ? pl[1] : pl[0];
}

/* Block round-robin with B blocks of b = n/B columns (b even or b == 1):
 *  phase I  (steps 0..b-2): flat RR inside every block;
 *  phase II (B-1 rounds of b steps): rounds of flat RR over blocks; in round
 *  rr, block pair (beta, beta') runs b steps, step tt pairing column j of beta
 *  with column (j+tt) mod b of beta'.  n-1 steps, n/2 disjoint pairs each.
 *  Pairs listed block-pair by block-pair; (p, q) with p < q.                */
int orc_strategy_pairs(int64_t n, int64_t B, int64_t step, int32_t *pairs)
{
  if (n < 2 || (n & 1) || B < 2 || n % B) return ORC_EINVAL;
  int64_t b = n / B;
  if (b > 1 && (b & 1)) return ORC_EINVAL;
  if (step < 0 || step >= n - 1) return ORC_EINVAL;
  int64_t l = 0;
  if (step < b - 1) {
    for (int64_t beta = 0; beta < B; ++beta)
      for (int64_t i = 0; i < b / 2; ++i) {
        int64_t x, y;
        circle(b, step, i, &x, &y);
        pairs[2 * l] = (int32_t)(beta * b + x);
        pairs[2 * l + 1] = (int32_t)(beta * b + y);
        ++l;
      }
    return ORC_OK;
  }
  int64_t s2 = step - (b - 1);
  int64_t rr = s2 / b, tt = s2 % b;
  for (int64_t i = 0; i < B / 2; ++i) {
    int64_t be, bf;
    circle(B, rr, i, &be, &bf);
    for (int64_t j = 0; j < b; ++j) {
      int64_t x = be * b + j, y = bf * b + (j + tt) % b;
      pairs[2 * l] = (int32_t)(x < y ? x : y);
      pairs[2 * l + 1] = (int32_t)(x < y ? y : x);
      ++l;
    }
  }
  return ORC_OK;
}

/* rescale check points (R#21): start of phase I and of every phase-II round */
int orc_strategy_is_checkpoint(int64_t n, int64_t B, int64_t step)
{
  int64_t b = n / B;
  if (step == 0) return 1;
  if (step < b - 1) return 0;
  return ((step - (b - 1)) % b) == 0;
}

/* ================================================================ driver
 * Alg 4.1 zvjsvd / dvjsvd with s = 1, P = I, the scaled norms
 * of R#14, the rescaling heuristic of P:1071-1115 (Eqs. skn/skr, exact integer
 * floors R#28), finalize of P:1473-1485 and the sort of R#24.               */

/* floor(lg(omega / (varsigma m))) (real) / floor(lg(omega/(varsigma m sqrt2))) (complex) */
int orc_Fm(int cplx, int64_t m)
{
  int k = 0;
  while ((m >> (k + 1)) > 0) ++k; /* k = floor(lg m) */
  if (!cplx) return 1022 - k;
  /* m^2 >= 2^(2k+1)  <=>  lg m >= k + 1/2 */
  unsigned __int128 mm = (unsigned __int128)m * (unsigned __int128)m;
  unsigned __int128 th = (unsigned __int128)1 << (2 * k + 1);
  return 1021 - k - (mm >= th ? 1 : 0);
}

/* M-tilde: max over components of |entry|, NaN -> inf */
static double maxnorm(int cplx, int64_t m, int64_t n, const double *G, int64_t ldg)
{
  double x = 0.0;
  int64_t w = cplx ? 2 : 1;
  for (int64_t j = 0; j < n; ++j)
    for (int64_t i = 0; i < w * m; ++i) x = fmax(x, fmin(fabs(G[w * j * ldg + i]), INFINITY));
  return x;
}

static void scale_matrix(int cplx, int64_t m, int64_t n, double *G, int64_t ldg, int s)
{
  int64_t w = cplx ? 2 : 1;
  for (int64_t j = 0; j < n; ++j)
    for (int64_t i = 0; i < w * m; ++i) G[w * j * ldg + i] = scalbn(G[w * j * ldg + i], s);
}

/* s0_adjust: an integer added to the initial scaling exponent s0 of Eq. (skn)
 * (0 = the paper's s0 = s_[0]).  Any s0 with a finite G1 is safe: the Eq. (skr)
 * check at step 0 downscales a G1 that is too large, so a positive adjustment
 * is the way to make the rescale of P:1071-1115 fire (with the paper's s0 it
 * cannot: DESIGN.md R#40).  *scale_out (optional) receives the final s, the
 * effective scaling exponent: G = 2^s (iteration matrix without scaling).   */
int orc_gesvj(int cplx, int64_t m, int64_t n, double *A, int64_t lda, double *V, int64_t ldv,
              double *sigma, double *sigma_e, double *sigma_f, int64_t B, int32_t max_sweeps,
              int32_t *sweeps_done, int64_t *tps, int32_t s0_adjust, int32_t *scale_out,
              const orc_rspec *R)
{
  if (m < n || n < 2 || (n & 1) || lda < m || ldv < n || !rspec_ok(R) || max_sweeps < 0)
    return ORC_EINVAL;
  if (B != n && (n % B || ((n / B) & 1))) return ORC_EINVAL;
  if (s0_adjust < -2200 || s0_adjust > 2200) return ORC_EINVAL;
  const int64_t w = cplx ? 2 : 1;
  /* line 1: M0, s0, G1 = 2^s0 G0 (Eq. skn) */
  double Mt = maxnorm(cplx, m, n, A, lda);
  if (isinf(Mt)) return ORC_ENONFINITE;
  if (Mt == 0.0) return ORC_ERANK;
  const int Fm = orc_Fm(cplx, m);
  const int Kr = cplx ? 1020 : 1022; /* floor(lg(omega/varsigma)) [-1]: Eq. skr */
  int s = Fm - (int)logb(Mt) - 1 + s0_adjust;
  if ((int)logb(Mt) + s > 1023) return ORC_EINVAL; /* G1 would overflow */
  scale_matrix(cplx, m, n, A, lda, s);
  Mt = scalbn(Mt, s);
  /* line 2: V = I */
  for (int64_t j = 0; j < n; ++j)
    for (int64_t i = 0; i < w * n; ++i) V[w * j * ldv + i] = (i == w * j) ? 1.0 : 0.0;
  double *ce = (double *)malloc(sizeof(double) * (size_t)n);
  double *cf = (double *)malloc(sizeof(double) * (size_t)n);
  int32_t *pairs = (int32_t *)malloc(sizeof(int32_t) * (size_t)n);
  double upsilon = orc_upsilon(m);
  int32_t C = 0;
  int converged = 0;
  for (C = 0; C < max_sweeps; ++C) { /* line 3 */
    int64_t T = 0;
    for (int64_t k = 0; k < n - 1; ++k) { /* line 5 */
      if (orc_strategy_is_checkpoint(n, B, k)) { /* line 6 (R#21) */
        int sk = Kr - (int)logb(Mt);
        if (sk < 0) {
          int sn = Fm - (int)logb(Mt) - 1;
          scale_matrix(cplx, m, n, A, lda, sn);
          Mt = scalbn(Mt, sn);
          s += sn;
        }
      }
      orc_strategy_pairs(n, B, k, pairs);
      int64_t t = 0;
      double M = 0.0;
      orc_step(cplx, m, n, n, A, lda, V, ldv, pairs, n / 2, upsilon, R, ce, cf, &t, &M);
      T += t;
      Mt = fmax(Mt, M); /* line 38 */
    }
    if (tps) tps[C] = T;
    if (T == 0) { /* line 40 */
      converged = 1;
      ++C;
      break;
    }
  }
  if (sweeps_done) *sweeps_done = C;
  if (scale_out) *scale_out = s;
  /* the column norms of the final iterate, recomputed with the same R (R#23):
   * if converged they equal those of the last sweep (no column changed). */
  for (int64_t j = 0; j < n; ++j) orc_colnorm(cplx, m, A + w * j * lda, R, &ce[j], &cf[j]);
  if (!converged) {
    /* line 41: "if C < S then normalize ..." -- not converged (C = S): A keeps
     * the iteration matrix G = U Sigma' (scaled by 2^s), V is left as is, and
     * sigma holds Sigma' = (e_j, f_j), the norms of G's columns in column order,
     * not backscaled by s and not sorted (R#25).               */
    for (int64_t j = 0; j < n; ++j) {
      if (sigma_e) sigma_e[j] = ce[j];
      if (sigma_f) sigma_f[j] = cf[j];
      if (sigma) sigma[j] = isinf(ce[j]) ? 0.0 : scalbn(cf[j], (int)ce[j]);
    }
    free(ce);
    free(cf);
    free(pairs);
    return ORC_ENOCONV;
  }
  /* finalize: u_j = 2^{-e_j} g_j / f_j, e_j = e_j - s */
  for (int64_t j = 0; j < n; ++j) {
    double *g = A + w * j * lda;
    if (!isinf(ce[j])) {
      int ej = (int)ce[j];
      for (int64_t i = 0; i < w * m; ++i) g[i] = scalbn(g[i], -ej) / cf[j];
      ce[j] = ce[j] - s;
    }
  }
  /* sort sigma non-increasing (R#24): by (e, f) descending, ties by index */
  int64_t *perm = (int64_t *)malloc(sizeof(int64_t) * (size_t)n);
  for (int64_t j = 0; j < n; ++j) perm[j] = j;
  for (int64_t i = 1; i < n; ++i) { /* stable insertion sort */
    int64_t pj = perm[i], k = i - 1;
    while (k >= 0) {
      int64_t pk = perm[k];
      int greater = (ce[pj] > ce[pk]) || (ce[pj] == ce[pk] && cf[pj] > cf[pk]);
      if (!greater) break;
      perm[k + 1] = pk;
      --k;
    }
    perm[k + 1] = pj;
  }
  double *tmpA = (double *)malloc(sizeof(double) * (size_t)(w * m * n));
  double *tmpV = (double *)malloc(sizeof(double) * (size_t)(w * n * n));
  for (int64_t j = 0; j < n; ++j) {
    memcpy(tmpA + w * j * m, A + w * perm[j] * lda, sizeof(double) * (size_t)(w * m));
    memcpy(tmpV + w * j * n, V + w * perm[j] * ldv, sizeof(double) * (size_t)(w * n));
  }
  for (int64_t j = 0; j < n; ++j) {
    memcpy(A + w * j * lda, tmpA + w * j * m, sizeof(double) * (size_t)(w * m));
    memcpy(V + w * j * ldv, tmpV + w * j * n, sizeof(double) * (size_t)(w * n));
    double e = ce[perm[j]], f = cf[perm[j]];
    if (sigma_e) sigma_e[j] = e;
    if (sigma_f) sigma_f[j] = f;
    if (sigma) sigma[j] = isinf(e) ? 0.0 : scalbn(f, (int)fmax(fmin(e, 1e5), -1e5));
  }
  free(tmpA);
  free(tmpV);
  free(perm);
  free(ce);
  free(cf);
  free(pairs);
  return ORC_OK;
}

/* A batch of independent SVDs (configuration 4); OpenMP over matrices. */
int orc_gesvj_batched(int cplx, int64_t batch, int64_t m, int64_t n, double *A, int64_t lda,
                      int64_t strideA, double *V, int64_t ldv, int64_t strideV, double *sigma,
                      int32_t max_sweeps, int32_t *sweeps_done, int32_t *status,
                      int32_t s0_adjust, int32_t *scale_out, const orc_rspec *R)
{
  const int64_t w = cplx ? 2 : 1;
#pragma omp parallel for schedule(static)
  for (int64_t b = 0; b < batch; ++b) {
    int32_t sw = 0, sc = 0;
    int st = orc_gesvj(cplx, m, n, A + w * b * strideA, lda, V + w * b * strideV, ldv,
                       sigma + b * n, NULL, NULL, n, max_sweeps, &sw, NULL, s0_adjust, &sc, R);
    if (sweeps_done) sweeps_done[b] = sw;
    if (status) status[b] = st;
    if (scale_out) scale_out[b] = sc;
  }
  return ORC_OK;
}

int orc_num_threads(void)
{
#ifdef _OPENMP
  return omp_get_max_threads();
#else
  return 1;
#endif
}

/* ======================================================================
 * NEXT-3: the one-pass "(e, f)" Frobenius norm of Alg SM6.3,
 * with s lanes, statement by statement.  Exponents are held as doubles
 * (integral or -inf) exactly as in the paper; every exponent operation is
 * exact.  Readings (R#35-R#38):
 *   R#35  E(x) = getexp = floor(lg|x|) (subnormals exact, E(0) = -inf);
 *         F(x) = getmant in [1,2) with F(0) = 1, so that 0 = (-inf, 1) as the
 *         paper states; scalef(x, y) = x 2^y with one rounding,
 *         scalef(x, -inf) = +-0, scalef(-inf, y) = -inf.
 *   R#36  the lane of element i (0-based) is i mod s; x is zero-padded to a
 *         multiple of s (Eq. pad0; zeros leave a partial sum unchanged);
 *         complex: each iteration takes the real parts, then the imaginary
 *         parts.
 *   R#37  lsb of an exponent: cvtpd_epi64(e) & 1, with -inf -> INT64_MIN ->
 *         0; max(NaN, -inf) = -inf (R#4).
 *   R#38  the final partial sums are sorted by Eq. (vsort) (the sorted
 *         sequence is unique: equal keys are equal pairs), then reduced
 *         pairwise (Eq. redj, SM6.3.2: reduction = 0) or sequentially
 *         (Eq. reds, SM6.3.3: reduction = 1); s a power of two.
 * ====================================================================== */
static double ef_E(double x) { return x == 0.0 ? -INFINITY : (double)ilogb(x); }
static double ef_F(double x)
{
  if (x == 0.0) return 1.0;
  return scalbn(fabs(x), -ilogb(x));
}
static double ef_scalef(double x, double y)
{
  if (isinf(y)) return y < 0 ? copysign(0.0, x) : copysign(INFINITY, x);
  if (isinf(x)) return x;
  double yy = floor(y);
  if (yy > 4000.0) yy = 4000.0; /* saturates: the result is +-inf either way */
  if (yy < -4000.0) yy = -4000.0; /* ... or +-0 */
  return scalbn(x, (int)yy);
}
static double ef_max(double a, double b) { return isnan(a) ? b : (a > b ? a : b); }
static double ef_lsb(double e)
{
  if (isinf(e)) return 0.0; /* cvtpd_epi64(-inf) = INT64_MIN, & 1 = 0 */
  return (double)(((int64_t)e) & 1);
}
/* a <= b by Eq. (vsort) */
static int ef_le(double ea, double fa, double eb, double fb)
{
  return (ea < eb) || (ea == eb && fa <= fb);
}

/* one update r_{i+1} = fma(|x_i|, |x_i|, r_i) of one lane (Alg SM6.3 lines 5-13) */
static void ef_update(double *e, double *f, double x)
{
  const double eh_lsb = ef_lsb(*e);                      /* line 5-6 */
  const double ep = *e - eh_lsb;                         /* e' (even or -inf) */
  const double fp = ef_scalef(*f, eh_lsb);               /* f' */
  const double ei = ef_E(x), fi = ef_F(x);               /* line 8 */
  const double eh = ef_scalef(ei, 1.0);                  /* line 9: 2 e_i */
  const double emax = ef_max(eh, ep);                    /*   e'^(i+1) = e_max */
  const double eh1 = ef_max(eh - emax, -INFINITY);       /* line 10 */
  const double epp = ef_max(ep - emax, -INFINITY);
  const double eh2 = ef_scalef(eh1, -1.0);               /* line 11 */
  const double fh = ef_scalef(fi, eh2);
  const double fhp = ef_scalef(fp, epp);
  const double fpn = fma(fh, fh, fhp);                   /* line 12 */
  *f = ef_F(fpn);
  *e = emax + ef_E(fpn);                                 /* line 13 */
}

/* (a) + (b) for a <= b by Eq. (vsort): Eq. (redj) / (reds), normalised */
static void ef_add_sorted(double ea, double fa, double eb, double fb, double *e, double *f)
{
  const double fpr = fma(ef_scalef(1.0, ef_max(ea - eb, -INFINITY)), fa, fb);
  *f = ef_F(fpr);
  *e = eb + ef_E(fpr);
}

/* ||x||_F of one column (m elements, complex: interleaved) as (e'', f'');
 * e2/f2 (optional) receive (e, f) of ||x||_F^2 */
int orc_norm_ef(int cplx, int64_t m, const double *x, int s, int reduction, double *e_out,
                double *f_out, double *e2, double *f2)
{
  if (s < 1 || s > 4096 || (s & (s - 1)) || m < 0) return ORC_EINVAL;
  double *le = (double *)malloc(sizeof(double) * s), *lf = (double *)malloc(sizeof(double) * s);
  if (!le || !lf) { free(le); free(lf); return ORC_EINVAL; }
  for (int l = 0; l < s; ++l) { le[l] = -INFINITY; lf[l] = 1.0; } /* line 2: r_0 = 0 */
  const int64_t iters = (m + s - 1) / s;
  for (int64_t it = 0; it < iters; ++it) {
    for (int part = 0; part < (cplx ? 2 : 1); ++part) {  /* complex: Re, then Im */
      for (int l = 0; l < s; ++l) {
        const int64_t i = it * s + l;
        const double xi = i < m ? (cplx ? x[2 * i + part] : x[i]) : 0.0; /* Eq. pad0 */
        ef_update(&le[l], &lf[l], xi);
      }
    }
  }
  /* line 15: sort by Eq. (vsort) (insertion sort: any correct sort gives the same sequence) */
  for (int a = 1; a < s; ++a) {
    const double ke = le[a], kf = lf[a];
    int b = a - 1;
    while (b >= 0 && !ef_le(le[b], lf[b], ke, kf)) { le[b + 1] = le[b]; lf[b + 1] = lf[b]; --b; }
    le[b + 1] = ke; lf[b + 1] = kf;
  }
  double e, f;
  if (reduction == 0) { /* lines 16-22: pairwise, Eq. (redj) */
    for (int w = s; w > 1; w /= 2)
      for (int i = 0; i < w / 2; ++i)
        ef_add_sorted(le[2 * i], lf[2 * i], le[2 * i + 1], lf[2 * i + 1], &le[i], &lf[i]);
  } else { /* Eq. (reds): sequential, swapping out-of-order neighbours */
    for (int i = 0; i + 1 < s; ++i) {
      if (!ef_le(le[i], lf[i], le[i + 1], lf[i + 1])) {
        double t = le[i]; le[i] = le[i + 1]; le[i + 1] = t;
        t = lf[i]; lf[i] = lf[i + 1]; lf[i + 1] = t;
      }
      ef_add_sorted(le[i], lf[i], le[i + 1], lf[i + 1], &le[i + 1], &lf[i + 1]);
    }
    le[0] = le[s - 1]; lf[0] = lf[s - 1];
  }
  e = le[0]; f = lf[0];
  free(le); free(lf);
  if (e2) *e2 = e;
  if (f2) *f2 = f;
  /* line 23: the square root, SM6.1 */
  double ep = e, fp = f;
  if (!isinf(e) && fmod(e, 2.0) != 0.0) { fp = 2.0 * f; ep = e - 1.0; }
  *e_out = isinf(ep) ? ep : ep / 2.0;
  *f_out = sqrt(fp);
  return ORC_OK;
}

/* ======================================================================
 * NEXT-4: the real Gram-Schmidt orthogonalization dgsscl of Alg SM8.1 /
 * Eq. (DGS), one pair, statement by statement:
 *   -psi = -(a21' (f_q / f_p))                       (line 1; R#39)
 *   x = scalef(g_p, -e_p); y = scalef(g_q, -e_q)      (line 4)
 *   g_q' = scalef(fma(-psi, x, y), e_q)               (line 5)
 * g_p is unchanged.  (e_j, f_j) = ||g_j|| are inputs (> 0, finite); a pair
 * with a zero column (e = -inf, R#19) is left as it is.
 * ====================================================================== */
void orc_dgsscl(int64_t m, const double *gp, double *gq, double ep, double fp, double eq,
                double fq, double a21)
{
  if (isinf(ep) || isinf(eq)) return; /* a zero column (R#19): nothing to orthogonalise */
  const double mpsi = -(a21 * (fq / fp));
  for (int64_t i = 0; i < m; ++i) {
    const double x = scalbn(gp[i], (int)-ep);
    const double y = scalbn(gq[i], (int)-eq);
    gq[i] = scalbn(fma(mpsi, x, y), (int)eq);
  }
}

/* the number of OpenMP threads the batched oracle entry points use (timing
 * only: results do not depend on it) */
void orc_set_num_threads(int t)
{
#ifdef _OPENMP
  if (t > 0) omp_set_num_threads(t);
#else
  (void)t;
#endif
}
