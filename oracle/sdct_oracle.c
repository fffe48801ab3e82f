/*
 * TEST INFRASTRUCTURE — NOT PRODUCT CODE.
 *
 * Plain-C restatement of the reference CPU algorithm for the hot path
 * (arXiv 2110.01172 three-stage DCT; reference = /root/reference/proj).
 * Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline leg may
 * load this library, and only as the checker — never as the measured or
 * shipped path.  Every function names the reference file:line it restates.
 *
 * Pinning: tests/test_oracle.py checks this restatement against golden
 * vectors produced by the unmodified reference (tests/golden/make_golden.py
 * -> tests/golden/*.npz) and against scipy.fft.dctn.
 *
 * Conventions (reference proj/include/sdct/dct2d.hpp:1-19):
 *   dct_2d  = sum x cos cos (== scipy dctn type 2 / 4)
 *   idct_2d = dctn type 3 / 4, round trip N1 N2 / 4
 *   dct_3d  = dctn / 8,         round trip N1 N2 N3 / 8
 * All arithmetic is fp64, row-major.
 */
#include <complex.h>
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

typedef double complex cd;

static const double kPi = 3.14159265358979323846264338327950288;

/* dct1d.hpp:70-72 */
static size_t parity_embed(size_t m, size_t n) {
  return (m <= (n - 1) / 2) ? 2 * m : 2 * n - 2 * m - 1;
}
/* dct1d.hpp:77-79 */
static size_t parity_source(size_t m, size_t n) {
  return (m % 2 == 0) ? m / 2 : n - (m + 1) / 2;
}

/* dct1d.cpp:41-48: a(k) = e^{-j pi k / (2N)} */
static cd* quarter_wave(size_t n) {
  cd* t = (cd*)malloc(sizeof(cd) * n);
  for (size_t k = 0; k < n; ++k) {
    double ph = -kPi * (double)k / (2.0 * (double)n);
    t[k] = cos(ph) + I * sin(ph);
  }
  return t;
}

/* ---- FFT workspace: rfft.cpp:24-111 (radix-2 DIT + Bluestein) ---------- */
typedef struct {
  size_t n, fft_n;
  size_t* bitrev;
  cd* tw;       /* e^{-j 2 pi k / fft_n}, k < fft_n/2 */
  cd* chirp;    /* Bluestein only */
  cd* chirp_sp;
} fftws;

static int is_pow2(size_t n) { return n && !(n & (n - 1)); }

static void pow2_fft(const fftws* w, cd* d, size_t n, int inverse) { /* rfft.cpp:65-89 */
  for (size_t i = 0; i < n; ++i) {
    size_t j = w->bitrev[i];
    if (i < j) { cd t = d[i]; d[i] = d[j]; d[j] = t; }
  }
  for (size_t len = 2; len <= n; len <<= 1) {
    size_t half = len >> 1, stride = n / len;
    for (size_t s = 0; s < n; s += len)
      for (size_t k = 0; k < half; ++k) {
        cd tw = w->tw[k * stride];
        double wre = creal(tw), wim = inverse ? -cimag(tw) : cimag(tw);
        cd lo = d[s + k], hi = d[s + k + half];
        double vre = creal(hi) * wre - cimag(hi) * wim;
        double vim = creal(hi) * wim + cimag(hi) * wre;
        d[s + k] = (creal(lo) + vre) + I * (cimag(lo) + vim);
        d[s + k + half] = (creal(lo) - vre) + I * (cimag(lo) - vim);
      }
  }
}

static void ws_init(fftws* w, size_t n) { /* rfft.cpp:24-63 */
  memset(w, 0, sizeof(*w));
  w->n = n;
  size_t p = 1;
  while (p < 2 * n - 1) p <<= 1;
  w->fft_n = is_pow2(n) ? n : p;
  size_t fn = w->fft_n, lg = 0;
  while (((size_t)1 << lg) < fn) ++lg;
  w->bitrev = (size_t*)malloc(sizeof(size_t) * fn);
  for (size_t i = 0; i < fn; ++i) {
    size_t r = 0;
    for (size_t b = 0; b < lg; ++b) r |= ((i >> b) & 1u) << (lg - 1 - b);
    w->bitrev[i] = r;
  }
  w->tw = (cd*)malloc(sizeof(cd) * (fn / 2 + 1));
  for (size_t k = 0; k < fn / 2; ++k) {
    double ph = -2.0 * kPi * (double)k / (double)fn;
    w->tw[k] = cos(ph) + I * sin(ph);
  }
  if (!is_pow2(n)) {
    w->chirp = (cd*)malloc(sizeof(cd) * n);
    for (size_t m = 0; m < n; ++m) {
      size_t sq = (m * m) % (2 * n);
      double ph = -kPi * (double)sq / (double)n;
      w->chirp[m] = cos(ph) + I * sin(ph);
    }
    w->chirp_sp = (cd*)calloc(fn, sizeof(cd));
    w->chirp_sp[0] = conj(w->chirp[0]);
    for (size_t m = 1; m < n; ++m) {
      w->chirp_sp[m] = conj(w->chirp[m]);
      w->chirp_sp[fn - m] = conj(w->chirp[m]);
    }
    pow2_fft(w, w->chirp_sp, fn, 0);
  }
}

static void ws_free(fftws* w) {
  free(w->bitrev); free(w->tw); free(w->chirp); free(w->chirp_sp);
}

static void ws_transform(const fftws* w, cd* d, int inverse) { /* rfft.cpp:91-111 */
  size_t n = w->n;
  if (n == 1) return;
  if (!w->chirp) { pow2_fft(w, d, n, inverse); return; }
  if (inverse) {
    for (size_t i = 0; i < n; ++i) d[i] = conj(d[i]);
    ws_transform(w, d, 0);
    for (size_t i = 0; i < n; ++i) d[i] = conj(d[i]);
    return;
  }
  size_t fn = w->fft_n;
  cd* wk = (cd*)calloc(fn, sizeof(cd));
  for (size_t m = 0; m < n; ++m) wk[m] = d[m] * w->chirp[m];
  pow2_fft(w, wk, fn, 0);
  for (size_t m = 0; m < fn; ++m) wk[m] *= w->chirp_sp[m];
  pow2_fft(w, wk, fn, 1);
  double inv = 1.0 / (double)fn;
  for (size_t k = 0; k < n; ++k) d[k] = w->chirp[k] * wk[k] * inv;
  free(wk);
}

/* Strided axis transform over a stored complex tensor: rfft.cpp:152-178 */
static void cfft_axis(cd* data, const size_t* dims, int rank, int axis, const fftws* w,
                      int inverse) {
  size_t n = dims[axis], inner = 1, outer = 1;
  for (int a = axis + 1; a < rank; ++a) inner *= dims[a];
  for (int a = 0; a < axis; ++a) outer *= dims[a];
  if (n == 1) return;
  cd* s = (cd*)malloc(sizeof(cd) * n);
  for (size_t line = 0; line < outer * inner; ++line) {
    size_t o = line / inner, i = line % inner;
    cd* p = data + o * n * inner + i;
    for (size_t k = 0; k < n; ++k) s[k] = p[k * inner];
    ws_transform(w, s, inverse);
    for (size_t k = 0; k < n; ++k) p[k * inner] = s[k];
  }
  free(s);
}

/* rfft_nd: rfft.cpp:182-210. Returns the one-sided spectrum (last axis h). */
static cd* rfft_nd(const double* x, const size_t* dims, int rank) {
  size_t nl = dims[rank - 1], h = nl / 2 + 1, rows = 1;
  for (int a = 0; a < rank - 1; ++a) rows *= dims[a];
  size_t sd[4];
  for (int a = 0; a < rank; ++a) sd[a] = dims[a];
  sd[rank - 1] = h;
  fftws ws[4];
  for (int a = 0; a < rank; ++a) ws_init(&ws[a], dims[a]);
  cd* out = (cd*)malloc(sizeof(cd) * rows * h);
  cd* s = (cd*)malloc(sizeof(cd) * nl);
  for (size_t r = 0; r < rows; ++r) {
    for (size_t k = 0; k < nl; ++k) s[k] = x[r * nl + k];
    ws_transform(&ws[rank - 1], s, 0);
    memcpy(out + r * h, s, sizeof(cd) * h);
  }
  free(s);
  for (int a = rank - 1; a-- > 0;) cfft_axis(out, sd, rank, a, &ws[a], 0);
  for (int a = 0; a < rank; ++a) ws_free(&ws[a]);
  return out;
}

/* irfft_nd: rfft.cpp:212-245 (unnormalised, Hermitian fill of the last axis). */
static double* irfft_nd(const cd* spec, const size_t* dims, int rank) {
  size_t nl = dims[rank - 1], h = nl / 2 + 1, rows = 1;
  for (int a = 0; a < rank - 1; ++a) rows *= dims[a];
  size_t sd[4];
  for (int a = 0; a < rank; ++a) sd[a] = dims[a];
  sd[rank - 1] = h;
  fftws ws[4];
  for (int a = 0; a < rank; ++a) ws_init(&ws[a], dims[a]);
  cd* work = (cd*)malloc(sizeof(cd) * rows * h);
  memcpy(work, spec, sizeof(cd) * rows * h);
  for (int a = rank - 1; a-- > 0;) cfft_axis(work, sd, rank, a, &ws[a], 1);
  double* out = (double*)malloc(sizeof(double) * rows * nl);
  cd* s = (cd*)malloc(sizeof(cd) * nl);
  for (size_t r = 0; r < rows; ++r) {
    for (size_t k = 0; k < h; ++k) s[k] = work[r * h + k];
    for (size_t k = h; k < nl; ++k) s[k] = conj(work[r * h + (nl - k)]);
    ws_transform(&ws[rank - 1], s, 1);
    for (size_t k = 0; k < nl; ++k) out[r * nl + k] = creal(s[k]);
  }
  free(s);
  free(work);
  for (int a = 0; a < rank; ++a) ws_free(&ws[a]);
  return out;
}

/* ---- 2D: dct2d.cpp ------------------------------------------------------ */

/* dct_2d (dct2d.cpp:367-387, Direct orientation): parity gather (48-70),
 * rfft_nd, merged postprocess (82-115). */
void sdct_oracle_dct_2d(const double* x, size_t n1, size_t n2, double* y) {
  double* xr = (double*)malloc(sizeof(double) * n1 * n2);
  for (size_t i = 0; i < n1; ++i)
    for (size_t j = 0; j < n2; ++j)
      xr[i * n2 + j] = x[parity_embed(i, n1) * n2 + parity_embed(j, n2)];
  size_t dims[2] = {n1, n2};
  cd* sp = rfft_nd(xr, dims, 2);
  size_t h2 = n2 / 2 + 1;
  cd* ta = quarter_wave(n1);
  cd* tb = quarter_wave(n2);
  for (size_t q1 = 0; q1 <= n1 / 2; ++q1)
    for (size_t q2 = 0; q2 < h2; ++q2) {
      size_t r1 = (n1 - q1) % n1, r2 = (n2 - q2) % n2;
      int deg1 = r1 == q1, deg2 = r2 == q2;
      cd a = ta[q1], b = tb[q2];
      cd x1 = sp[q1 * h2 + q2];
      cd x2 = deg1 ? x1 : sp[r1 * h2 + q2];
      cd ax1 = a * x1, ax2 = conj(a) * x2;
      cd s = b * (ax1 + ax2);
      y[q1 * n2 + q2] = 0.5 * creal(s);
      if (!deg2) y[q1 * n2 + r2] = -0.5 * cimag(s);
      if (!deg1) {
        cd t = b * (ax1 - ax2);
        y[r1 * n2 + q2] = -0.5 * cimag(t);
        if (!deg2) y[r1 * n2 + r2] = -0.5 * creal(t);
      }
    }
  free(xr); free(sp); free(ta); free(tb);
}

/* idct_family_2d (dct2d.cpp:410-437): merged inverse preprocess (161-198),
 * irfft_nd, inverse parity gather with 1/4 and optional sign (214-238).
 * mode: 0 = IDCT, 1 = reverse axis 0 (idxst_idct), 2 = reverse axis 1
 * (idct_idxst) — transforms_ext.cpp:269-279. */
void sdct_oracle_idct_family_2d(const double* x, size_t n1, size_t n2, int mode, double* y) {
  size_t h2 = n2 / 2 + 1;
  cd* ta = quarter_wave(n1);
  cd* tb = quarter_wave(n2);
  cd* sp = (cd*)calloc(n1 * h2, sizeof(cd));
#define FETCH(ii, jj, out)                                        \
  do {                                                            \
    size_t i_ = (ii), j_ = (jj);                                  \
    (out) = 0.0;                                                  \
    if (i_ != n1 && j_ != n2) {                                   \
      int ok = 1;                                                 \
      if (mode == 1) { if (i_ == 0) ok = 0; else i_ = n1 - i_; }  \
      if (mode == 2) { if (j_ == 0) ok = 0; else j_ = n2 - j_; }  \
      if (ok) (out) = x[i_ * n2 + j_];                            \
    }                                                             \
  } while (0)
  for (size_t q1 = 0; q1 <= n1 / 2; ++q1)
    for (size_t m2 = 0; m2 < h2; ++m2) {
      double p, q, r, s;
      FETCH(q1, m2, p);
      FETCH(n1 - q1, n2 - m2, q);
      FETCH(n1 - q1, m2, r);
      FETCH(q1, n2 - m2, s);
      cd wb = conj(tb[m2]);
      cd w1b = conj(ta[q1]) * wb;
      sp[q1 * h2 + m2] = w1b * ((p - q) - I * (r + s));
      size_t r1 = (n1 - q1) % n1;
      if (r1 != q1) {
        cd w2b = conj(ta[r1]) * wb;
        sp[r1 * h2 + m2] = w2b * ((r - s) - I * (p + q));
      }
    }
#undef FETCH
  size_t dims[2] = {n1, n2};
  double* z = irfft_nd(sp, dims, 2);
  int sign_axis = mode == 1 ? 0 : mode == 2 ? 1 : -1;
  for (size_t k1 = 0; k1 < n1; ++k1)
    for (size_t k2 = 0; k2 < n2; ++k2) {
      double v = 0.25 * z[parity_source(k1, n1) * n2 + parity_source(k2, n2)];
      if (sign_axis == 0 && (k1 & 1u)) v = -v;
      if (sign_axis == 1 && (k2 & 1u)) v = -v;
      y[k1 * n2 + k2] = v;
    }
  free(sp); free(z); free(ta); free(tb);
}

/* ---- 3D: transforms_ext.cpp -------------------------------------------- */

/* dct_3d (transforms_ext.cpp:322-350): parity_pass3 (165-183), rfft_nd,
 * fused_post3 (99-161). */
void sdct_oracle_dct_3d(const double* x, size_t n1, size_t n2, size_t n3, double* y) {
  size_t N = n1 * n2 * n3;
  double* xr = (double*)malloc(sizeof(double) * N);
  for (size_t i = 0; i < n1; ++i)
    for (size_t j = 0; j < n2; ++j)
      for (size_t k = 0; k < n3; ++k)
        xr[(i * n2 + j) * n3 + k] =
            x[(parity_embed(i, n1) * n2 + parity_embed(j, n2)) * n3 + parity_embed(k, n3)];
  size_t dims[3] = {n1, n2, n3};
  cd* sp = rfft_nd(xr, dims, 3);
  size_t h3 = n3 / 2 + 1;
  cd* ta = quarter_wave(n1);
  cd* tb = quarter_wave(n2);
  cd* tc = quarter_wave(n3);
#define PUT(i, j, k, v) y[((i) * n2 + (j)) * n3 + (k)] = (v)
  for (size_t q1 = 0; q1 <= n1 / 2; ++q1)
    for (size_t q2 = 0; q2 <= n2 / 2; ++q2)
      for (size_t q3 = 0; q3 < h3; ++q3) {
        size_t m1 = (n1 - q1) % n1, m2 = (n2 - q2) % n2, m3 = (n3 - q3) % n3;
        int deg1 = m1 == q1, deg2 = m2 == q2, deg3 = m3 == q3;
        cd f1 = sp[(q1 * n2 + q2) * h3 + q3];
        cd f2 = deg1 ? f1 : sp[(m1 * n2 + q2) * h3 + q3];
        cd f3 = deg2 ? f1 : sp[(q1 * n2 + m2) * h3 + q3];
        cd f4 = deg1 ? f3 : (deg2 ? f2 : sp[(m1 * n2 + m2) * h3 + q3]);
        cd a = ta[q1], b = tb[q2], c = tc[q3];
        cd ab = a * b, cb = conj(a) * b;
        cd t1 = ab * f1, t2 = cb * f2, t3 = conj(cb) * f3, t4 = conj(ab) * f4;
        cd s12 = t1 + t2, s34 = t3 + t4;
        cd u00 = c * (s12 + s34);
        PUT(q1, q2, q3, 0.25 * creal(u00));
        if (!deg3) PUT(q1, q2, m3, -0.25 * cimag(u00));
        if (!deg2) {
          cd u01 = c * (s12 - s34);
          PUT(q1, m2, q3, -0.25 * cimag(u01));
          if (!deg3) PUT(q1, m2, m3, -0.25 * creal(u01));
        }
        if (!deg1) {
          cd d12 = t1 - t2, d34 = t3 - t4;
          cd u10 = c * (d12 + d34);
          PUT(m1, q2, q3, -0.25 * cimag(u10));
          if (!deg3) PUT(m1, q2, m3, -0.25 * creal(u10));
          if (!deg2) {
            cd u11 = c * (d12 - d34);
            PUT(m1, m2, q3, -0.25 * creal(u11));
            if (!deg3) PUT(m1, m2, m3, 0.25 * cimag(u11));
          }
        }
      }
#undef PUT
  free(xr); free(sp); free(ta); free(tb); free(tc);
}

/* idct_3d (transforms_ext.cpp:359-387): idct_pre3 (187-216), irfft_nd,
 * inverse parity_pass3 with 1/8. */
void sdct_oracle_idct_3d(const double* x, size_t n1, size_t n2, size_t n3, double* y) {
  size_t h3 = n3 / 2 + 1;
  cd* ta = quarter_wave(n1);
  cd* tb = quarter_wave(n2);
  cd* tc = quarter_wave(n3);
  cd* sp = (cd*)malloc(sizeof(cd) * n1 * n2 * h3);
#define F(i, j, k) (((i) == n1 || (j) == n2 || (k) == n3) ? 0.0 : x[((i) * n2 + (j)) * n3 + (k)])
  for (size_t i = 0; i < n1; ++i)
    for (size_t j = 0; j < n2; ++j)
      for (size_t k = 0; k < h3; ++k) {
        size_t r1 = n1 - i, r2 = n2 - j, r3 = n3 - k;
        double re = (F(i, j, k) - F(r1, r2, k)) - (F(r1, j, r3) + F(i, r2, r3));
        double im = F(r1, r2, r3) - ((F(r1, j, k) + F(i, r2, k)) + F(i, j, r3));
        cd w = (conj(ta[i]) * conj(tb[j])) * conj(tc[k]);
        sp[(i * n2 + j) * h3 + k] = w * (re + I * im);
      }
#undef F
  size_t dims[3] = {n1, n2, n3};
  double* z = irfft_nd(sp, dims, 3);
  for (size_t i = 0; i < n1; ++i)
    for (size_t j = 0; j < n2; ++j)
      for (size_t k = 0; k < n3; ++k)
        y[(i * n2 + j) * n3 + k] =
            0.125 *
            z[(parity_source(i, n1) * n2 + parity_source(j, n2)) * n3 + parity_source(k, n3)];
  free(sp); free(z); free(ta); free(tb); free(tc);
}

/* ---- direct-sum oracles: oracle.cpp:37-106 (plain sums; Kahan omitted) -- */

void sdct_oracle_dct_direct_1d(const double* x, size_t n, double* y) {
  for (size_t k = 0; k < n; ++k) {
    double acc = 0.0, c = 0.0;
    for (size_t m = 0; m < n; ++m) {
      double v = x[m] * cos(kPi / (double)n * ((double)m + 0.5) * (double)k);
      double t = acc + (v - c);
      c = (t - acc) - (v - c);
      acc = t;
    }
    y[k] = acc;
  }
}

void sdct_oracle_idct_direct_1d(const double* x, size_t n, double* y) {
  for (size_t k = 0; k < n; ++k) {
    double acc = 0.5 * x[0], c = 0.0;
    for (size_t m = 1; m < n; ++m) {
      double v = x[m] * cos(kPi / (double)n * (double)m * ((double)k + 0.5));
      double t = acc + (v - c);
      c = (t - acc) - (v - c);
      acc = t;
    }
    y[k] = acc;
  }
}

void sdct_oracle_idxst_direct_1d(const double* x, size_t n, double* y) {
  double* sh = (double*)malloc(sizeof(double) * n);
  sh[0] = 0.0;
  for (size_t m = 1; m < n; ++m) sh[m] = x[n - m];
  sdct_oracle_idct_direct_1d(sh, n, y);
  for (size_t k = 1; k < n; k += 2) y[k] = -y[k];
  free(sh);
}

void sdct_oracle_dct_direct_2d(const double* x, size_t n1, size_t n2, double* y) {
  for (size_t k1 = 0; k1 < n1; ++k1)
    for (size_t k2 = 0; k2 < n2; ++k2) {
      double acc = 0.0, c = 0.0;
      for (size_t m1 = 0; m1 < n1; ++m1) {
        double c1 = cos(kPi / (double)n1 * ((double)m1 + 0.5) * (double)k1);
        for (size_t m2 = 0; m2 < n2; ++m2) {
          double c2 = cos(kPi / (double)n2 * ((double)m2 + 0.5) * (double)k2);
          double v = x[m1 * n2 + m2] * c1 * c2;
          double t = acc + (v - c);
          c = (t - acc) - (v - c);
          acc = t;
        }
      }
      y[k1 * n2 + k2] = acc;
    }
}

/* force_demo_fields (proj/src/force.cpp:11-37): a = dct_2d(density);
 * a1 = a w1/(w1^2+w2^2), a2 = a w2/(w1^2+w2^2), w_d = pi k_d / n_d, DC -> 0
 * (force.cpp:22-31); xi1 = idct_idxst_2d(a1), xi2 = idxst_idct_2d(a2)
 * (force.cpp:34-35). */
void sdct_oracle_force_fields_2d(const double* x, size_t n1, size_t n2, double* xi1, double* xi2) {
  const double pi = 3.14159265358979323846;
  double* a = (double*)malloc(n1 * n2 * sizeof(double));
  double* a1 = (double*)malloc(n1 * n2 * sizeof(double));
  double* a2 = (double*)malloc(n1 * n2 * sizeof(double));
  sdct_oracle_dct_2d(x, n1, n2, a);
  for (size_t k1 = 0; k1 < n1; ++k1) {
    const double w1 = pi * (double)k1 / (double)n1;
    for (size_t k2 = 0; k2 < n2; ++k2) {
      const double w2 = pi * (double)k2 / (double)n2;
      const double den = w1 * w1 + w2 * w2;
      const double v = a[k1 * n2 + k2];
      a1[k1 * n2 + k2] = den > 0.0 ? v * w1 / den : 0.0;
      a2[k1 * n2 + k2] = den > 0.0 ? v * w2 / den : 0.0;
    }
  }
  sdct_oracle_idct_family_2d(a1, n1, n2, 2, xi1);
  sdct_oracle_idct_family_2d(a2, n1, n2, 1, xi2);
  free(a);
  free(a1);
  free(a2);
}

/* ---- row-column baselines ------------------------------------------------
 * dct_rows (dct2d.cpp:248-290): per row, parity reorder, rfft_row, then
 * y(k) = Re(tw(k) X(k)) with X(k) = conj X(n-k) past the stored half.
 * inverse_rows (transforms_ext.cpp:40-88): v(k) = (x(k), -x(n-k)) [cosine] or
 * (x(n-k), -x(k)) [sine, 0 at k = 0] times conj tw(k), irfft_row, then
 * y(m) = 1/2 t(ps(m)), odd m negated for the sine embedding. */
static void rows_pass(const double* x, size_t rows, size_t n, int inverse, int sine, double* y) {
  size_t h = n / 2 + 1;
  cd* tw = quarter_wave(n);
  fftws w;
  ws_init(&w, n);
  cd* s = (cd*)malloc(sizeof(cd) * n);
  for (size_t r = 0; r < rows; ++r) {
    const double* xr = x + r * n;
    double* yr = y + r * n;
    if (!inverse) {
      for (size_t m = 0; m < n; ++m) s[m] = xr[parity_embed(m, n)];
      ws_transform(&w, s, 0);
      for (size_t k = 0; k < n; ++k) {
        cd v = k < h ? s[k] : conj(s[n - k]);
        yr[k] = creal(tw[k]) * creal(v) - cimag(tw[k]) * cimag(v);
      }
    } else {
      for (size_t k = 0; k < h; ++k) {
        cd v;
        if (sine) v = (k == 0) ? 0.0 : xr[n - k] - I * xr[k];
        else v = xr[k] - I * (k == 0 ? 0.0 : xr[n - k]);
        s[k] = conj(tw[k]) * v;
      }
      for (size_t k = h; k < n; ++k) s[k] = conj(s[n - k]);
      ws_transform(&w, s, 1);
      for (size_t m = 0; m < n; ++m) {
        double v = 0.5 * creal(s[parity_source(m, n)]);
        yr[m] = (sine && (m & 1u)) ? -v : v;
      }
    }
  }
  free(s);
  ws_free(&w);
  free(tw);
}

static void transpose_2d(const double* x, size_t r, size_t c, double* y) {
  for (size_t i = 0; i < r; ++i)
    for (size_t j = 0; j < c; ++j) y[j * r + i] = x[i * c + j];
}

/* dct_2d_rowcol (dct2d.cpp:395-406) for kind 0; composite_2d_rowcol
 * (transforms_ext.cpp:287-301) for kind 1 (IdctIdxst: sine along axis 1) and
 * kind 2 (IdxstIdct: sine along axis 0). */
void sdct_oracle_rowcol_2d(const double* x, size_t n1, size_t n2, int kind, double* y) {
  double* a = (double*)malloc(sizeof(double) * n1 * n2);
  double* b = (double*)malloc(sizeof(double) * n1 * n2);
  int inv = kind != 0;
  rows_pass(x, n1, n2, inv, kind == 1, a);
  transpose_2d(a, n1, n2, b);
  rows_pass(b, n2, n1, inv, kind == 2, a);
  transpose_2d(a, n2, n1, y);
  free(a);
  free(b);
}
