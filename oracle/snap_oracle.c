/*
 * snap_oracle.c -- CPU restatement of the reference SNAP force path.
 *
 * TEST INFRASTRUCTURE ONLY (see snap_oracle.h).  Every function below cites
 * the reference file:line it restates; paths are relative to
 * /root/reference/proj/include/snapforge/.  Floating-point expressions keep
 * the reference's operation order so that, compiled with the same flags
 * (-O2 -ffp-contract=off), results are bitwise identical to the reference.
 */
#include "snap_oracle.h"

#include <math.h>
#include <stdarg.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

typedef struct {
  double re, im;
} cplx;

static char g_err[512];

static int fail(const char* fmt, ...) {
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(g_err, sizeof g_err, fmt, ap);
  va_end(ap);
  return -1;
}

const char* orc_last_error(void) { return g_err; }

static const double kPi = 3.14159265358979323846; /* angular_basis.hpp:32 */

/* ------------------------------------------------------------------------ */
/* Rng: std::mt19937_64 with pinned mappings (rng.hpp:19-56)                */
/* ------------------------------------------------------------------------ */
typedef struct {
  uint64_t mt[312];
  int mti;
} rng_t;

static void rng_seed(rng_t* r, uint64_t seed) {
  r->mt[0] = seed;
  for (int i = 1; i < 312; ++i)
    r->mt[i] = 6364136223846793005ULL * (r->mt[i - 1] ^ (r->mt[i - 1] >> 62)) +
               (uint64_t)i;
  r->mti = 312;
}

static uint64_t rng_next(rng_t* r) {
  static const uint64_t UM = 0xFFFFFFFF80000000ULL, LM = 0x7FFFFFFFULL;
  if (r->mti >= 312) {
    for (int i = 0; i < 312; ++i) {
      uint64_t x = (r->mt[i] & UM) | (r->mt[(i + 1) % 312] & LM);
      uint64_t xa = x >> 1;
      if (x & 1ULL) xa ^= 0xB5026F5AA96619E9ULL;
      r->mt[i] = r->mt[(i + 156) % 312] ^ xa;
    }
    r->mti = 0;
  }
  uint64_t y = r->mt[r->mti++];
  y ^= (y >> 29) & 0x5555555555555555ULL;
  y ^= (y << 17) & 0x71D67FFFEDA60000ULL;
  y ^= (y << 37) & 0xFFF7EEE000000000ULL;
  y ^= y >> 43;
  return y;
}

/* rng.hpp:24-26 */
static double rng_uniform01(rng_t* r) {
  return (double)(rng_next(r) >> 11) * 0x1.0p-53;
}
/* rng.hpp:29 */
static double rng_uniform(rng_t* r, double lo, double hi) {
  return lo + (hi - lo) * rng_uniform01(r);
}
/* rng.hpp:37-49 */
static void rng_unit_vector(rng_t* r, double out[3]) {
  for (;;) {
    double u = rng_uniform(r, -1.0, 1.0);
    double v = rng_uniform(r, -1.0, 1.0);
    double s = u * u + v * v;
    if (s >= 1.0 || s == 0.0) continue;
    double f = 2.0 * sqrt(1.0 - s);
    out[0] = u * f;
    out[1] = v * f;
    out[2] = 1.0 - 2.0 * s;
    return;
  }
}

void orc_rng_stream(uint64_t seed, int n, double* out) {
  rng_t r;
  rng_seed(&r, seed);
  for (int i = 0; i < n; ++i) out[i] = rng_uniform01(&r);
}

/* ------------------------------------------------------------------------ */
/* Index bookkeeping (halfint_index.hpp)                                    */
/* ------------------------------------------------------------------------ */
static int full_block(int t) { return (t + 1) * (t + 1); } /* :93 */
static int half_block(int t) { return (t / 2 + 1) * (t + 1); } /* :96 */

int orc_u_full_total(int T) { /* :143-147 */
  int n = 0;
  for (int t = 0; t <= T; ++t) n += full_block(t);
  return n;
}
int orc_u_half_total(int T) { /* :149-153 */
  int n = 0;
  for (int t = 0; t <= T; ++t) n += half_block(t);
  return n;
}

/* enumerate_bispectrum_triples :132-141 */
int orc_triples(int T, int* out) {
  int n = 0;
  for (int j1 = 0; j1 <= T; ++j1)
    for (int j2 = 0; j2 <= j1; ++j2)
      for (int j = j1 - j2; j <= (j1 + j2 < T ? j1 + j2 : T); j += 2)
        if (j >= j1) {
          if (out) {
            out[3 * n] = j1;
            out[3 * n + 1] = j2;
            out[3 * n + 2] = j;
          }
          ++n;
        }
  return n;
}
int orc_n_triples(int T) { return orc_triples(T, NULL); }

/* coupling tuples, HalfIntIndexMaps::build :184-198 */
int orc_tuples(int T, int* out) {
  int n = 0, elem = 0, cgo = 0;
  for (int j1 = 0; j1 <= T; ++j1)
    for (int j2 = 0; j2 <= j1; ++j2)
      for (int j = j1 - j2; j <= (j1 + j2 < T ? j1 + j2 : T); j += 2) {
        if (out) {
          out[5 * n] = j1;
          out[5 * n + 1] = j2;
          out[5 * n + 2] = j;
          out[5 * n + 3] = elem;
          out[5 * n + 4] = cgo;
        }
        ++n;
        elem += half_block(j);
        cgo += (j1 + 1) * (j2 + 1);
      }
  return n;
}
int orc_n_tuples(int T) { return orc_tuples(T, NULL); }

int orc_z_total_elements(int T) {
  int n = 0;
  for (int j1 = 0; j1 <= T; ++j1)
    for (int j2 = 0; j2 <= j1; ++j2)
      for (int j = j1 - j2; j <= (j1 + j2 < T ? j1 + j2 : T); j += 2)
        n += half_block(j);
  return n;
}
int orc_cg_total(int T) {
  int n = 0;
  for (int j1 = 0; j1 <= T; ++j1)
    for (int j2 = 0; j2 <= j1; ++j2)
      for (int j = j1 - j2; j <= (j1 + j2 < T ? j1 + j2 : T); j += 2)
        n += (j1 + 1) * (j2 + 1);
  return n;
}

/* z_loop_bounds :262-276 ; out = ma1min, ma2max, na, mb1min, mb2max, nb */
void orc_z_loop_bounds(int j1, int j2, int j, int mb, int ma, int out[6]) {
  int t = 2 * ma - j;
  int ma1min = t + j1 - j2 < 0 ? 0 : (t + j1 - j2) / 2;
  int ma2max = (t - (2 * ma1min - j1) + j2) / 2;
  int hi = (t + j2 + j1) / 2;
  int na = (j1 < hi ? j1 : hi) - ma1min + 1;
  t = 2 * mb - j;
  int mb1min = t + j1 - j2 < 0 ? 0 : (t + j1 - j2) / 2;
  int mb2max = (t - (2 * mb1min - j1) + j2) / 2;
  hi = (t + j2 + j1) / 2;
  int nb = (j1 < hi ? j1 : hi) - mb1min + 1;
  out[0] = ma1min;
  out[1] = ma2max;
  out[2] = na;
  out[3] = mb1min;
  out[4] = mb2max;
  out[5] = nb;
}

/* Dense (j1,j2,j) lookups, HalfIntIndexMaps :104-123 */
typedef struct {
  int T;
  int nhalf, nfull, ntrip, ntup, cgtot;
  int* half_off; /* T+2 */
  int* full_off; /* T+2 */
  int* triples;  /* 3*ntrip */
  int* tuples;   /* 5*ntup */
  int* triple_flat;
  int* cg_flat;
} maps_t;

static int dense(const maps_t* m, int a, int b, int c) {
  return (a * (m->T + 1) + b) * (m->T + 1) + c;
}

static void maps_free(maps_t* m) {
  free(m->half_off);
  free(m->full_off);
  free(m->triples);
  free(m->tuples);
  free(m->triple_flat);
  free(m->cg_flat);
}

static void maps_build(maps_t* m, int T) { /* HalfIntIndexMaps::build :155-200 */
  m->T = T;
  m->half_off = (int*)calloc((size_t)T + 2, sizeof(int));
  m->full_off = (int*)calloc((size_t)T + 2, sizeof(int));
  for (int t = 0; t <= T; ++t) {
    m->full_off[t + 1] = m->full_off[t] + full_block(t);
    m->half_off[t + 1] = m->half_off[t] + half_block(t);
  }
  m->nhalf = m->half_off[T + 1];
  m->nfull = m->full_off[T + 1];
  m->ntrip = orc_triples(T, NULL);
  m->triples = (int*)malloc(sizeof(int) * 3 * (size_t)(m->ntrip + 1));
  orc_triples(T, m->triples);
  m->ntup = orc_tuples(T, NULL);
  m->tuples = (int*)malloc(sizeof(int) * 5 * (size_t)(m->ntup + 1));
  orc_tuples(T, m->tuples);
  m->cgtot = orc_cg_total(T);
  size_t nd = (size_t)(T + 1) * (T + 1) * (T + 1);
  m->triple_flat = (int*)malloc(sizeof(int) * nd);
  m->cg_flat = (int*)malloc(sizeof(int) * nd);
  for (size_t i = 0; i < nd; ++i) m->triple_flat[i] = m->cg_flat[i] = -1;
  for (int l = 0; l < m->ntrip; ++l)
    m->triple_flat[dense(m, m->triples[3 * l], m->triples[3 * l + 1],
                         m->triples[3 * l + 2])] = l;
  for (int t = 0; t < m->ntup; ++t)
    m->cg_flat[dense(m, m->tuples[5 * t], m->tuples[5 * t + 1],
                     m->tuples[5 * t + 2])] = m->tuples[5 * t + 4];
}

/* ------------------------------------------------------------------------ */
/* Coupling coefficients (angular_basis.hpp)                                */
/* ------------------------------------------------------------------------ */
static double factorial(int n) { /* :38-47 */
  static double table[65];
  static int init = 0;
  if (!init) {
    table[0] = 1.0;
    for (int i = 1; i <= 64; ++i) table[i] = table[i - 1] * i;
    init = 1;
  }
  return table[n];
}

static double rootpq(int p, int q) { /* :52-63 */
  return sqrt((double)p / (double)q);
}

static double deltacg(int j1, int j2, int j) { /* :66-70 */
  double sfaccg = factorial((j1 + j2 + j) / 2 + 1);
  return sqrt(factorial((j1 + j2 - j) / 2) * factorial((j1 - j2 + j) / 2) *
              factorial((-j1 + j2 + j) / 2) / sfaccg);
}

static int imax(int a, int b) { return a > b ? a : b; }
static int imin(int a, int b) { return a < b ? a : b; }

int orc_cg_table(int T, double* out) { /* compute_cg_table :151-196 */
  int ntup = orc_tuples(T, NULL);
  int* tup = (int*)malloc(sizeof(int) * 5 * (size_t)ntup);
  orc_tuples(T, tup);
  int total = orc_cg_total(T);
  for (int i = 0; i < total; ++i) out[i] = 0.0;
  for (int q = 0; q < ntup; ++q) {
    const int j1 = tup[5 * q], j2 = tup[5 * q + 1], j = tup[5 * q + 2];
    int idx = tup[5 * q + 4];
    for (int m1 = 0; m1 <= j1; ++m1) {
      const int aa2 = 2 * m1 - j1;
      for (int m2 = 0; m2 <= j2; ++m2, ++idx) {
        const int bb2 = 2 * m2 - j2;
        const int m = (aa2 + bb2 + j) / 2;
        if (m < 0 || m > j) continue;
        double sum = 0.0;
        const int zlo = imax(0, imax(-(j - j2 + aa2) / 2, -(j - j1 - bb2) / 2));
        const int zhi =
            imin((j1 + j2 - j) / 2, imin((j1 - aa2) / 2, (j2 + bb2) / 2));
        for (int zz = zlo; zz <= zhi; ++zz) {
          const double ifac = (zz % 2) ? -1.0 : 1.0;
          sum += ifac / (factorial(zz) * factorial((j1 + j2 - j) / 2 - zz) *
                         factorial((j1 - aa2) / 2 - zz) *
                         factorial((j2 + bb2) / 2 - zz) *
                         factorial((j - j2 + aa2) / 2 + zz) *
                         factorial((j - j1 - bb2) / 2 + zz));
        }
        const int cc2 = 2 * m - j;
        double norm = sqrt(factorial((j1 + aa2) / 2) * factorial((j1 - aa2) / 2) *
                           factorial((j2 + bb2) / 2) * factorial((j2 - bb2) / 2) *
                           factorial((j + cc2) / 2) * factorial((j - cc2) / 2) *
                           (j + 1));
        out[idx] = sum * deltacg(j1, j2, j) * norm;
      }
    }
  }
  free(tup);
  return 0;
}

/* ------------------------------------------------------------------------ */
/* Radial switching and 3-sphere map (angular_basis.hpp:78-139)              */
/* ------------------------------------------------------------------------ */
static void switching_function(double r, double rcut, double rmin0, double* fc,
                               double* dfc) { /* :78-87 */
  if (r <= rmin0) {
    *fc = 1.0;
    *dfc = 0.0;
    return;
  }
  if (r >= rcut) {
    *fc = 0.0;
    *dfc = 0.0;
    return;
  }
  const double scale = kPi / (rcut - rmin0);
  *fc = 0.5 * (cos((r - rmin0) * scale) + 1.0);
  *dfc = -0.5 * sin((r - rmin0) * scale) * scale;
}

typedef struct {
  double r, theta0, z0;
  double rhat[3];
  cplx a, b, da[3], db[3];
} sphere_map;

static int map_to_3sphere(const double disp[3], double rcut, double rmin0,
                          double rfac0, sphere_map* m) { /* :102-139 */
  if (!(rcut > rmin0)) return fail("map_to_3sphere: Rcut must exceed rmin0");
  const double x = disp[0], y = disp[1], z = disp[2];
  const double rsq = x * x + y * y + z * z;
  if (!(rsq > 0.0)) return fail("map_to_3sphere: zero-length displacement");
  const double r = sqrt(rsq);
  if (!(r < rcut)) return fail("map_to_3sphere: displacement at or beyond Rcut");
  m->r = r;
  const double rscale0 = rfac0 * kPi / (rcut - rmin0);
  m->theta0 = (r - rmin0) * rscale0;
  m->z0 = r / tan(m->theta0);
  const double r0inv = 1.0 / sqrt(rsq + m->z0 * m->z0);
  m->a.re = r0inv * m->z0;
  m->a.im = -r0inv * z;
  m->b.re = r0inv * y;
  m->b.im = -r0inv * x;
  const double dz0dr = m->z0 / r - (r * rscale0) * (rsq + m->z0 * m->z0) / rsq;
  const double dr0invdr = -r0inv * r0inv * r0inv * (r + m->z0 * dz0dr);
  m->rhat[0] = x / r;
  m->rhat[1] = y / r;
  m->rhat[2] = z / r;
  for (int k = 0; k < 3; ++k) {
    const double dr0inv = dr0invdr * m->rhat[k];
    m->da[k].re = dz0dr * m->rhat[k] * r0inv + m->z0 * dr0inv;
    m->da[k].im = -z * dr0inv;
    m->db[k].re = y * dr0inv;
    m->db[k].im = -x * dr0inv;
  }
  m->da[2].im += -r0inv;
  m->db[0].im += -r0inv;
  m->db[1].re += r0inv;
  return 0;
}

int orc_map_to_3sphere(const double disp[3], double rcut, double rmin0,
                       double rfac0, double* out) {
  sphere_map m;
  if (map_to_3sphere(disp, rcut, rmin0, rfac0, &m)) return -1;
  out[0] = m.r;
  out[1] = m.a.re;
  out[2] = m.a.im;
  out[3] = m.b.re;
  out[4] = m.b.im;
  for (int k = 0; k < 3; ++k) {
    out[5 + 2 * k] = m.da[k].re;
    out[6 + 2 * k] = m.da[k].im;
    out[11 + 2 * k] = m.db[k].re;
    out[12 + 2 * k] = m.db[k].im;
    out[16 + k] = m.rhat[k];
  }
  return 0;
}

/* ------------------------------------------------------------------------ */
/* Level recursions (angular_basis.hpp:232-329)                              */
/* ------------------------------------------------------------------------ */
static void wigner_u_level_half(cplx a, cplx b, int t, const cplx* prev,
                                cplx* cur) { /* :232-257 */
  const int cols = t + 1;
  const int cols_prev = t;
  for (int mb = 0; 2 * mb <= t; ++mb) {
    cplx* row = cur + mb * cols;
    row[0].re = 0.0;
    row[0].im = 0.0;
    const int mirror_prev = 2 * mb > t - 1;
    for (int ma = 0; ma < t; ++ma) {
      cplx up;
      if (!mirror_prev) {
        up = prev[mb * cols_prev + ma];
      } else {
        cplx s = prev[(t - 1 - mb) * cols_prev + (t - 1 - ma)];
        const double sign = ((ma + mb) & 1) ? -1.0 : 1.0;
        up.re = sign * s.re;
        up.im = -sign * s.im;
      }
      double rp = rootpq(t - ma, t - mb);
      row[ma].re += rp * (a.re * up.re + a.im * up.im);
      row[ma].im += rp * (a.re * up.im - a.im * up.re);
      rp = rootpq(ma + 1, t - mb);
      row[ma + 1].re = -rp * (b.re * up.re + b.im * up.im);
      row[ma + 1].im = -rp * (b.re * up.im - b.im * up.re);
    }
  }
}

static void wigner_du_level_half(cplx a, cplx b, cplx da, cplx db, int t,
                                 const cplx* uprev, const cplx* duprev,
                                 cplx* ducur) { /* :262-296 */
  const int cols = t + 1;
  const int cols_prev = t;
  for (int mb = 0; 2 * mb <= t; ++mb) {
    cplx* row = ducur + mb * cols;
    row[0].re = 0.0;
    row[0].im = 0.0;
    const int mirror_prev = 2 * mb > t - 1;
    for (int ma = 0; ma < t; ++ma) {
      cplx up, dup;
      if (!mirror_prev) {
        up = uprev[mb * cols_prev + ma];
        dup = duprev[mb * cols_prev + ma];
      } else {
        const int src = (t - 1 - mb) * cols_prev + (t - 1 - ma);
        const double sign = ((ma + mb) & 1) ? -1.0 : 1.0;
        cplx su = uprev[src];
        cplx sd = duprev[src];
        up.re = sign * su.re;
        up.im = -sign * su.im;
        dup.re = sign * sd.re;
        dup.im = -sign * sd.im;
      }
      double rp = rootpq(t - ma, t - mb);
      row[ma].re += rp * (da.re * up.re + da.im * up.im + a.re * dup.re +
                          a.im * dup.im);
      row[ma].im += rp * (da.re * up.im - da.im * up.re + a.re * dup.im -
                          a.im * dup.re);
      rp = rootpq(ma + 1, t - mb);
      row[ma + 1].re = -rp * (db.re * up.re + db.im * up.im + b.re * dup.re +
                              b.im * dup.im);
      row[ma + 1].im = -rp * (db.re * up.im - db.im * up.re + b.re * dup.im -
                              b.im * dup.re);
    }
  }
}

static void wigner_u_recursion_half(cplx a, cplx b, int T, cplx* out) {
  /* :300-329, half storage */
  out[0].re = 1.0;
  out[0].im = 0.0;
  int off = 1, off_prev = 0;
  for (int t = 1; t <= T; ++t) {
    wigner_u_level_half(a, b, t, out + off_prev, out + off);
    off_prev = off;
    off += half_block(t);
  }
}

int orc_wigner_u_half(const double disp[3], double rcut, double rmin0,
                      double rfac0, int T, double* out) {
  sphere_map m;
  if (map_to_3sphere(disp, rcut, rmin0, rfac0, &m)) return -1;
  wigner_u_recursion_half(m.a, m.b, T, (cplx*)out);
  return 0;
}

/* ------------------------------------------------------------------------ */
/* Pipeline helpers (snap_core.hpp)                                          */
/* ------------------------------------------------------------------------ */

/* UtotView::get over logical half storage :190-199 */
static cplx utot_get(const cplx* uh, const maps_t* m, int t, int mb, int ma) {
  if (2 * mb <= t) return uh[m->half_off[t] + mb * (t + 1) + ma];
  cplx v = uh[m->half_off[t] + (t - mb) * (t + 1) + (t - ma)];
  const double sign = ((ma + mb) & 1) ? -1.0 : 1.0;
  cplx r;
  r.re = sign * v.re;
  r.im = -sign * v.im;
  return r;
}

/* expand_utot_full :237-245 */
static void expand_utot_full(const cplx* uh, const maps_t* m, cplx* out) {
  for (int t = 0; t <= m->T; ++t) {
    cplx* blk = out + m->full_off[t];
    for (int mb = 0; mb <= t; ++mb)
      for (int ma = 0; ma <= t; ++ma) blk[mb * (t + 1) + ma] = utot_get(uh, m, t, mb, ma);
  }
}

/* z_element over a flat full stack :249-279 */
static cplx z_element(const cplx* ufull, int off1, int off2, const double* cgb,
                      int j1, int j2, int j, int mb, int ma) {
  int zb[6];
  orc_z_loop_bounds(j1, j2, j, mb, ma, zb);
  cplx zsum = {0.0, 0.0};
  int mb1 = zb[3], mb2 = zb[4];
  int icgb = mb1 * (j2 + 1) + mb2;
  for (int ib = 0; ib < zb[5]; ++ib) {
    cplx suma = {0.0, 0.0};
    int ma1 = zb[0], ma2 = zb[1];
    int icga = ma1 * (j2 + 1) + ma2;
    const cplx* row1 = ufull + off1 + mb1 * (j1 + 1);
    const cplx* row2 = ufull + off2 + mb2 * (j2 + 1);
    for (int ia = 0; ia < zb[2]; ++ia) {
      const cplx u1 = row1[ma1];
      const cplx u2 = row2[ma2];
      const double c = cgb[icga];
      suma.re += c * (u1.re * u2.re - u1.im * u2.im);
      suma.im += c * (u1.re * u2.im + u1.im * u2.re);
      ++ma1;
      --ma2;
      icga += j2;
    }
    zsum.re += cgb[icgb] * suma.re;
    zsum.im += cgb[icgb] * suma.im;
    ++mb1;
    --mb2;
    icgb += j2;
  }
  return zsum;
}

/* fold_beta :308-322 */
static double fold_beta(const maps_t* m, const double* beta, int j1, int j2,
                        int j) {
  if (j >= j1) {
    const double b = beta[m->triple_flat[dense(m, j1, j2, j)]];
    if (j1 == j) return (j2 == j) ? 3.0 * b : 2.0 * b;
    return b;
  }
  if (j >= j2) {
    const double b = beta[m->triple_flat[dense(m, j, j2, j1)]];
    const double ratio = (double)(j1 + 1) / (double)(j + 1);
    return (j2 == j ? 2.0 * b : b) * ratio;
  }
  const double b = beta[m->triple_flat[dense(m, j2, j, j1)]];
  return b * (double)(j1 + 1) / (double)(j + 1);
}

static double re_mul_conj(cplx x, cplx y) { return x.re * y.re + x.im * y.im; }

/* b_contract over a flat full level block :579-598 */
static void b_contract(const cplx* zblk, const cplx* ublk, int j, double* bval,
                       double* resid) {
  double acc = 0.0, mid_re = 0.0, mid_im = 0.0;
  const int cols = j + 1;
  for (int mb = 0; 2 * mb < j; ++mb)
    for (int ma = 0; ma <= j; ++ma) {
      const cplx uu = ublk[mb * cols + ma];
      acc += re_mul_conj(zblk[mb * cols + ma], uu);
    }
  if ((j & 1) == 0) {
    const int mb = j / 2;
    for (int ma = 0; ma <= j; ++ma) {
      const cplx z = zblk[mb * cols + ma];
      const cplx uu = ublk[mb * cols + ma];
      mid_re += re_mul_conj(z, uu);
      mid_im += z.im * uu.re - z.re * uu.im;
    }
  }
  *bval = 2.0 * acc + mid_re;
  *resid = fabs(mid_im);
}

static int validate(const orc_problem* p) { /* Problem::validate :89-118 */
  if (p->natoms <= 0) return fail("problem: no atoms");
  if (p->nweights <= 0) return fail("problem: empty weight table");
  if (!(p->rcut > p->rmin0)) return fail("problem: Rcut must exceed rmin0");
  if (p->twojmax < 0) return fail("problem: twojmax < 0");
  const double rc2 = p->rcut * p->rcut;
  for (int i = 0; i < p->natoms; ++i) {
    const int ti = p->types ? p->types[i] : 0;
    if (ti < 0 || ti >= p->nweights)
      return fail("problem: atom type outside weight table");
    if (p->numneigh[i] < 0 || p->numneigh[i] > p->stride)
      return fail("problem: neighbor count outside stride");
    for (int k = 0; k < p->numneigh[i]; ++k) {
      const int idx = p->nbr[(size_t)i * p->stride + k];
      const double* d = p->disp + ((size_t)i * p->stride + k) * 3;
      if (idx < 0 || idx >= p->natoms) return fail("problem: neighbor index out of range");
      if (idx == i) return fail("problem: self neighbor");
      const double r2 = d[0] * d[0] + d[1] * d[1] + d[2] * d[2];
      if (!(r2 > 0.0)) return fail("problem: zero-length neighbor displacement");
      if (!(r2 < rc2)) return fail("problem: neighbor at or beyond Rcut");
    }
  }
  if (p->nbeta != orc_n_triples(p->twojmax))
    return fail("problem: beta length must match the triple count");
  return 0;
}

static double weight_of(const orc_problem* p, int i) { /* :83-85 */
  return p->weights[p->types ? p->types[i] : 0];
}

/* ------------------------------------------------------------------------ */
/* The deterministic fused pipeline (pipeline.hpp:206-303, adjoint branch)   */
/* ------------------------------------------------------------------------ */
int orc_run(const orc_problem* p, double* forces, double* eatom, double* etotal,
            double* ulisttot_out, double* ylist_out, double* delist_out,
            double* blist_out) {
  if (validate(p)) return -1;
  const int T = p->twojmax;
  const int N = p->natoms, S = p->stride;
  maps_t m;
  maps_build(&m, T);
  const int nh = m.nhalf, nf = m.nfull;
  double* cg = (double*)malloc(sizeof(double) * (size_t)(m.cgtot + 1));
  orc_cg_table(T, cg);

  cplx* utot = (cplx*)calloc((size_t)N * nh, sizeof(cplx));
  cplx* ylist = (cplx*)calloc((size_t)N * nh, sizeof(cplx));
  double* delist = (double*)calloc((size_t)N * S * 3 + 1, sizeof(double));
  cplx* uscr = (cplx*)malloc(sizeof(cplx) * (size_t)nh);
  cplx* ufull = (cplx*)malloc(sizeof(cplx) * (size_t)nf);

  /* --- compute_U, half storage, deterministic (snap_core.hpp:369-453) --- */
  if (p->self_flag) {
    for (int a = 0; a < N; ++a)
      for (int t = 0; t <= T; ++t)
        for (int mb = 0; mb <= t / 2; ++mb) {
          cplx* e = utot + (size_t)a * nh + m.half_off[t] + mb * (t + 1) + mb;
          e->re = p->wself;
          e->im = 0.0;
        }
  }
  for (int i = 0; i < N; ++i)
    for (int k = 0; k < p->numneigh[i]; ++k) {
      const size_t pk = (size_t)i * S + k;
      sphere_map map;
      if (map_to_3sphere(p->disp + pk * 3, p->rcut, p->rmin0, p->rfac0, &map))
        goto error;
      double fc, dfc;
      switching_function(map.r, p->rcut, p->rmin0, &fc, &dfc);
      const double sfac = weight_of(p, p->nbr[pk]) * fc;
      wigner_u_recursion_half(map.a, map.b, T, uscr);
      cplx* tgt = utot + (size_t)i * nh;
      for (int e = 0; e < nh; ++e) {
        const double vr = sfac * uscr[e].re, vi = sfac * uscr[e].im;
        tgt[e].re += vr;
        tgt[e].im += vi;
      }
    }

  /* --- compute_B_from_U + compute_energy (snap_core.hpp:642-701) --- */
  if (eatom || etotal || blist_out) {
    double tot = 0.0;
    cplx* zscr = (cplx*)malloc(sizeof(cplx) * (size_t)half_block(T));
    for (int a = 0; a < N; ++a) {
      expand_utot_full(utot + (size_t)a * nh, &m, ufull);
      double e = 0.0;
      for (int l = 0; l < m.ntrip; ++l) {
        const int j1 = m.triples[3 * l], j2 = m.triples[3 * l + 1],
                  j = m.triples[3 * l + 2];
        const double* cgb = cg + m.cg_flat[dense(&m, j1, j2, j)];
        int ee = 0;
        for (int mb = 0; 2 * mb <= j; ++mb)
          for (int ma = 0; ma <= j; ++ma, ++ee)
            zscr[ee] = z_element(ufull, m.full_off[j1], m.full_off[j2], cgb, j1,
                                 j2, j, mb, ma);
        double bval, resid;
        b_contract(zscr, ufull + m.full_off[j], j, &bval, &resid);
        const double denom = fabs(bval) > 1.0 ? fabs(bval) : 1.0;
        if (resid > 1e-11 * denom) { /* check_b_residue :600-608 */
          free(zscr);
          fail("bispectrum imaginary residue %g at triple (%d,%d,%d)", resid, j1,
               j2, j);
          goto error;
        }
        if (blist_out) blist_out[(size_t)a * m.ntrip + l] = bval;
        e += p->beta[l] * bval; /* compute_energy :692-699 */
      }
      if (eatom) eatom[a] = e;
      tot += e;
    }
    if (etotal) *etotal = tot;
    free(zscr);
  }

  /* --- compute_Y, atom-owned path (snap_core.hpp:1128-1171) --- */
  {
    double* folded = (double*)malloc(sizeof(double) * (size_t)m.ntup);
    for (int q = 0; q < m.ntup; ++q)
      folded[q] = fold_beta(&m, p->beta, m.tuples[5 * q], m.tuples[5 * q + 1],
                            m.tuples[5 * q + 2]);
    for (int a = 0; a < N; ++a) {
      expand_utot_full(utot + (size_t)a * nh, &m, ufull);
      cplx* yloc = ylist + (size_t)a * nh;
      for (int q = 0; q < m.ntup; ++q) {
        const int j1 = m.tuples[5 * q], j2 = m.tuples[5 * q + 1],
                  j = m.tuples[5 * q + 2];
        const double betaj = folded[q];
        const double* cgb = cg + m.tuples[5 * q + 4];
        cplx* ydst = yloc + m.half_off[j];
        for (int mb = 0; 2 * mb <= j; ++mb)
          for (int ma = 0; ma <= j; ++ma) {
            const cplx z = z_element(ufull, m.full_off[j1], m.full_off[j2], cgb,
                                     j1, j2, j, mb, ma);
            cplx* y = ydst + mb * (j + 1) + ma;
            y->re += betaj * z.re;
            y->im += betaj * z.im;
          }
      }
    }
    free(folded);
  }

  /* --- compute_fused_dE, deterministic (snap_core.hpp:1274-1396) --- */
  {
    const int maxblk = half_block(T);
    cplx* bufs = (cplx*)calloc((size_t)maxblk * 8, sizeof(cplx));
    for (int i = 0; i < N; ++i) {
      const cplx* yf = ylist + (size_t)i * nh;
      for (int k = 0; k < p->numneigh[i]; ++k) {
        const size_t pk = (size_t)i * S + k;
        sphere_map map;
        if (map_to_3sphere(p->disp + pk * 3, p->rcut, p->rmin0, p->rfac0, &map)) {
          free(bufs);
          goto error;
        }
        double fc, dfc;
        switching_function(map.r, p->rcut, p->rmin0, &fc, &dfc);
        const double w = weight_of(p, p->nbr[pk]);
        const double sfac = w * fc, dsfac = w * dfc;
        double dsf[3], acc[3];
        for (int d = 0; d < 3; ++d) {
          dsf[d] = dsfac * map.rhat[d];
          acc[d] = 0.5 * dsf[d] * yf[0].re;
        }
        cplx* uprev = bufs;
        cplx* ucur = bufs + maxblk;
        cplx *dprev[3], *dcur[3];
        uprev[0].re = 1.0;
        uprev[0].im = 0.0;
        for (int d = 0; d < 3; ++d) {
          dprev[d] = bufs + (2 + 2 * d) * maxblk;
          dcur[d] = bufs + (3 + 2 * d) * maxblk;
          dprev[d][0].re = 0.0;
          dprev[d][0].im = 0.0;
        }
        for (int t = 1; t <= T; ++t) {
          wigner_u_level_half(map.a, map.b, t, uprev, ucur);
          for (int d = 0; d < 3; ++d)
            wigner_du_level_half(map.a, map.b, map.da[d], map.db[d], t, uprev,
                                 dprev[d], dcur[d]);
          const int cols = t + 1;
          const cplx* ylev = yf + m.half_off[t];
          for (int mb = 0; 2 * mb <= t; ++mb) {
            const int middle = (2 * mb == t);
            const int ma_end = middle ? t / 2 : t;
            for (int ma = 0; ma <= ma_end; ++ma) {
              const int e = mb * cols + ma;
              const cplx y = ylev[e];
              const double wgt = (middle && 2 * ma == t) ? 0.5 : 1.0;
              for (int d = 0; d < 3; ++d) {
                cplx duw;
                duw.re = dsf[d] * ucur[e].re + sfac * dcur[d][e].re;
                duw.im = dsf[d] * ucur[e].im + sfac * dcur[d][e].im;
                acc[d] += wgt * re_mul_conj(duw, y);
              }
            }
          }
          cplx* tmp = uprev;
          uprev = ucur;
          ucur = tmp;
          for (int d = 0; d < 3; ++d) {
            tmp = dprev[d];
            dprev[d] = dcur[d];
            dcur[d] = tmp;
          }
        }
        for (int d = 0; d < 3; ++d) delist[pk * 3 + d] = 2.0 * acc[d];
      }
    }
    free(bufs);
  }

  /* --- scatter_forces, deterministic (snap_core.hpp:889-899) --- */
  if (forces) {
    for (int s = 0; s < N * 3; ++s) forces[s] = 0.0;
    for (int i = 0; i < N; ++i)
      for (int k = 0; k < p->numneigh[i]; ++k) {
        const size_t pk = (size_t)i * S + k;
        const double* de = delist + pk * 3;
        const int kk = p->nbr[pk];
        for (int d = 0; d < 3; ++d) {
          forces[i * 3 + d] += de[d];
          forces[kk * 3 + d] -= de[d];
        }
      }
  }
  if (ulisttot_out) memcpy(ulisttot_out, utot, sizeof(cplx) * (size_t)N * nh);
  if (ylist_out) memcpy(ylist_out, ylist, sizeof(cplx) * (size_t)N * nh);
  if (delist_out) memcpy(delist_out, delist, sizeof(double) * (size_t)N * S * 3);

  free(cg);
  free(utot);
  free(ylist);
  free(delist);
  free(uscr);
  free(ufull);
  maps_free(&m);
  return 0;
error:
  free(cg);
  free(utot);
  free(ylist);
  free(delist);
  free(uscr);
  free(ufull);
  maps_free(&m);
  return -1;
}

/* ------------------------------------------------------------------------ */
/* Problem generators                                                        */
/* ------------------------------------------------------------------------ */
int orc_bcc(int nx, int ny, int nz, double a, double jitter, uint64_t seed,
            int T, double* pos, double* beta) {
  rng_t r;
  rng_seed(&r, seed);
  const int nt = orc_n_triples(T);
  for (int l = 0; l < nt; ++l) beta[l] = rng_uniform(&r, -1.0, 1.0); /* harness.hpp:208-213 */
  int n = 0;
  for (int cz = 0; cz < nz; ++cz)
    for (int cy = 0; cy < ny; ++cy)
      for (int cx = 0; cx < nx; ++cx)
        for (int bsi = 0; bsi < 2; ++bsi) {
          const double h = 0.5 * bsi;
          double base[3] = {(cx + h) * a, (cy + h) * a, (cz + h) * a};
          for (int d = 0; d < 3; ++d)
            pos[n * 3 + d] = base[d] + rng_uniform(&r, -jitter, jitter);
          ++n;
        }
  return n;
}

/* harness.hpp:82-90 */
static double wrap_coord(double x, double box) {
  double w = x - box * floor(x / box);
  return w >= box ? w - box : w;
}
static double min_image(double d, double box) {
  return d - box * nearbyint(d / box);
}

typedef struct {
  int idx;
  double d[3];
} nb_t;

static int cmp_nb(const void* x, const void* y) {
  const nb_t* a = (const nb_t*)x;
  const nb_t* b = (const nb_t*)y;
  return (a->idx > b->idx) - (a->idx < b->idx);
}

/* build_neighborlist (harness.hpp:119-202), direct O(n^2) scan: the result
 * does not depend on traversal order (lists are sorted by index and the
 * minimum-image displacement is odd-symmetric), so this is bitwise equal to
 * the reference's cell-list construction. */
int orc_build_neighborlist(const double* pos, int n, const double box[3],
                           double rcut, int maxstride, int* numneigh, int* nbr,
                           double* disp) {
  for (int d = 0; d < 3; ++d) {
    if (!(box[d] > 0.0) || !(rcut > 0.0))
      return fail("build_neighborlist: box and Rcut must be positive");
    if (!(rcut <= 0.5 * box[d]))
      return fail("build_neighborlist: Rcut must not exceed box/2");
  }
  double* w = (double*)malloc(sizeof(double) * 3 * (size_t)(n + 1));
  for (int i = 0; i < n; ++i)
    for (int c = 0; c < 3; ++c) w[i * 3 + c] = wrap_coord(pos[i * 3 + c], box[c]);
  const double rc2 = rcut * rcut;
  int cap = 64;
  nb_t** lists = (nb_t**)malloc(sizeof(nb_t*) * (size_t)(n + 1));
  int* cnt = (int*)calloc((size_t)n + 1, sizeof(int));
  int* capv = (int*)malloc(sizeof(int) * (size_t)(n + 1));
  for (int i = 0; i < n; ++i) {
    lists[i] = (nb_t*)malloc(sizeof(nb_t) * (size_t)cap);
    capv[i] = cap;
  }
  for (int i = 0; i < n; ++i)
    for (int k = i + 1; k < n; ++k) {
      double d[3];
      for (int c = 0; c < 3; ++c) d[c] = min_image(w[k * 3 + c] - w[i * 3 + c], box[c]);
      const double r2 = d[0] * d[0] + d[1] * d[1] + d[2] * d[2];
      if (r2 < rc2) {
        int ab[2] = {i, k};
        for (int s = 0; s < 2; ++s) {
          int x = ab[s];
          if (cnt[x] == capv[x]) {
            capv[x] *= 2;
            lists[x] = (nb_t*)realloc(lists[x], sizeof(nb_t) * (size_t)capv[x]);
          }
          nb_t* e = &lists[x][cnt[x]++];
          e->idx = s == 0 ? k : i;
          for (int c = 0; c < 3; ++c) e->d[c] = s == 0 ? d[c] : -d[c];
        }
      }
    }
  int mx = 0;
  for (int i = 0; i < n; ++i) {
    qsort(lists[i], (size_t)cnt[i], sizeof(nb_t), cmp_nb);
    if (cnt[i] > mx) mx = cnt[i];
  }
  for (int i = 0; i < n; ++i) {
    if (numneigh) numneigh[i] = cnt[i];
    if (mx <= maxstride && nbr && disp)
      for (int k = 0; k < cnt[i]; ++k) {
        nbr[(size_t)i * maxstride + k] = lists[i][k].idx;
        for (int c = 0; c < 3; ++c)
          disp[((size_t)i * maxstride + k) * 3 + c] = lists[i][k].d[c];
      }
    free(lists[i]);
  }
  free(lists);
  free(cnt);
  free(capv);
  free(w);
  return mx;
}

/* tests/test_support.hpp:21-64 */
int orc_make_cluster(int natoms, int T, uint64_t seed, int ntypes, double* pos,
                     int* types, double* weights, int* numneigh, int* nbr,
                     double* disp, double* beta) {
  const double kRcut = 4.7;
  rng_t r;
  rng_seed(&r, seed);
  const double side = 0.8 * kRcut;
  for (int i = 0; i < natoms; ++i)
    for (int d = 0; d < 3; ++d) pos[i * 3 + d] = rng_uniform(&r, 0.0, side);
  if (natoms > 1) {
    pos[3] = pos[0] + 1.3;
    pos[4] = pos[1] + 0.4;
    pos[5] = pos[2] - 0.2;
  }
  for (int t = 0; t < ntypes; ++t) weights[t] = t == 0 ? 1.0 : rng_uniform(&r, 0.2, 0.9);
  for (int i = 0; i < natoms; ++i) types[i] = i % ntypes;
  int mx = 0;
  for (int i = 0; i < natoms; ++i) {
    int c = 0;
    for (int k = 0; k < natoms; ++k) {
      if (i == k) continue;
      double d[3], r2 = 0.0;
      for (int q = 0; q < 3; ++q) {
        d[q] = pos[k * 3 + q] - pos[i * 3 + q];
        r2 += d[q] * d[q];
      }
      if (r2 > 0.0 && r2 < 0.98 * kRcut * kRcut) {
        nbr[(size_t)i * natoms + c] = k;
        for (int q = 0; q < 3; ++q) disp[((size_t)i * natoms + c) * 3 + q] = d[q];
        ++c;
      }
    }
    numneigh[i] = c;
    if (c > mx) mx = c;
  }
  const int nt = orc_n_triples(T);
  for (int l = 0; l < nt; ++l) beta[l] = rng_uniform(&r, -1.0, 1.0);
  return mx;
}

/* harness.hpp:230-262 */
int orc_generate_synthetic(int natoms, int nnbor, int T, double rcut,
                           uint64_t seed, int* numneigh, int* nbr, double* disp,
                           double* beta) {
  rng_t r;
  rng_seed(&r, seed);
  const int nt = orc_n_triples(T);
  for (int l = 0; l < nt; ++l) beta[l] = rng_uniform(&r, -1.0, 1.0);
  if (natoms < 2) {
    for (int i = 0; i < natoms; ++i) numneigh[i] = 0;
    return 0;
  }
  for (int i = 0; i < natoms; ++i) {
    numneigh[i] = nnbor;
    for (int t = 0; t < nnbor; ++t) {
      double dir[3];
      rng_unit_vector(&r, dir);
      const double rr = rcut * rng_uniform(&r, 0.3, 0.95);
      const size_t pk = (size_t)i * nnbor + t;
      nbr[pk] = (i + 1 + t % (natoms - 1)) % natoms;
      disp[pk * 3 + 0] = dir[0] * rr;
      disp[pk * 3 + 1] = dir[1] * rr;
      disp[pk * 3 + 2] = dir[2] * rr;
    }
  }
  return nnbor;
}
