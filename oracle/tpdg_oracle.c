/* tpdg oracle -- CPU restatement of the reference hot path. TEST INFRASTRUCTURE ONLY.
 * See tpdg_oracle.h for scope and layouts. Reference citations are relative to
 * /root/reference/proj/include/tpdg/. Build with -ffp-contract=off.
 */
#include "tpdg_oracle.h"

#include <math.h>
#include <stdlib.h>
#include <string.h>

#define MAXQ 64

static void *xcalloc(size_t n, size_t sz) {
  void *p = calloc(n ? n : 1, sz);
  if (!p) abort();
  return p;
}

/* ======================================================================
 * libstdc++ <random> restated (std::mt19937_64, generate_canonical<double,53>,
 * uniform_real_distribution, normal_distribution polar method). Used by the
 * reference for the Lanczos start vector (tensor/lanczos.hpp:61-72) and by the
 * tests for seeded RHS vectors (tests/support/test_rng.hpp:20-25).
 * ====================================================================== */
typedef struct {
  uint64_t mt[312];
  int idx;
} mt64;

static void mt64_seed(mt64 *r, uint64_t seed) {
  r->mt[0] = seed;
  for (int i = 1; i < 312; ++i) r->mt[i] = 6364136223846793005ULL * (r->mt[i - 1] ^ (r->mt[i - 1] >> 62)) + (uint64_t)i;
  r->idx = 312;
}

static uint64_t mt64_next(mt64 *r) {
  if (r->idx >= 312) {
    for (int i = 0; i < 312; ++i) {
      const uint64_t y = (r->mt[i] & 0xFFFFFFFF80000000ULL) | (r->mt[(i + 1) % 312] & 0x7FFFFFFFULL);
      uint64_t v = r->mt[(i + 156) % 312] ^ (y >> 1);
      if (y & 1ULL) v ^= 0xB5026F5AA96619E9ULL;
      r->mt[i] = v;
    }
    r->idx = 0;
  }
  uint64_t z = r->mt[r->idx++];
  z ^= (z >> 29) & 0x5555555555555555ULL;
  z ^= (z << 17) & 0x71D67FFFEDA60000ULL;
  z ^= (z << 37) & 0xFFF7EEE000000000ULL;
  z ^= z >> 43;
  return z;
}

static double canonical(mt64 *r) {
  const double sum = (double)mt64_next(r);
  double ret = sum / 18446744073709551616.0; /* 2^64 */
  if (ret >= 1.0) ret = nextafter(1.0, 0.0);
  return ret;
}

void or_uniform_vector(uint64_t seed, long n, double scale, double *out) {
  mt64 r;
  mt64_seed(&r, seed);
  for (long i = 0; i < n; ++i) out[i] = canonical(&r) * (scale - (-scale)) + (-scale);
}

void or_seeded_unit_vector(long n, uint64_t seed, double *out) {
  mt64 r;
  mt64_seed(&r, seed);
  int saved_ok = 0;
  double saved = 0.0, nrm = 0.0;
  while (nrm == 0.0) {
    for (long i = 0; i < n; ++i) {
      double ret;
      if (saved_ok) {
        saved_ok = 0;
        ret = saved;
      } else {
        double x, y, r2;
        do {
          x = 2.0 * canonical(&r) - 1.0;
          y = 2.0 * canonical(&r) - 1.0;
          r2 = x * x + y * y;
        } while (r2 > 1.0 || r2 == 0.0);
        const double mult = sqrt(-2 * log(r2) / r2);
        saved = x * mult;
        saved_ok = 1;
        ret = y * mult;
      }
      out[i] = ret * 1.0 + 0.0;
    }
    double s = 0.0;
    for (long i = 0; i < n; ++i) s += out[i] * out[i];
    nrm = sqrt(s);
  }
  for (long i = 0; i < n; ++i) out[i] /= nrm;
}

/* ======================================================================
 * Sum-factorization kernels (ops/kernels.hpp).
 * ====================================================================== */

/* dst = M along `axis`, first axis fastest (ops/kernels.hpp:11-32); M nout x nin. */
static void axis_apply(const double *m, int nout, int nin, int dim, const int *ext, int axis, const double *src,
                       double *dst) {
  long inner = 1, outer = 1;
  for (int k = 0; k < axis; ++k) inner *= ext[k];
  for (int k = axis + 1; k < dim; ++k) outer *= ext[k];
  for (long o = 0; o < outer; ++o) {
    const double *sp = src + o * nin * inner;
    double *tp = dst + o * nout * inner;
    for (long k = 0; k < nout * inner; ++k) tp[k] = 0.0;
    for (int j = 0; j < nin; ++j)
      for (int i = 0; i < nout; ++i) {
        const double mij = m[i * nin + j];
        if (mij == 0.0) continue;
        for (long t = 0; t < inner; ++t) tp[i * inner + t] += mij * sp[j * inner + t];
      }
  }
}

/* vals(mu^d) = G x..x G coeff (ops/kernels.hpp:60-78). */
static void eval_at_quad(const or_sys *s, const double *coeff, double *vals) {
  const int n = s->q, mu = s->mu;
  int ext[3] = {n, n, n};
  double *a = (double *)xcalloc((size_t)mu * mu * n, sizeof(double));
  if (s->dim == 2) {
    axis_apply(s->g, mu, n, 2, ext, 0, coeff, a);
    ext[0] = mu;
    axis_apply(s->g, mu, n, 2, ext, 1, a, vals);
  } else {
    double *b = (double *)xcalloc((size_t)mu * mu * n, sizeof(double));
    axis_apply(s->g, mu, n, 3, ext, 0, coeff, a);
    ext[0] = mu;
    axis_apply(s->g, mu, n, 3, ext, 1, a, b);
    ext[1] = mu;
    axis_apply(s->g, mu, n, 3, ext, 2, b, vals);
    free(b);
  }
  free(a);
}

/* out(q^d) += (GW|DW) x .. field (ops/kernels.hpp:82-104); dslot -1 = all GW. */
static void integrate_back(const or_sys *s, int dslot, const double *field, double *out) {
  const int n = s->q, mu = s->mu;
  int ext[3] = {mu, mu, mu};
  double *c = (double *)xcalloc((size_t)n * mu * mu, sizeof(double));
  double *d = (double *)xcalloc((size_t)n * n * mu, sizeof(double));
  if (s->dim == 2) {
    axis_apply(dslot == 0 ? s->dw : s->gw, n, mu, 2, ext, 0, field, c);
    ext[0] = n;
    axis_apply(dslot == 1 ? s->dw : s->gw, n, mu, 2, ext, 1, c, d);
    for (int i = 0; i < n * n; ++i) out[i] += d[i];
  } else {
    double *e = (double *)xcalloc((size_t)n * n * n, sizeof(double));
    axis_apply(dslot == 0 ? s->dw : s->gw, n, mu, 3, ext, 0, field, c);
    ext[0] = n;
    axis_apply(dslot == 1 ? s->dw : s->gw, n, mu, 3, ext, 1, c, d);
    ext[1] = n;
    axis_apply(dslot == 2 ? s->dw : s->gw, n, mu, 3, ext, 2, d, e);
    for (int i = 0; i < n * n * n; ++i) out[i] += e[i];
    free(e);
  }
  free(c);
  free(d);
}

/* dg/mesh.hpp:44-67 */
static void face_tangents(int dim, int axis, int *t0, int *t1) {
  if (dim == 2) {
    *t0 = axis == 0 ? 1 : 0;
    *t1 = -1;
  } else if (axis == 0) {
    *t0 = 1;
    *t1 = 2;
  } else if (axis == 1) {
    *t0 = 0;
    *t1 = 2;
  } else {
    *t0 = 0;
    *t1 = 1;
  }
}

static void orient(int dim, int code, int n, int a, int b, int *oa, int *ob) {
  if (dim == 2) {
    *oa = code == 0 ? a : n - 1 - a;
    *ob = 0;
    return;
  }
  int u = (code & 4) ? b : a, v = (code & 4) ? a : b;
  if (code & 1) u = n - 1 - u;
  if (code & 2) v = n - 1 - v;
  *oa = u;
  *ob = v;
}

static int flat3(int n, const int idx[3]) { return (idx[2] * n + idx[1]) * n + idx[0]; }

/* face_trace (ops/discretization.hpp:89-129) */
static void face_trace(const or_sys *s, int face, const double *coeff, double *vals) {
  const int n = s->q, mu = s->mu, axis = face / 2, layer = (face % 2) == 0 ? 0 : n - 1;
  if (s->dim == 2) {
    double f[MAXQ];
    for (int j = 0; j < n; ++j) f[j] = axis == 0 ? coeff[j * n + layer] : coeff[layer * n + j];
    for (int a = 0; a < mu; ++a) {
      double acc = 0.0;
      for (int j = 0; j < n; ++j) acc += s->g[a * n + j] * f[j];
      vals[a] = acc;
    }
    return;
  }
  int t0, t1;
  face_tangents(3, axis, &t0, &t1);
  double *f = (double *)xcalloc((size_t)n * n, sizeof(double));
  double *wa = (double *)xcalloc((size_t)n * mu, sizeof(double));
  for (int j1 = 0; j1 < n; ++j1)
    for (int j0 = 0; j0 < n; ++j0) {
      int idx[3];
      idx[axis] = layer;
      idx[t0] = j0;
      idx[t1] = j1;
      f[j1 * n + j0] = coeff[flat3(n, idx)];
    }
  for (int a = 0; a < mu; ++a)
    for (int j1 = 0; j1 < n; ++j1) {
      double acc = 0.0;
      for (int j0 = 0; j0 < n; ++j0) acc += s->g[a * n + j0] * f[j1 * n + j0];
      wa[j1 * mu + a] = acc;
    }
  for (int bb = 0; bb < mu; ++bb)
    for (int a = 0; a < mu; ++a) {
      double acc = 0.0;
      for (int j1 = 0; j1 < n; ++j1) acc += s->g[bb * n + j1] * wa[j1 * mu + a];
      vals[bb * mu + a] = acc;
    }
  free(f);
  free(wa);
}

/* face_lift (ops/discretization.hpp:133-166) */
static void face_lift(const or_sys *s, int face, const double *gq, double *out) {
  const int n = s->q, mu = s->mu, axis = face / 2, layer = (face % 2) == 0 ? 0 : n - 1;
  if (s->dim == 2) {
    for (int j = 0; j < n; ++j) {
      double acc = 0.0;
      for (int a = 0; a < mu; ++a) acc += s->g[a * n + j] * gq[a];
      if (axis == 0)
        out[j * n + layer] += acc;
      else
        out[layer * n + j] += acc;
    }
    return;
  }
  int t0, t1;
  face_tangents(3, axis, &t0, &t1);
  double *wa = (double *)xcalloc((size_t)n * mu, sizeof(double));
  for (int j0 = 0; j0 < n; ++j0)
    for (int bb = 0; bb < mu; ++bb) {
      double acc = 0.0;
      for (int a = 0; a < mu; ++a) acc += s->g[a * n + j0] * gq[bb * mu + a];
      wa[j0 * mu + bb] = acc;
    }
  for (int j1 = 0; j1 < n; ++j1)
    for (int j0 = 0; j0 < n; ++j0) {
      double acc = 0.0;
      for (int bb = 0; bb < mu; ++bb) acc += s->g[bb * n + j1] * wa[j0 * mu + bb];
      int idx[3];
      idx[axis] = layer;
      idx[t0] = j0;
      idx[t1] = j1;
      out[flat3(n, idx)] += acc;
    }
  free(wa);
}

static long npe_of(const or_sys *s) { return s->dim == 2 ? (long)s->q * s->q : (long)s->q * s->q * s->q; }
static long nqv_of(const or_sys *s) { return s->dim == 2 ? (long)s->mu * s->mu : (long)s->mu * s->mu * s->mu; }
static long nqf_of(const or_sys *s) { return s->dim == 2 ? (long)s->mu : (long)s->mu * s->mu; }

/* neighbor_trace (ops/discretization.hpp:170-181) */
static void neighbor_trace(const or_sys *s, int e, int face, const double *u, int c, double *vals) {
  const int64_t *fc = s->conn + ((size_t)e * 2 * s->dim + face) * 3;
  const long npe = npe_of(s), nqf = nqf_of(s);
  double *wb = (double *)xcalloc((size_t)nqf, sizeof(double));
  face_trace(s, (int)fc[1], u + ((size_t)fc[0] * s->n_c + c) * npe, wb);
  const int mu = s->mu;
  for (long qq = 0; qq < nqf; ++qq) {
    int qa, qb;
    orient(s->dim, (int)fc[2], mu, (int)(qq % mu), s->dim == 3 ? (int)(qq / mu) : 0, &qa, &qb);
    vals[qq] = wb[(s->dim == 3 ? qb * mu : 0) + qa];
  }
  free(wb);
}

/* element_diag_apply (ops/linearized.hpp:107-162): vout += a M v + b J_ee v */
void or_elem_diag_apply(const or_sys *s, int e, double a, double b, int small_mode, const double *vin,
                        double *vout) {
  const int nc = s->n_c, d = s->dim;
  const long npe = npe_of(s), nqv = nqv_of(s), nqf = nqf_of(s);
  double *vals = (double *)xcalloc((size_t)nc * nqv, sizeof(double));
  double *field = (double *)xcalloc((size_t)nqv, sizeof(double));
  for (int c = 0; c < nc; ++c) eval_at_quad(s, vin + (size_t)c * npe, vals + (size_t)c * nqv);
  const double *jd = s->jdet + (size_t)e * nqv;
  if (a != 0.0)
    for (int c = 0; c < nc; ++c) {
      for (long qq = 0; qq < nqv; ++qq) field[qq] = a * jd[qq] * vals[(size_t)c * nqv + qq];
      integrate_back(s, -1, field, vout + (size_t)c * npe);
    }
  if (b != 0.0) {
    for (int dir = 0; dir < d; ++dir) {
      const double *dft = s->dft + (((size_t)e * d + dir) * nqv) * nc * nc;
      for (int r = 0; r < nc; ++r) {
        for (long qq = 0; qq < nqv; ++qq) {
          double acc = 0.0;
          if (!small_mode) {
            for (int c = 0; c < nc; ++c) acc += dft[(size_t)qq * nc * nc + r * nc + c] * vals[(size_t)c * nqv + qq];
          } else {
            acc = dft[(size_t)qq * nc * nc + r * nc + r] * vals[(size_t)r * nqv + qq];
          }
          field[qq] = b * acc;
        }
        integrate_back(s, dir, field, vout + (size_t)r * npe);
      }
    }
    double *tm = (double *)xcalloc((size_t)nc * nqf, sizeof(double));
    double *gq = (double *)xcalloc((size_t)nqf, sizeof(double));
    for (int f = 0; f < 2 * d; ++f) {
      for (int c = 0; c < nc; ++c) face_trace(s, f, vin + (size_t)c * npe, tm + (size_t)c * nqf);
      const double *dfm = s->dfm + (((size_t)e * 2 * d + f) * nqf) * nc * nc;
      const double *fw = s->face_w + ((size_t)e * 2 * d + f) * nqf;
      for (int r = 0; r < nc; ++r) {
        for (long qq = 0; qq < nqf; ++qq) {
          double acc = 0.0;
          if (!small_mode) {
            for (int c = 0; c < nc; ++c) acc += dfm[(size_t)qq * nc * nc + r * nc + c] * tm[(size_t)c * nqf + qq];
          } else {
            acc = dfm[(size_t)qq * nc * nc + r * nc + r] * tm[(size_t)r * nqf + qq];
          }
          gq[qq] = -b * fw[qq] * acc;
        }
        face_lift(s, f, gq, vout + (size_t)r * npe);
      }
    }
    free(tm);
    free(gq);
  }
  free(vals);
  free(field);
}

/* jacobian_apply (ops/linearized.hpp:201-240) */
void or_jv(const or_sys *s, double a, double b, int small_mode, const double *vin, double *vout) {
  const int nc = s->n_c, d = s->dim;
  const long npe = npe_of(s), nqf = nqf_of(s), blk = (long)nc * npe;
  memset(vout, 0, sizeof(double) * (size_t)s->n_elements * blk);
  double *tp = (double *)xcalloc((size_t)nc * nqf, sizeof(double));
  double *gq = (double *)xcalloc((size_t)nqf, sizeof(double));
  for (int e = 0; e < s->n_elements; ++e) {
    or_elem_diag_apply(s, e, a, b, small_mode, vin + (size_t)e * blk, vout + (size_t)e * blk);
    for (int f = 0; f < 2 * d; ++f) {
      const int64_t *fc = s->conn + ((size_t)e * 2 * d + f) * 3;
      if (fc[0] < 0) continue;
      for (int c = 0; c < nc; ++c) neighbor_trace(s, e, f, vin, c, tp + (size_t)c * nqf);
      const double *dfp = s->dfp + (((size_t)e * 2 * d + f) * nqf) * nc * nc;
      const double *fw = s->face_w + ((size_t)e * 2 * d + f) * nqf;
      for (int r = 0; r < nc; ++r) {
        for (long qq = 0; qq < nqf; ++qq) {
          double acc = 0.0;
          if (!small_mode) {
            for (int c = 0; c < nc; ++c) acc += dfp[(size_t)qq * nc * nc + r * nc + c] * tp[(size_t)c * nqf + qq];
          } else {
            acc = dfp[(size_t)qq * nc * nc + r * nc + r] * tp[(size_t)r * nqf + qq];
          }
          gq[qq] = -b * fw[qq] * acc;
        }
        face_lift(s, f, gq, vout + (size_t)e * blk + (size_t)r * npe);
      }
    }
  }
  free(tp);
  free(gq);
}

/* assemble_diag_block(_small) (ops/linearized.hpp:245-285): probing with unit vectors. */
void or_assemble_block(const or_sys *s, int e, double a, double b, int small_mode, int comp, double *blk) {
  const long npe = npe_of(s), nfull = (long)s->n_c * npe;
  const long n = small_mode ? npe : nfull;
  double *vin = (double *)xcalloc((size_t)nfull, sizeof(double));
  double *vout = (double *)xcalloc((size_t)nfull, sizeof(double));
  const long off = small_mode ? (long)comp * npe : 0;
  for (long j = 0; j < n; ++j) {
    vin[off + j] = 1.0;
    memset(vout, 0, sizeof(double) * (size_t)nfull);
    or_elem_diag_apply(s, e, a, b, small_mode, vin, vout);
    for (long i = 0; i < n; ++i) blk[i * n + j] = vout[off + i];
    vin[off + j] = 0.0;
  }
  free(vin);
  free(vout);
}

/* ======================================================================
 * Matrix-free shuffled products of one element block (ops/shuffled.hpp:22-505).
 * ====================================================================== */
typedef struct {
  const or_sys *s;
  int e, small_mode, comp, ncb;
  double a, b;
} shuf_ctx;

static double sh_dft(const shuf_ctx *k, int dir, long qv, int r, int c) {
  const int nc = k->s->n_c, d = k->s->dim;
  const int rr = k->small_mode ? k->comp : r, cc = k->small_mode ? k->comp : c;
  return k->s->dft[((((size_t)k->e * d + dir) * nqv_of(k->s)) + qv) * nc * nc + rr * nc + cc];
}
static double sh_dfm(const shuf_ctx *k, int f, long qf, int r, int c) {
  const int nc = k->s->n_c, d = k->s->dim;
  const int rr = k->small_mode ? k->comp : r, cc = k->small_mode ? k->comp : c;
  return k->s->dfm[((((size_t)k->e * 2 * d + f) * nqf_of(k->s)) + qf) * nc * nc + rr * nc + cc];
}

#define GM(a, j) (S->g[(a) * q + (j)])
#define DM(a, j) (S->d[(a) * q + (j)])

/* ElementShuffled::apply_2d (ops/shuffled.hpp:65-147): u = Atilde v */
static void shuf_apply_2d(const shuf_ctx *k, const double *v, double *u) {
  const or_sys *S = k->s;
  const int q = S->q, mu = S->mu, nc = k->ncb, m1 = nc * q;
  const double a = k->a, b = k->b;
  double tgg[MAXQ], tdg[MAXQ], sm[MAXQ];
  for (int al = 0; al < mu; ++al) {
    double sg = 0.0, sd = 0.0;
    for (int ec = 0; ec < q; ++ec) {
      double cg = 0.0, cd = 0.0;
      for (int ar = 0; ar < q; ++ar) {
        cg += GM(al, ar) * v[ec * q + ar];
        cd += DM(al, ar) * v[ec * q + ar];
      }
      sg += GM(al, ec) * cg;
      sd += GM(al, ec) * cd;
    }
    tgg[al] = sg;
    tdg[al] = sd;
  }
  const double *jd = S->jdet + (size_t)k->e * mu * mu;
  double *r1 = (double *)xcalloc((size_t)nc * nc * mu, sizeof(double));
  double *r2 = (double *)xcalloc((size_t)nc * nc * mu, sizeof(double));
  for (int be = 0; be < mu; ++be) sm[be] = 0.0;
  for (int be = 0; be < mu; ++be)
    for (int al = 0; al < mu; ++al) {
      const int qv = be * mu + al;
      const double w = S->w[al];
      sm[be] += w * jd[qv] * tgg[al];
      if (b != 0.0)
        for (int cr = 0; cr < nc; ++cr)
          for (int cc = 0; cc < nc; ++cc) {
            r1[(cr * nc + cc) * mu + be] += w * sh_dft(k, 0, qv, cr, cc) * tdg[al];
            r2[(cr * nc + cc) * mu + be] += w * sh_dft(k, 1, qv, cr, cc) * tgg[al];
          }
    }
  for (int cc = 0; cc < nc; ++cc)
    for (int dc = 0; dc < q; ++dc)
      for (int cr = 0; cr < nc; ++cr)
        for (int br = 0; br < q; ++br) {
          double acc = 0.0;
          for (int be = 0; be < mu; ++be) {
            const double wb = S->w[be];
            double val = 0.0;
            if (cr == cc && a != 0.0) val += a * sm[be];
            if (b != 0.0) val += b * r1[(cr * nc + cc) * mu + be];
            acc += wb * GM(be, br) * GM(be, dc) * val;
            if (b != 0.0) acc += wb * DM(be, br) * GM(be, dc) * b * r2[(cr * nc + cc) * mu + be];
          }
          u[(cc * q + dc) * m1 + cr * q + br] = acc;
        }
  if (b != 0.0) {
    for (int f = 0; f < 4; ++f) {
      const double *fw = S->face_w + ((size_t)k->e * 4 + f) * mu;
      const int layer = (f % 2) == 0 ? 0 : q - 1;
      if (f / 2 == 0) {
        const double vc = v[layer * q + layer];
        for (int cc = 0; cc < nc; ++cc)
          for (int dc = 0; dc < q; ++dc)
            for (int cr = 0; cr < nc; ++cr)
              for (int br = 0; br < q; ++br) {
                double acc = 0.0;
                for (int be = 0; be < mu; ++be) acc += fw[be] * sh_dfm(k, f, be, cr, cc) * GM(be, br) * GM(be, dc);
                u[(cc * q + dc) * m1 + cr * q + br] -= b * acc * vc;
              }
      } else {
        for (int cc = 0; cc < nc; ++cc)
          for (int cr = 0; cr < nc; ++cr) {
            double acc = 0.0;
            for (int al = 0; al < mu; ++al) acc += fw[al] * sh_dfm(k, f, al, cr, cc) * tgg[al];
            u[(cc * q + layer) * m1 + cr * q + layer] -= b * acc;
          }
      }
    }
  }
  free(r1);
  free(r2);
}

/* ElementShuffled::apply_t_2d (ops/shuffled.hpp:149-234): v = Atilde^T u */
static void shuf_apply_t_2d(const shuf_ctx *k, const double *u, double *v) {
  const or_sys *S = k->s;
  const int q = S->q, mu = S->mu, nc = k->ncb, m1 = nc * q;
  const double a = k->a, b = k->b;
#define UU(cr, br, cc, dc) u[((cc) * q + (dc)) * m1 + (cr) * q + (br)]
  double *hgg = (double *)xcalloc((size_t)nc * nc * mu, sizeof(double));
  double *hdg = (double *)xcalloc((size_t)nc * nc * mu, sizeof(double));
  for (int cr = 0; cr < nc; ++cr)
    for (int cc = 0; cc < nc; ++cc)
      for (int be = 0; be < mu; ++be) {
        double sg = 0.0, sd = 0.0;
        for (int dc = 0; dc < q; ++dc) {
          double cg = 0.0, cd = 0.0;
          for (int br = 0; br < q; ++br) {
            cg += GM(be, br) * UU(cr, br, cc, dc);
            cd += DM(be, br) * UU(cr, br, cc, dc);
          }
          sg += GM(be, dc) * cg;
          sd += GM(be, dc) * cd;
        }
        hgg[(cr * nc + cc) * mu + be] = sg;
        hdg[(cr * nc + cc) * mu + be] = sd;
      }
  const double *jd = S->jdet + (size_t)k->e * mu * mu;
  double km[MAXQ], k1[MAXQ], k2[MAXQ];
  for (int al = 0; al < mu; ++al) km[al] = k1[al] = k2[al] = 0.0;
  for (int be = 0; be < mu; ++be) {
    const double wb = S->w[be];
    for (int al = 0; al < mu; ++al) {
      const int qv = be * mu + al;
      const double w = S->w[al] * wb;
      double smass = 0.0;
      for (int c = 0; c < nc; ++c) smass += hgg[(c * nc + c) * mu + be];
      km[al] += w * jd[qv] * smass;
      if (b != 0.0) {
        double s1 = 0.0, s2 = 0.0;
        for (int cr = 0; cr < nc; ++cr)
          for (int cc = 0; cc < nc; ++cc) {
            s1 += sh_dft(k, 0, qv, cr, cc) * hgg[(cr * nc + cc) * mu + be];
            s2 += sh_dft(k, 1, qv, cr, cc) * hdg[(cr * nc + cc) * mu + be];
          }
        k1[al] += w * s1;
        k2[al] += w * s2;
      }
    }
  }
  for (int ec = 0; ec < q; ++ec)
    for (int ar = 0; ar < q; ++ar) {
      double acc = 0.0;
      for (int al = 0; al < mu; ++al) {
        acc += GM(al, ar) * GM(al, ec) * (a * km[al] + b * k2[al]);
        acc += DM(al, ar) * GM(al, ec) * b * k1[al];
      }
      v[ec * q + ar] = acc;
    }
  if (b != 0.0) {
    for (int f = 0; f < 4; ++f) {
      const double *fw = S->face_w + ((size_t)k->e * 4 + f) * mu;
      const int layer = (f % 2) == 0 ? 0 : q - 1;
      if (f / 2 == 0) {
        double acc = 0.0;
        for (int be = 0; be < mu; ++be) {
          double sc = 0.0;
          for (int cr = 0; cr < nc; ++cr)
            for (int cc = 0; cc < nc; ++cc) sc += sh_dfm(k, f, be, cr, cc) * hgg[(cr * nc + cc) * mu + be];
          acc += fw[be] * sc;
        }
        v[layer * q + layer] -= b * acc;
      } else {
        for (int al = 0; al < mu; ++al) {
          double sc = 0.0;
          for (int cr = 0; cr < nc; ++cr)
            for (int cc = 0; cc < nc; ++cc) sc += sh_dfm(k, f, al, cr, cc) * UU(cr, layer, cc, layer);
          const double coef = b * fw[al] * sc;
          for (int ec = 0; ec < q; ++ec)
            for (int ar = 0; ar < q; ++ar) v[ec * q + ar] -= coef * GM(al, ar) * GM(al, ec);
        }
      }
    }
  }
#undef UU
  free(hgg);
  free(hdg);
}

/* ElementShuffled::apply_3d (ops/shuffled.hpp:238-367): u = Atilde v, O(p^5) */
static void shuf_apply_3d(const shuf_ctx *k, const double *v, double *u) {
  const or_sys *S = k->s;
  const int q = S->q, mu = S->mu, nc = k->ncb, m1 = nc * q, q2 = q * q;
  const double a = k->a, b = k->b;
#define VV(a1, a2, e1, e2) v[((size_t)(e2) * q + (e1)) * q2 + (a2) * q + (a1)]
  const size_t n4 = (size_t)mu * q * q * q;
  double *a1g = (double *)xcalloc(n4, sizeof(double));
  double *a1d = (double *)xcalloc(n4, sizeof(double));
  for (int al = 0; al < mu; ++al)
    for (int e2 = 0; e2 < q; ++e2)
      for (int e1 = 0; e1 < q; ++e1)
        for (int a2 = 0; a2 < q; ++a2) {
          double sg = 0.0, sd = 0.0;
          for (int ar = 0; ar < q; ++ar) {
            sg += GM(al, ar) * VV(ar, a2, e1, e2);
            sd += DM(al, ar) * VV(ar, a2, e1, e2);
          }
          const size_t idx = (((size_t)al * q + a2) * q + e1) * q + e2;
          a1g[idx] = sg;
          a1d[idx] = sd;
        }
  double *t4x = (double *)xcalloc((size_t)mu * mu, sizeof(double));
  double *t4y = (double *)xcalloc((size_t)mu * mu, sizeof(double));
  double *t4g = (double *)xcalloc((size_t)mu * mu, sizeof(double));
  for (int al = 0; al < mu; ++al)
    for (int be = 0; be < mu; ++be) {
      double sx = 0.0, sy = 0.0, sg = 0.0;
      for (int e2 = 0; e2 < q; ++e2)
        for (int e1 = 0; e1 < q; ++e1) {
          double cx = 0.0, cy = 0.0, cg = 0.0;
          for (int a2 = 0; a2 < q; ++a2) {
            const size_t idg = (((size_t)al * q + a2) * q + e1) * q + e2;
            cx += GM(be, a2) * a1d[idg];
            cy += DM(be, a2) * a1g[idg];
            cg += GM(be, a2) * a1g[idg];
          }
          const double gee = GM(al, e1) * GM(be, e2);
          sx += gee * cx;
          sy += gee * cy;
          sg += gee * cg;
        }
      t4x[al * mu + be] = sx;
      t4y[al * mu + be] = sy;
      t4g[al * mu + be] = sg;
    }
  const double *jd = S->jdet + (size_t)k->e * mu * mu * mu;
  double rm[MAXQ];
  double *r1 = (double *)xcalloc((size_t)nc * nc * mu, sizeof(double));
  double *r2 = (double *)xcalloc((size_t)nc * nc * mu, sizeof(double));
  double *r3 = (double *)xcalloc((size_t)nc * nc * mu, sizeof(double));
  for (int g = 0; g < mu; ++g) rm[g] = 0.0;
  for (int ga = 0; ga < mu; ++ga)
    for (int be = 0; be < mu; ++be)
      for (int al = 0; al < mu; ++al) {
        const int qv = (ga * mu + be) * mu + al;
        const double w = S->w[al] * S->w[be];
        rm[ga] += w * jd[qv] * t4g[al * mu + be];
        if (b != 0.0)
          for (int cr = 0; cr < nc; ++cr)
            for (int cc = 0; cc < nc; ++cc) {
              const size_t rc = ((size_t)cr * nc + cc) * mu + ga;
              r1[rc] += w * sh_dft(k, 0, qv, cr, cc) * t4x[al * mu + be];
              r2[rc] += w * sh_dft(k, 1, qv, cr, cc) * t4y[al * mu + be];
              r3[rc] += w * sh_dft(k, 2, qv, cr, cc) * t4g[al * mu + be];
            }
      }
  for (int cc = 0; cc < nc; ++cc)
    for (int d3 = 0; d3 < q; ++d3)
      for (int cr = 0; cr < nc; ++cr)
        for (int b3 = 0; b3 < q; ++b3) {
          double acc = 0.0;
          for (int ga = 0; ga < mu; ++ga) {
            const double wg = S->w[ga];
            double val = 0.0;
            if (cr == cc && a != 0.0) val += a * rm[ga];
            if (b != 0.0) val += b * (r1[(cr * nc + cc) * mu + ga] + r2[(cr * nc + cc) * mu + ga]);
            acc += wg * GM(ga, b3) * GM(ga, d3) * val;
            if (b != 0.0) acc += wg * DM(ga, b3) * GM(ga, d3) * b * r3[(cr * nc + cc) * mu + ga];
          }
          u[(cc * q + d3) * m1 + cr * q + b3] = acc;
        }
  if (b != 0.0) {
    double wbuf[MAXQ];
    for (int f = 0; f < 6; ++f) {
      const double *fw = S->face_w + ((size_t)k->e * 6 + f) * mu * mu;
      const int layer = (f % 2) == 0 ? 0 : q - 1;
      const int axis = f / 2;
      if (axis == 2) {
        for (int cc = 0; cc < nc; ++cc)
          for (int cr = 0; cr < nc; ++cr) {
            double acc = 0.0;
            for (int be = 0; be < mu; ++be)
              for (int al = 0; al < mu; ++al)
                acc += fw[be * mu + al] * sh_dfm(k, f, be * mu + al, cr, cc) * t4g[al * mu + be];
            u[(cc * q + layer) * m1 + cr * q + layer] -= b * acc;
          }
        continue;
      }
      for (int al = 0; al < mu; ++al) {
        double acc = 0.0;
        for (int ej = 0; ej < q; ++ej)
          for (int aj = 0; aj < q; ++aj) {
            const double vv = axis == 0 ? VV(layer, aj, layer, ej) : VV(aj, layer, ej, layer);
            acc += GM(al, ej) * GM(al, aj) * vv;
          }
        wbuf[al] = acc;
      }
      for (int cc = 0; cc < nc; ++cc)
        for (int d3 = 0; d3 < q; ++d3)
          for (int cr = 0; cr < nc; ++cr)
            for (int b3 = 0; b3 < q; ++b3) {
              double acc = 0.0;
              for (int be = 0; be < mu; ++be) {
                double inner = 0.0;
                for (int al = 0; al < mu; ++al) inner += fw[be * mu + al] * sh_dfm(k, f, be * mu + al, cr, cc) * wbuf[al];
                acc += GM(be, b3) * GM(be, d3) * inner;
              }
              u[(cc * q + d3) * m1 + cr * q + b3] -= b * acc;
            }
    }
  }
#undef VV
  free(a1g);
  free(a1d);
  free(t4x);
  free(t4y);
  free(t4g);
  free(r1);
  free(r2);
  free(r3);
}

/* ElementShuffled::apply_t_3d (ops/shuffled.hpp:369-503): v = Atilde^T u */
static void shuf_apply_t_3d(const shuf_ctx *k, const double *u, double *v) {
  const or_sys *S = k->s;
  const int q = S->q, mu = S->mu, nc = k->ncb, m1 = nc * q, q2 = q * q;
  const double a = k->a, b = k->b;
#define UU(cr, b3, cc, d3) u[((cc) * q + (d3)) * m1 + (cr) * q + (b3)]
  double *hgg = (double *)xcalloc((size_t)nc * nc * mu, sizeof(double));
  double *hdg = (double *)xcalloc((size_t)nc * nc * mu, sizeof(double));
  for (int cr = 0; cr < nc; ++cr)
    for (int cc = 0; cc < nc; ++cc)
      for (int ga = 0; ga < mu; ++ga) {
        double sg = 0.0, sd = 0.0;
        for (int d3 = 0; d3 < q; ++d3) {
          double cg = 0.0, cd = 0.0;
          for (int b3 = 0; b3 < q; ++b3) {
            cg += GM(ga, b3) * UU(cr, b3, cc, d3);
            cd += DM(ga, b3) * UU(cr, b3, cc, d3);
          }
          sg += GM(ga, d3) * cg;
          sd += GM(ga, d3) * cd;
        }
        hgg[(cr * nc + cc) * mu + ga] = sg;
        hdg[(cr * nc + cc) * mu + ga] = sd;
      }
  const double *jd = S->jdet + (size_t)k->e * mu * mu * mu;
  double *kx = (double *)xcalloc((size_t)mu * mu, sizeof(double));
  double *ky = (double *)xcalloc((size_t)mu * mu, sizeof(double));
  double *kg = (double *)xcalloc((size_t)mu * mu, sizeof(double));
  for (int ga = 0; ga < mu; ++ga) {
    const double wg = S->w[ga];
    for (int be = 0; be < mu; ++be)
      for (int al = 0; al < mu; ++al) {
        const int qv = (ga * mu + be) * mu + al;
        const double w = S->w[al] * S->w[be] * wg;
        double smass = 0.0;
        for (int c = 0; c < nc; ++c) smass += hgg[(c * nc + c) * mu + ga];
        kg[al * mu + be] += a * w * jd[qv] * smass;
        if (b != 0.0) {
          double s1 = 0.0, s2 = 0.0, s3 = 0.0;
          for (int cr = 0; cr < nc; ++cr)
            for (int cc = 0; cc < nc; ++cc) {
              const double hg = hgg[(cr * nc + cc) * mu + ga];
              const double hd = hdg[(cr * nc + cc) * mu + ga];
              s1 += sh_dft(k, 0, qv, cr, cc) * hg;
              s2 += sh_dft(k, 1, qv, cr, cc) * hg;
              s3 += sh_dft(k, 2, qv, cr, cc) * hd;
            }
          kx[al * mu + be] += b * w * s1;
          ky[al * mu + be] += b * w * s2;
          kg[al * mu + be] += b * w * s3;
        }
      }
  }
  if (b != 0.0)
    for (int f = 4; f < 6; ++f) {
      const double *fw = S->face_w + ((size_t)k->e * 6 + f) * mu * mu;
      const int layer = (f % 2) == 0 ? 0 : q - 1;
      for (int be = 0; be < mu; ++be)
        for (int al = 0; al < mu; ++al) {
          double sc = 0.0;
          for (int cr = 0; cr < nc; ++cr)
            for (int cc = 0; cc < nc; ++cc) sc += sh_dfm(k, f, be * mu + al, cr, cc) * UU(cr, layer, cc, layer);
          kg[al * mu + be] -= b * fw[be * mu + al] * sc;
        }
    }
  const size_t n3 = (size_t)mu * q * q;
  double *p1x = (double *)xcalloc(n3, sizeof(double));
  double *p1y = (double *)xcalloc(n3, sizeof(double));
  double *p1g = (double *)xcalloc(n3, sizeof(double));
  for (int al = 0; al < mu; ++al)
    for (int a2 = 0; a2 < q; ++a2)
      for (int e2 = 0; e2 < q; ++e2) {
        double sx = 0.0, sy = 0.0, sg = 0.0;
        for (int be = 0; be < mu; ++be) {
          const double ge2 = GM(be, e2);
          sx += GM(be, a2) * ge2 * kx[al * mu + be];
          sy += DM(be, a2) * ge2 * ky[al * mu + be];
          sg += GM(be, a2) * ge2 * kg[al * mu + be];
        }
        const size_t idx = ((size_t)al * q + a2) * q + e2;
        p1x[idx] = sx;
        p1y[idx] = sy;
        p1g[idx] = sg;
      }
  for (int e2 = 0; e2 < q; ++e2)
    for (int e1 = 0; e1 < q; ++e1)
      for (int a2 = 0; a2 < q; ++a2)
        for (int a1 = 0; a1 < q; ++a1) {
          double acc = 0.0;
          for (int al = 0; al < mu; ++al) {
            const double ge1 = GM(al, e1);
            const size_t idx = ((size_t)al * q + a2) * q + e2;
            acc += DM(al, a1) * ge1 * p1x[idx];
            acc += GM(al, a1) * ge1 * (p1y[idx] + p1g[idx]);
          }
          v[((size_t)e2 * q + e1) * q2 + a2 * q + a1] = acc;
        }
  if (b != 0.0) {
    double lbuf[MAXQ];
    for (int f = 0; f < 4; ++f) {
      const double *fw = S->face_w + ((size_t)k->e * 6 + f) * mu * mu;
      const int layer = (f % 2) == 0 ? 0 : q - 1;
      const int axis = f / 2;
      for (int al = 0; al < mu; ++al) {
        double acc = 0.0;
        for (int be = 0; be < mu; ++be) {
          double sc = 0.0;
          for (int cr = 0; cr < nc; ++cr)
            for (int cc = 0; cc < nc; ++cc) sc += sh_dfm(k, f, be * mu + al, cr, cc) * hgg[(cr * nc + cc) * mu + be];
          acc += fw[be * mu + al] * sc;
        }
        lbuf[al] = acc;
      }
      for (int ej = 0; ej < q; ++ej)
        for (int aj = 0; aj < q; ++aj) {
          double acc = 0.0;
          for (int al = 0; al < mu; ++al) acc += GM(al, aj) * GM(al, ej) * lbuf[al];
          if (axis == 0)
            v[((size_t)ej * q + layer) * q2 + aj * q + layer] -= b * acc;
          else
            v[((size_t)layer * q + ej) * q2 + layer * q + aj] -= b * acc;
        }
    }
  }
#undef UU
  free(hgg);
  free(hdg);
  free(kx);
  free(ky);
  free(kg);
  free(p1x);
  free(p1y);
  free(p1g);
}
#undef GM
#undef DM

void or_shuffled(const or_sys *s, int e, double a, double b, int small_mode, int comp, int transpose,
                 const double *in, double *out) {
  shuf_ctx k = {s, e, small_mode, comp, small_mode ? 1 : s->n_c, a, b};
  if (s->dim == 2) {
    if (transpose) shuf_apply_t_2d(&k, in, out); else shuf_apply_2d(&k, in, out);
  } else {
    if (transpose) shuf_apply_t_3d(&k, in, out); else shuf_apply_3d(&k, in, out);
  }
}

/* ======================================================================
 * Small dense linear algebra (tensor/small_matrix.hpp, schur.hpp, sylvester.hpp,
 * svd_small.hpp).
 * ====================================================================== */
static double inf_norm(int rows, int cols, const double *a) {
  double m = 0.0;
  for (int i = 0; i < rows; ++i) {
    double s = 0.0;
    for (int j = 0; j < cols; ++j) s += fabs(a[i * cols + j]);
    m = fmax(m, s);
  }
  return m;
}

/* LuFactor ctor (tensor/small_matrix.hpp:143-172) */
int or_lu_factor(int n, const double *a, double *lu, int *perm) {
  memcpy(lu, a, sizeof(double) * (size_t)n * n);
  const double tol = 1e-14 * fmax(inf_norm(n, n, a), 1e-300);
  for (int i = 0; i < n; ++i) perm[i] = i;
  for (int k = 0; k < n; ++k) {
    int piv = k;
    double best = fabs(lu[k * n + k]);
    for (int i = k + 1; i < n; ++i) {
      const double v = fabs(lu[i * n + k]);
      if (v > best) {
        best = v;
        piv = i;
      }
    }
    if (best < tol) return OR_SINGULAR;
    if (piv != k) {
      for (int j = 0; j < n; ++j) {
        const double t = lu[k * n + j];
        lu[k * n + j] = lu[piv * n + j];
        lu[piv * n + j] = t;
      }
      const int t = perm[k];
      perm[k] = perm[piv];
      perm[piv] = t;
    }
    const double inv = 1.0 / lu[k * n + k];
    for (int i = k + 1; i < n; ++i) {
      const double m = lu[i * n + k] * inv;
      lu[i * n + k] = m;
      for (int j = k + 1; j < n; ++j) lu[i * n + j] -= m * lu[k * n + j];
    }
  }
  return OR_OK;
}

/* LuFactor::solve (tensor/small_matrix.hpp:177-187) */
void or_lu_solve(int n, const double *lu, const int *perm, const double *b, double *x) {
  for (int i = 0; i < n; ++i) x[i] = b[perm[i]];
  for (int i = 0; i < n; ++i)
    for (int j = 0; j < i; ++j) x[i] -= lu[i * n + j] * x[j];
  for (int i = n - 1; i >= 0; --i) {
    for (int j = i + 1; j < n; ++j) x[i] -= lu[i * n + j] * x[j];
    x[i] /= lu[i * n + i];
  }
}

static void rot_left(double *m, int n, int i, int j, double c, double s, int lo, int hi) {
  for (int k = lo; k < hi; ++k) {
    const double x = m[i * n + k], y = m[j * n + k];
    m[i * n + k] = c * x + s * y;
    m[j * n + k] = -s * x + c * y;
  }
}
static void rot_right(double *m, int n, int i, int j, double c, double s, int lo, int hi) {
  for (int k = lo; k < hi; ++k) {
    const double x = m[k * n + i], y = m[k * n + j];
    m[k * n + i] = c * x + s * y;
    m[k * n + j] = -s * x + c * y;
  }
}

/* hessenberg (tensor/schur.hpp:38-79) */
static void hessenberg(int n, double *h, double *q) {
  double v[MAXQ * 2];
  for (int k = 0; k + 2 < n; ++k) {
    double norm = 0.0;
    for (int i = k + 1; i < n; ++i) norm += h[i * n + k] * h[i * n + k];
    norm = sqrt(norm);
    if (norm == 0.0) continue;
    const double alpha = h[(k + 1) * n + k] >= 0.0 ? -norm : norm;
    double vn2 = 0.0;
    for (int i = k + 1; i < n; ++i) {
      v[i] = h[i * n + k];
      if (i == k + 1) v[i] -= alpha;
      vn2 += v[i] * v[i];
    }
    if (vn2 == 0.0) continue;
    const double beta = 2.0 / vn2;
    for (int j = k; j < n; ++j) {
      double dot = 0.0;
      for (int i = k + 1; i < n; ++i) dot += v[i] * h[i * n + j];
      dot *= beta;
      for (int i = k + 1; i < n; ++i) h[i * n + j] -= dot * v[i];
    }
    for (int i = 0; i < n; ++i) {
      double dot = 0.0;
      for (int j = k + 1; j < n; ++j) dot += h[i * n + j] * v[j];
      dot *= beta;
      for (int j = k + 1; j < n; ++j) h[i * n + j] -= dot * v[j];
    }
    for (int i = 0; i < n; ++i) {
      double dot = 0.0;
      for (int j = k + 1; j < n; ++j) dot += q[i * n + j] * v[j];
      dot *= beta;
      for (int j = k + 1; j < n; ++j) q[i * n + j] -= dot * v[j];
    }
    for (int i = k + 2; i < n; ++i) h[i * n + k] = 0.0;
    h[(k + 1) * n + k] = alpha;
  }
}

/* standardize_2x2 (tensor/schur.hpp:86-113) */
static void standardize_2x2(int n, double *h, double *q, int l) {
  const double a = h[l * n + l], b = h[l * n + l + 1], c = h[(l + 1) * n + l], d = h[(l + 1) * n + l + 1];
  if (c == 0.0) return;
  const double th1 = 0.5 * atan2(d - a, b + c);
  double cc = cos(th1), ss = sin(th1);
  const double bt = cc * cc * b - ss * ss * c + cc * ss * (d - a);
  const double ct = cc * cc * c - ss * ss * b + cc * ss * (d - a);
  const int real_pair = bt * ct >= 0.0;
  double th = th1;
  if (real_pair) {
    double th2;
    if (bt == 0.0)
      th2 = (ct == 0.0) ? 0.0 : 2.0 * atan(1.0);
    else
      th2 = atan(sqrt(ct / bt));
    th += th2;
  }
  cc = cos(th);
  ss = sin(th);
  rot_left(h, n, l, l + 1, cc, ss, 0, n);
  rot_right(h, n, l, l + 1, cc, ss, 0, n);
  rot_right(q, n, l, l + 1, cc, ss, 0, n);
  if (real_pair) h[(l + 1) * n + l] = 0.0;
}

/* real_schur (tensor/schur.hpp:119-232) */
int or_real_schur(int n, const double *cin, double *q, double *h) {
  memcpy(h, cin, sizeof(double) * (size_t)n * n);
  for (int i = 0; i < n * n; ++i) q[i] = 0.0;
  for (int i = 0; i < n; ++i) q[i * n + i] = 1.0;
  for (int i = 0; i < n * n; ++i)
    if (!isfinite(cin[i])) return OR_SHAPE;
  if (n == 1) return OR_OK;
  hessenberg(n, h, q);
  const double eps = 2.3e-16;
  const double hnorm = fmax(inf_norm(n, n, h), 1e-300);
  int m = n - 1, iter = 0, total = 0;
  const int budget = 60 * n;
  double v[3];
#define H(i, j) h[(i) * n + (j)]
  while (m >= 0) {
    if (++total > budget) return OR_CONVERGENCE;
    int l = m;
    while (l > 0) {
      const double s = fabs(H(l - 1, l - 1)) + fabs(H(l, l));
      if (fabs(H(l, l - 1)) <= eps * fmax(s, hnorm)) {
        H(l, l - 1) = 0.0;
        break;
      }
      --l;
    }
    if (l == m) {
      m -= 1;
      iter = 0;
      continue;
    }
    if (l == m - 1) {
      standardize_2x2(n, h, q, l);
      m -= 2;
      iter = 0;
      continue;
    }
    ++iter;
    double x, y, z;
    if (iter % 11 == 0) {
      const double s = fabs(H(m, m - 1)) + fabs(H(m - 1, m - 2));
      const double sh = H(m, m) + 0.75 * s;
      const double tdet = sh * sh - 0.4375 * s * s;
      x = H(l, l) * H(l, l) + H(l, l + 1) * H(l + 1, l) - 2.0 * sh * H(l, l) + tdet;
      y = H(l + 1, l) * (H(l, l) + H(l + 1, l + 1) - 2.0 * sh);
      z = (l + 2 <= m) ? H(l + 1, l) * H(l + 2, l + 1) : 0.0;
    } else {
      const double tr = H(m - 1, m - 1) + H(m, m);
      const double det = H(m - 1, m - 1) * H(m, m) - H(m - 1, m) * H(m, m - 1);
      x = H(l, l) * H(l, l) + H(l, l + 1) * H(l + 1, l) - tr * H(l, l) + det;
      y = H(l + 1, l) * (H(l, l) + H(l + 1, l + 1) - tr);
      z = (l + 2 <= m) ? H(l + 1, l) * H(l + 2, l + 1) : 0.0;
    }
    for (int k = l; k <= m - 1; ++k) {
      const int len = (k + 2 <= m) ? 3 : 2;
      v[0] = x;
      v[1] = y;
      v[2] = (len == 3) ? z : 0.0;
      double nrm = 0.0;
      for (int i = 0; i < len; ++i) nrm += v[i] * v[i];
      nrm = sqrt(nrm);
      if (nrm != 0.0) {
        const double alpha = v[0] >= 0.0 ? -nrm : nrm;
        v[0] -= alpha;
        double vn2 = 0.0;
        for (int i = 0; i < len; ++i) vn2 += v[i] * v[i];
        if (vn2 != 0.0) {
          const double beta = 2.0 / vn2;
          const int row_hi = (k + len < n) ? k + len : n;
          const int col_lo = (k > l) ? k - 1 : l;
          for (int j = col_lo; j < n; ++j) {
            double dot = 0.0;
            for (int i = 0; i < len; ++i) dot += v[i] * H(k + i, j);
            dot *= beta;
            for (int i = 0; i < len; ++i) H(k + i, j) -= dot * v[i];
          }
          const int row_top = ((m < k + len) ? m : k + len) + 1;
          for (int i = 0; i < row_top; ++i) {
            double dot = 0.0;
            for (int j = k; j < row_hi; ++j) dot += H(i, j) * v[j - k];
            dot *= beta;
            for (int j = k; j < row_hi; ++j) H(i, j) -= dot * v[j - k];
          }
          for (int i = 0; i < n; ++i) {
            double dot = 0.0;
            for (int j = k; j < row_hi; ++j) dot += q[i * n + j] * v[j - k];
            dot *= beta;
            for (int j = k; j < row_hi; ++j) q[i * n + j] -= dot * v[j - k];
          }
        }
      }
      x = H(k + 1, k);
      if (k + 2 <= m) y = H(k + 2, k);
      if (k + 3 <= m) z = H(k + 3, k);
    }
    for (int i = l + 2; i <= m; ++i)
      for (int j = l; j <= i - 2; ++j) H(i, j) = 0.0;
  }
  for (int l = 0; l + 1 < n; ++l)
    if (H(l + 1, l) != 0.0) standardize_2x2(n, h, q, l);
#undef H
  return OR_OK;
}

/* quasi_triangular_eigenvalues (tensor/schur.hpp:235-266); returns count */
static int quasi_eigs(int n, const double *t, double *re, double *im) {
  int i = 0, k = 0;
  while (i < n) {
    if (i + 1 < n && t[(i + 1) * n + i] != 0.0) {
      const double a = t[i * n + i], b = t[i * n + i + 1], c = t[(i + 1) * n + i], d = t[(i + 1) * n + i + 1];
      const double tr = 0.5 * (a + d);
      const double disc = tr * tr - (a * d - b * c);
      if (disc >= 0.0) {
        const double sq = sqrt(disc);
        re[k] = tr + sq; im[k++] = 0.0;
        re[k] = tr - sq; im[k++] = 0.0;
      } else {
        const double sq = sqrt(-disc);
        re[k] = tr; im[k++] = sq;
        re[k] = tr; im[k++] = -sq;
      }
      i += 2;
    } else {
      re[k] = t[i * n + i];
      im[k++] = 0.0;
      ++i;
    }
  }
  return k;
}

/* check_sylvester_pair (precond/ksvd.hpp:61-73) */
static int check_sylvester_pair(int n1, const double *t1, int n2, const double *t2) {
  double re1[2 * MAXQ], im1[2 * MAXQ], re2[2 * MAXQ], im2[2 * MAXQ];
  const int k1 = quasi_eigs(n1, t1, re1, im1), k2 = quasi_eigs(n2, t2, re2, im2);
  const double scale = inf_norm(n1, n1, t1) + inf_norm(n2, n2, t2);
  for (int i = 0; i < k1; ++i)
    for (int j = 0; j < k2; ++j) {
      const double re = re1[i] + re2[j], im = im1[i] + im2[j];
      if (sqrt(re * re + im * im) < 1e-12 * fmax(scale, 1e-300)) return OR_SINGULAR;
    }
  return OR_OK;
}

/* solve_tiny<4> (tensor/sylvester.hpp:34-59) */
static int solve_tiny(double a[4][4], double bv[4], int n, double tol) {
  for (int k = 0; k < n; ++k) {
    int piv = k;
    for (int i = k + 1; i < n; ++i)
      if (fabs(a[i][k]) > fabs(a[piv][k])) piv = i;
    if (fabs(a[piv][k]) < tol) return OR_SINGULAR;
    if (piv != k) {
      for (int j = 0; j < 4; ++j) {
        const double t = a[piv][j];
        a[piv][j] = a[k][j];
        a[k][j] = t;
      }
      const double t = bv[piv];
      bv[piv] = bv[k];
      bv[k] = t;
    }
    const double inv = 1.0 / a[k][k];
    for (int i = k + 1; i < n; ++i) {
      const double m = a[i][k] * inv;
      if (m == 0.0) continue;
      for (int j = k; j < n; ++j) a[i][j] -= m * a[k][j];
      bv[i] -= m * bv[k];
    }
  }
  for (int i = n - 1; i >= 0; --i) {
    for (int j = i + 1; j < n; ++j) bv[i] -= a[i][j] * bv[j];
    bv[i] /= a[i][i];
  }
  return OR_OK;
}

static int quasi_blocks(int n, const double *t, int *start, int *size) {
  int i = 0, nb = 0;
  while (i < n) {
    if (i + 1 < n && t[(i + 1) * n + i] != 0.0) {
      start[nb] = i; size[nb++] = 2; i += 2;
    } else {
      start[nb] = i; size[nb++] = 1; ++i;
    }
  }
  return nb;
}

/* sylvester_solve (tensor/sylvester.hpp:72-127): T1 X + X T2^T = B */
int or_sylvester(int n1, int n2, const double *t1, const double *t2, const double *bm, double *x) {
  int s1[2 * MAXQ], z1[2 * MAXQ], s2[2 * MAXQ], z2[2 * MAXQ];
  const int nb1 = quasi_blocks(n1, t1, s1, z1), nb2 = quasi_blocks(n2, t2, s2, z2);
  const double tol = 1e-14 * fmax(inf_norm(n1, n1, t1) + inf_norm(n2, n2, t2), 1e-300);
  double *r = (double *)xcalloc((size_t)2 * n2, sizeof(double));
  for (int i = 0; i < n1 * n2; ++i) x[i] = 0.0;
  for (int bi = nb1 - 1; bi >= 0; --bi) {
    const int i0 = s1[bi], isz = z1[bi];
    for (int a = 0; a < isz; ++a)
      for (int k = 0; k < n2; ++k) {
        double s = bm[(i0 + a) * n2 + k];
        for (int j = i0 + isz; j < n1; ++j) s -= t1[(i0 + a) * n1 + j] * x[j * n2 + k];
        r[a * n2 + k] = s;
      }
    for (int bj = nb2 - 1; bj >= 0; --bj) {
      const int k0 = s2[bj], ksz = z2[bj];
      for (int a = 0; a < isz; ++a)
        for (int kb = 0; kb < ksz; ++kb) {
          double s = r[a * n2 + k0 + kb];
          for (int l = k0 + ksz; l < n2; ++l) s -= t2[(k0 + kb) * n2 + l] * x[(i0 + a) * n2 + l];
          r[a * n2 + k0 + kb] = s;
        }
      double mm[4][4] = {{0}}, rhs[4] = {0};
      for (int a = 0; a < isz; ++a)
        for (int kb = 0; kb < ksz; ++kb) {
          const int row = a * ksz + kb;
          rhs[row] = r[a * n2 + k0 + kb];
          for (int a2 = 0; a2 < isz; ++a2)
            for (int kb2 = 0; kb2 < ksz; ++kb2) {
              double coef = 0.0;
              if (kb == kb2) coef += t1[(i0 + a) * n1 + i0 + a2];
              if (a == a2) coef += t2[(k0 + kb) * n2 + k0 + kb2];
              mm[row][a2 * ksz + kb2] = coef;
            }
        }
      if (solve_tiny(mm, rhs, isz * ksz, tol) != OR_OK) {
        free(r);
        return OR_SINGULAR;
      }
      for (int a = 0; a < isz; ++a)
        for (int kb = 0; kb < ksz; ++kb) x[(i0 + a) * n2 + k0 + kb] = rhs[a * ksz + kb];
    }
  }
  free(r);
  return OR_OK;
}

/* svd_small (tensor/svd_small.hpp:20-84): one-sided Jacobi; u m x k, v n x k, k = min(m,n) */
void or_svd_small(int m, int n, const double *a, double *u, double *sigma, double *v) {
  if (m < n) {
    double *at = (double *)xcalloc((size_t)m * n, sizeof(double));
    for (int i = 0; i < m; ++i)
      for (int j = 0; j < n; ++j) at[j * m + i] = a[i * n + j];
    or_svd_small(n, m, at, v, sigma, u);
    free(at);
    return;
  }
  double *w = (double *)xcalloc((size_t)m * n, sizeof(double));
  double *vv = (double *)xcalloc((size_t)n * n, sizeof(double));
  memcpy(w, a, sizeof(double) * (size_t)m * n);
  for (int i = 0; i < n; ++i) vv[i * n + i] = 1.0;
  double scale = 0.0;
  for (int i = 0; i < m * n; ++i) scale = fmax(scale, fabs(a[i]));
  scale = fmax(scale, 1e-300);
  const double tol = 1e-14;
  for (int sweep = 0; sweep < 60; ++sweep) {
    int rotated = 0;
    for (int p = 0; p < n - 1; ++p)
      for (int qq = p + 1; qq < n; ++qq) {
        double app = 0.0, aqq = 0.0, apq = 0.0;
        for (int i = 0; i < m; ++i) {
          app += w[i * n + p] * w[i * n + p];
          aqq += w[i * n + qq] * w[i * n + qq];
          apq += w[i * n + p] * w[i * n + qq];
        }
        if (fabs(apq) <= tol * scale * scale) continue;
        rotated = 1;
        const double zeta = (aqq - app) / (2.0 * apq);
        const double t = copysign(1.0, zeta) / (fabs(zeta) + sqrt(1.0 + zeta * zeta));
        const double c = 1.0 / sqrt(1.0 + t * t);
        const double s = c * t;
        for (int i = 0; i < m; ++i) {
          const double wp = w[i * n + p], wq = w[i * n + qq];
          w[i * n + p] = c * wp - s * wq;
          w[i * n + qq] = s * wp + c * wq;
        }
        for (int i = 0; i < n; ++i) {
          const double vp = vv[i * n + p], vq = vv[i * n + qq];
          vv[i * n + p] = c * vp - s * vq;
          vv[i * n + qq] = s * vp + c * vq;
        }
      }
    if (!rotated) break;
  }
  double sig[4 * MAXQ];
  int order[4 * MAXQ];
  for (int j = 0; j < n; ++j) {
    double s = 0.0;
    for (int i = 0; i < m; ++i) s += w[i * n + j] * w[i * n + j];
    sig[j] = sqrt(s);
    order[j] = j;
  }
  /* descending; insertion sort is what libstdc++ std::sort does for n <= 16 and
   * agrees with it for distinct values at any n */
  for (int i = 1; i < n; ++i) {
    const int key = order[i];
    int j = i - 1;
    while (j >= 0 && sig[key] > sig[order[j]]) {
      order[j + 1] = order[j];
      --j;
    }
    order[j + 1] = key;
  }
  for (int k = 0; k < n; ++k) {
    const int j = order[k];
    sigma[k] = sig[j];
    const double inv = sig[j] > 0.0 ? 1.0 / sig[j] : 0.0;
    for (int i = 0; i < m; ++i) u[i * n + k] = w[i * n + j] * inv;
    for (int i = 0; i < n; ++i) v[i * n + k] = vv[i * n + j];
  }
  free(w);
  free(vv);
}

/* ======================================================================
 * Lanczos KSVD (tensor/lanczos.hpp:85-190).
 * ====================================================================== */
typedef struct {
  int m1, n1, m2, n2;
  void (*apply)(const void *ctx, const double *x, double *y);
  void (*apply_t)(const void *ctx, const double *x, double *y);
  const void *ctx;
} lz_op;

static double norm2(const double *v, long n) {
  double s = 0.0;
  for (long i = 0; i < n; ++i) s += v[i] * v[i];
  return sqrt(s);
}

static void reorthogonalize(double *r, long n, double *const *basis, int nb) {
  for (int pass = 0; pass < 2; ++pass)
    for (int j = 0; j < nb; ++j) {
      double dot = 0.0;
      for (long i = 0; i < n; ++i) dot += basis[j][i] * r[i];
      for (long i = 0; i < n; ++i) r[i] -= dot * basis[j][i];
    }
}

/* factors out: r terms x (A: m1 x n1, B: m2 x n2); sigma out: r values */
static void lanczos_ksvd(const lz_op *op, int r, int max_iter, double breakdown, const double *start, double *fa,
                         double *fb, double *sig_out, int *iters_out) {
  const long nrows = (long)op->m1 * op->n1, ncols = (long)op->m2 * op->n2;
  for (long i = 0; i < (long)r * nrows; ++i) fa[i] = 0.0;
  for (long i = 0; i < (long)r * ncols; ++i) fb[i] = 0.0;
  for (int j = 0; j < r; ++j) sig_out[j] = 0.0;
  double **vs = (double **)xcalloc((size_t)max_iter + 2, sizeof(double *));
  double **us = (double **)xcalloc((size_t)max_iter + 2, sizeof(double *));
  double *alphas = (double *)xcalloc((size_t)max_iter + 2, sizeof(double));
  double *betas = (double *)xcalloc((size_t)max_iter + 2, sizeof(double));
  int nv = 0, nu = 0, na = 0, nbeta = 0;
  vs[nv] = (double *)xcalloc((size_t)ncols, sizeof(double));
  memcpy(vs[nv++], start, sizeof(double) * (size_t)ncols);
  double *work = (double *)xcalloc((size_t)nrows, sizeof(double));
  op->apply(op->ctx, vs[0], work);
  double alpha = norm2(work, nrows);
  const double tol = breakdown * fmax(alpha, 1e-300);
  if (alpha < 1e-300) {
    *iters_out = 0;
    free(work);
    free(vs[0]);
    free(vs); free(us); free(alphas); free(betas);
    return;
  }
  for (long i = 0; i < nrows; ++i) work[i] /= alpha;
  us[nu++] = work;
  alphas[na++] = alpha;
  int iters = 1;
  double *p = (double *)xcalloc((size_t)ncols, sizeof(double));
  double *rv = (double *)xcalloc((size_t)nrows, sizeof(double));
  while (na < max_iter) {
    op->apply_t(op->ctx, us[nu - 1], p);
    for (long i = 0; i < ncols; ++i) p[i] -= alphas[na - 1] * vs[nv - 1][i];
    reorthogonalize(p, ncols, vs, nv);
    const double beta = norm2(p, ncols);
    ++iters;
    if (beta < tol) break;
    for (long i = 0; i < ncols; ++i) p[i] /= beta;
    vs[nv] = (double *)xcalloc((size_t)ncols, sizeof(double));
    memcpy(vs[nv++], p, sizeof(double) * (size_t)ncols);
    betas[nbeta++] = beta;
    op->apply(op->ctx, vs[nv - 1], rv);
    for (long i = 0; i < nrows; ++i) rv[i] -= beta * us[nu - 1][i];
    reorthogonalize(rv, nrows, us, nu);
    alpha = norm2(rv, nrows);
    if (alpha < tol) break;
    for (long i = 0; i < nrows; ++i) rv[i] /= alpha;
    us[nu] = (double *)xcalloc((size_t)nrows, sizeof(double));
    memcpy(us[nu++], rv, sizeof(double) * (size_t)nrows);
    alphas[na++] = alpha;
  }
  const int ku = nu, kv = nv;
  double *bm = (double *)xcalloc((size_t)ku * kv, sizeof(double));
  for (int i = 0; i < ku; ++i) {
    bm[i * kv + i] = alphas[i];
    if (i + 1 < kv && i < nbeta) bm[i * kv + i + 1] = betas[i];
  }
  const int k = ku < kv ? ku : kv;
  double *bu = (double *)xcalloc((size_t)ku * k, sizeof(double));
  double *bs = (double *)xcalloc((size_t)k, sizeof(double));
  double *bv = (double *)xcalloc((size_t)kv * k, sizeof(double));
  or_svd_small(ku, kv, bm, bu, bs, bv);
  for (int j = 0; j < r; ++j) {
    if (j < k && bs[j] > 0.0) {
      sig_out[j] = bs[j];
      const double scale = sqrt(bs[j]);
      for (long i = 0; i < nrows; ++i) {
        double s = 0.0;
        for (int l = 0; l < ku; ++l) s += us[l][i] * bu[l * k + j];
        fa[(long)j * nrows + (i % op->m1) * op->n1 + i / op->m1] = scale * s;
      }
      for (long i = 0; i < ncols; ++i) {
        double s = 0.0;
        for (int l = 0; l < kv; ++l) s += vs[l][i] * bv[l * k + j];
        fb[(long)j * ncols + (i % op->m2) * op->n2 + i / op->m2] = scale * s;
      }
    }
  }
  *iters_out = iters;
  for (int i = 0; i < nv; ++i) free(vs[i]);
  for (int i = 0; i < nu; ++i) free(us[i]);
  free(vs); free(us); free(alphas); free(betas);
  free(p); free(rv); free(bm); free(bu); free(bs); free(bv);
}

static void elem_apply_cb(const void *ctx, const double *x, double *y) {
  const shuf_ctx *k = (const shuf_ctx *)ctx;
  if (k->s->dim == 2) shuf_apply_2d(k, x, y); else shuf_apply_3d(k, x, y);
}
static void elem_apply_t_cb(const void *ctx, const double *x, double *y) {
  const shuf_ctx *k = (const shuf_ctx *)ctx;
  if (k->s->dim == 2) shuf_apply_t_2d(k, x, y); else shuf_apply_t_3d(k, x, y);
}

typedef struct {
  int rows, cols;
  const double *m;
} dense_ctx;
/* matvec / matvec_transpose (tensor/small_matrix.hpp:116-135) */
static void dense_apply_cb(const void *ctx, const double *x, double *y) {
  const dense_ctx *d = (const dense_ctx *)ctx;
  for (int i = 0; i < d->rows; ++i) {
    double s = 0.0;
    for (int j = 0; j < d->cols; ++j) s += d->m[(long)i * d->cols + j] * x[j];
    y[i] = s;
  }
}
static void dense_apply_t_cb(const void *ctx, const double *x, double *y) {
  const dense_ctx *d = (const dense_ctx *)ctx;
  for (int j = 0; j < d->cols; ++j) y[j] = 0.0;
  for (int i = 0; i < d->rows; ++i) {
    const double xi = x[i];
    for (int j = 0; j < d->cols; ++j) y[j] += d->m[(long)i * d->cols + j] * xi;
  }
}

/* ======================================================================
 * KSVD preconditioner: form (precond/ksvd.hpp:252-372) and apply (:112-233).
 * ====================================================================== */
struct or_pc {
  int dim, n_c, q, small_mode, nblk, n1, nb, ncc; /* 2D: n1 x q; 3D: n1 x q x q */
  int blk_len;       /* unknowns per block */
  int flen;          /* doubles per factor record */
  double *fac;       /* raw factors per block */
  double *lu;        /* 2D: lu(a2) n1^2, lu(b1) q^2 ; 3D: lu(a1) n1^2, lu(b2), lu(c1) q^2 */
  int *perm;
  double *sq;        /* q1 (s1 dim^2), t1, q2, t2 */
  int s1n, s2n;
  int *has;
  double **fb_lu;
  int **fb_perm;
  int nfb;
  int64_t *fb_list;
};

static int pc_lu_len(const or_pc *pc) { return pc->dim == 2 ? pc->n1 * pc->n1 + pc->q * pc->q : pc->n1 * pc->n1 + 2 * pc->q * pc->q; }
static int pc_perm_len(const or_pc *pc) { return pc->dim == 2 ? pc->n1 + pc->q : pc->n1 + 2 * pc->q; }
static int pc_sq_len(const or_pc *pc) { return 2 * pc->s1n * pc->s1n + 2 * pc->s2n * pc->s2n; }

/* lu_solve_matrix (precond/ksvd.hpp:48-57) */
static void lu_solve_matrix(int n, const double *lu, const int *perm, int cols, const double *rhs, double *x) {
  double col[4 * MAXQ], sol[4 * MAXQ];
  for (int j = 0; j < cols; ++j) {
    for (int i = 0; i < n; ++i) col[i] = rhs[i * cols + j];
    or_lu_solve(n, lu, perm, col, sol);
    for (int i = 0; i < n; ++i) x[i * cols + j] = sol[i];
  }
}

/* make_factors_2d (precond/ksvd.hpp:75-89); writes lu/perm/sq of one block */
static int make_factors_2d(int n1, int n2, const double *a1, const double *b1, const double *a2, const double *b2,
                           double *lu, int *perm, double *sq) {
  double *lua2 = lu, *lub1 = lu + n1 * n1;
  int *pa2 = perm, *pb1 = perm + n1;
  if (or_lu_factor(n1, a2, lua2, pa2) != OR_OK) return OR_SINGULAR;
  if (or_lu_factor(n2, b1, lub1, pb1) != OR_OK) return OR_SINGULAR;
  double *c1 = (double *)xcalloc((size_t)n1 * n1, sizeof(double));
  double *c2 = (double *)xcalloc((size_t)n2 * n2, sizeof(double));
  lu_solve_matrix(n1, lua2, pa2, n1, a1, c1);
  lu_solve_matrix(n2, lub1, pb1, n2, b2, c2);
  double *q1 = sq, *t1 = sq + n1 * n1, *q2 = sq + 2 * n1 * n1, *t2 = q2 + n2 * n2;
  int st = or_real_schur(n1, c1, q1, t1);
  if (st == OR_OK) st = or_real_schur(n2, c2, q2, t2);
  /* NOTE: the reference lets ConvergenceError escape (process abort);
   * here a non-converged Schur form is routed to the same fallback as SingularError. */
  if (st == OR_OK) st = check_sylvester_pair(n1, t1, n2, t2);
  free(c1);
  free(c2);
  return st == OR_OK ? OR_OK : OR_SINGULAR;
}

/* make_factors_3d (precond/ksvd.hpp:91-108) */
static int make_factors_3d(int n1, int q, const double *a1, const double *b1, const double *c1, const double *b2,
                           const double *c2, double *lu, int *perm, double *sq) {
  double *lua1 = lu, *lub2 = lu + n1 * n1, *luc1 = lub2 + q * q;
  int *pa1 = perm, *pb2 = perm + n1, *pc1 = pb2 + q;
  if (or_lu_factor(n1, a1, lua1, pa1) != OR_OK) return OR_SINGULAR;
  if (or_lu_factor(q, b2, lub2, pb2) != OR_OK) return OR_SINGULAR;
  if (or_lu_factor(q, c1, luc1, pc1) != OR_OK) return OR_SINGULAR;
  double *g1 = (double *)xcalloc((size_t)q * q, sizeof(double));
  double *g2 = (double *)xcalloc((size_t)q * q, sizeof(double));
  lu_solve_matrix(q, lub2, pb2, q, b1, g1);
  lu_solve_matrix(q, luc1, pc1, q, c2, g2);
  double *q1 = sq, *t1 = sq + q * q, *q2 = sq + 2 * q * q, *t2 = q2 + q * q;
  int st = or_real_schur(q, g1, q1, t1);
  if (st == OR_OK) st = or_real_schur(q, g2, q2, t2);
  if (st == OR_OK) st = check_sylvester_pair(q, t1, q, t2);
  free(g1);
  free(g2);
  return st == OR_OK ? OR_OK : OR_SINGULAR;
}

static void set_identity(int n, double *m) {
  for (int i = 0; i < n * n; ++i) m[i] = 0.0;
  for (int i = 0; i < n; ++i) m[i * n + i] = 1.0;
}

/* shuffle_dense (tensor/shuffle.hpp:16-25) */
static void shuffle_dense(const double *a, int m1, int n1, int m2, int n2, double *t) {
  for (int i = 0; i < m1; ++i)
    for (int j = 0; j < n1; ++j)
      for (int r = 0; r < m2; ++r)
        for (int c = 0; c < n2; ++c)
          t[(long)(j * m1 + i) * (m2 * n2) + c * m2 + r] = a[(long)(i * m2 + r) * (n1 * n2) + j * n2 + c];
}

or_pc *or_form_ksvd(const or_sys *s, double a, double b, int small_mode, int terms, const double *start_vec,
                    const double *start_vec2) {
  or_pc *pc = (or_pc *)xcalloc(1, sizeof(or_pc));
  const int q = s->q, ncb = small_mode ? 1 : s->n_c;
  pc->dim = s->dim;
  pc->n_c = s->n_c;
  pc->q = q;
  pc->small_mode = small_mode;
  pc->nblk = s->n_elements * (small_mode ? s->n_c : 1);
  pc->n1 = ncb * q;
  pc->nb = q;
  pc->ncc = q;
  pc->blk_len = s->dim == 2 ? pc->n1 * q : pc->n1 * q * q;
  pc->flen = s->dim == 2 ? 2 * pc->n1 * pc->n1 + 2 * q * q : pc->n1 * pc->n1 + 4 * q * q;
  pc->s1n = s->dim == 2 ? pc->n1 : q;
  pc->s2n = q;
  pc->fac = (double *)xcalloc((size_t)pc->nblk * pc->flen, sizeof(double));
  pc->lu = (double *)xcalloc((size_t)pc->nblk * pc_lu_len(pc), sizeof(double));
  pc->perm = (int *)xcalloc((size_t)pc->nblk * pc_perm_len(pc), sizeof(int));
  pc->sq = (double *)xcalloc((size_t)pc->nblk * pc_sq_len(pc), sizeof(double));
  pc->has = (int *)xcalloc((size_t)pc->nblk, sizeof(int));
  pc->fb_lu = (double **)xcalloc((size_t)pc->nblk, sizeof(double *));
  pc->fb_perm = (int **)xcalloc((size_t)pc->nblk, sizeof(int *));
  pc->fb_list = (int64_t *)xcalloc((size_t)pc->nblk * 2, sizeof(int64_t));
  const int m1 = pc->n1, m2 = s->dim == 2 ? q : q * q;
  const int maxit = 2 * terms + 20; /* block_lanczos_config (precond/ksvd.hpp:238-243) */
  for (int e = 0; e < s->n_elements; ++e)
    for (int blk = 0; blk < (small_mode ? s->n_c : 1); ++blk) {
      const int idx = e * (small_mode ? s->n_c : 1) + blk;
      shuf_ctx k = {s, e, small_mode, blk, ncb, a, b};
      lz_op op = {m1, m1, m2, m2, elem_apply_cb, elem_apply_t_cb, &k};
      double *fac = pc->fac + (size_t)idx * pc->flen;
      double *lu = pc->lu + (size_t)idx * pc_lu_len(pc);
      int *perm = pc->perm + (size_t)idx * pc_perm_len(pc);
      double *sq = pc->sq + (size_t)idx * pc_sq_len(pc);
      int st;
      if (s->dim == 2) {
        double *fa = (double *)xcalloc((size_t)terms * m1 * m1, sizeof(double));
        double *fbm = (double *)xcalloc((size_t)terms * m2 * m2, sizeof(double));
        double sig[8];
        int its;
        lanczos_ksvd(&op, terms, maxit, 1e-12, start_vec, fa, fbm, sig, &its);
        double *a1 = fac, *b1 = fac + m1 * m1, *a2 = b1 + q * q, *b2 = a2 + m1 * m1;
        memcpy(a1, fa, sizeof(double) * m1 * m1);
        memcpy(b1, fbm, sizeof(double) * q * q);
        if (terms > 1) {
          memcpy(a2, fa + m1 * m1, sizeof(double) * m1 * m1);
          memcpy(b2, fbm + q * q, sizeof(double) * q * q);
        }
        if (terms < 2 || sig[1] <= 1e-12 * sig[0]) {
          set_identity(m1, a2);
          memset(b2, 0, sizeof(double) * q * q);
        }
        st = make_factors_2d(m1, q, a1, b1, a2, b2, lu, perm, sq);
        if (st != OR_OK) {
          /* swap terms (precond/ksvd.hpp:284-291) */
          double *tmp = (double *)xcalloc((size_t)pc->flen, sizeof(double));
          memcpy(tmp, a2, sizeof(double) * m1 * m1);
          memcpy(tmp + m1 * m1, b2, sizeof(double) * q * q);
          memcpy(tmp + m1 * m1 + q * q, a1, sizeof(double) * m1 * m1);
          memcpy(tmp + 2 * m1 * m1 + q * q, b1, sizeof(double) * q * q);
          memcpy(fac, tmp, sizeof(double) * pc->flen);
          free(tmp);
          st = make_factors_2d(m1, q, a1, b1, a2, b2, lu, perm, sq);
        }
        free(fa);
        free(fbm);
      } else {
        double *fa = (double *)xcalloc((size_t)m1 * m1, sizeof(double));
        double *d1 = (double *)xcalloc((size_t)m2 * m2, sizeof(double));
        double sig1[2];
        int its;
        lanczos_ksvd(&op, 1, 2 * 1 + 20, 1e-12, start_vec, fa, d1, sig1, &its);
        if (!(sig1[0] > 0.0)) {
          st = OR_SINGULAR;
        } else {
          double *sh = (double *)xcalloc((size_t)m2 * m2, sizeof(double));
          shuffle_dense(d1, q, q, q, q, sh);
          dense_ctx dc = {m2, m2, sh};
          lz_op op2 = {q, q, q, q, dense_apply_cb, dense_apply_t_cb, &dc};
          double *fb2 = (double *)xcalloc((size_t)terms * q * q, sizeof(double));
          double *fc2 = (double *)xcalloc((size_t)terms * q * q, sizeof(double));
          double sig[8];
          lanczos_ksvd(&op2, terms, maxit, 1e-12, start_vec2, fb2, fc2, sig, &its);
          double *a1 = fac, *b1 = fac + m1 * m1, *c1 = b1 + q * q, *b2 = c1 + q * q, *c2 = b2 + q * q;
          memcpy(a1, fa, sizeof(double) * m1 * m1);
          memcpy(b1, fb2, sizeof(double) * q * q);
          memcpy(c1, fc2, sizeof(double) * q * q);
          if (terms > 1) {
            memcpy(b2, fb2 + q * q, sizeof(double) * q * q);
            memcpy(c2, fc2 + q * q, sizeof(double) * q * q);
          }
          if (terms < 2 || sig[1] <= 1e-12 * sig[0]) {
            set_identity(q, b2);
            memset(c2, 0, sizeof(double) * q * q);
          }
          st = make_factors_3d(m1, q, a1, b1, c1, b2, c2, lu, perm, sq);
          if (st != OR_OK) {
            /* swap second-stage terms (precond/ksvd.hpp:353-358) */
            double tmp[MAXQ * MAXQ];
            memcpy(tmp, b1, sizeof(double) * q * q);
            memcpy(b1, b2, sizeof(double) * q * q);
            memcpy(b2, tmp, sizeof(double) * q * q);
            memcpy(tmp, c1, sizeof(double) * q * q);
            memcpy(c1, c2, sizeof(double) * q * q);
            memcpy(c2, tmp, sizeof(double) * q * q);
            st = make_factors_3d(m1, q, a1, b1, c1, b2, c2, lu, perm, sq);
          }
          free(sh);
          free(fb2);
          free(fc2);
        }
        free(fa);
        free(d1);
      }
      if (st == OR_OK) {
        pc->has[idx] = 1;
      } else {
        /* exact block LU fallback (precond/ksvd.hpp:292-300) */
        const int n = pc->blk_len;
        double *blkm = (double *)xcalloc((size_t)n * n, sizeof(double));
        or_assemble_block(s, e, a, b, small_mode, blk, blkm);
        pc->fb_lu[idx] = (double *)xcalloc((size_t)n * n, sizeof(double));
        pc->fb_perm[idx] = (int *)xcalloc((size_t)n, sizeof(int));
        or_lu_factor(n, blkm, pc->fb_lu[idx], pc->fb_perm[idx]);
        free(blkm);
        pc->fb_list[2 * pc->nfb] = e;
        pc->fb_list[2 * pc->nfb + 1] = small_mode ? blk : -1;
        pc->nfb++;
      }
    }
  return pc;
}

void or_pc_free(or_pc *pc) {
  if (!pc) return;
  for (int i = 0; i < pc->nblk; ++i) {
    free(pc->fb_lu[i]);
    free(pc->fb_perm[i]);
  }
  free(pc->fb_lu); free(pc->fb_perm); free(pc->fb_list);
  free(pc->fac); free(pc->lu); free(pc->perm); free(pc->sq); free(pc->has);
  free(pc);
}

int or_pc_num_fallbacks(const or_pc *pc) { return pc->nfb; }
void or_pc_fallbacks(const or_pc *pc, int64_t *out) { memcpy(out, pc->fb_list, sizeof(int64_t) * 2 * pc->nfb); }
int or_pc_has_factors(const or_pc *pc, int blk) { return pc->has[blk]; }
int or_pc_factor_len(const or_pc *pc) { return pc->flen; }
void or_pc_factors(const or_pc *pc, int blk, double *out) {
  memcpy(out, pc->fac + (size_t)blk * pc->flen, sizeof(double) * pc->flen);
}

int or_pc_record_len(const or_pc *pc) { return pc_lu_len(pc) + pc_sq_len(pc); }
int or_pc_piv_len(const or_pc *pc) { return pc_perm_len(pc); }
void or_pc_record(const or_pc *pc, int blk, double *rec, int *piv) {
  memcpy(rec, pc->lu + (size_t)blk * pc_lu_len(pc), sizeof(double) * pc_lu_len(pc));
  memcpy(rec + pc_lu_len(pc), pc->sq + (size_t)blk * pc_sq_len(pc), sizeof(double) * pc_sq_len(pc));
  memcpy(piv, pc->perm + (size_t)blk * pc_perm_len(pc), sizeof(int) * pc_perm_len(pc));
}

/* matmul (tensor/small_matrix.hpp:103-113): c = a (r x k) b (k x c) */
static void matmul(int r, int kk, int cc, const double *a, const double *b, double *c) {
  for (int i = 0; i < r * cc; ++i) c[i] = 0.0;
  for (int i = 0; i < r; ++i)
    for (int k = 0; k < kk; ++k) {
      const double aik = a[i * kk + k];
      if (aik == 0.0) continue;
      for (int j = 0; j < cc; ++j) c[i * cc + j] += aik * b[k * cc + j];
    }
}
static void transpose(int r, int c, const double *a, double *t) {
  for (int i = 0; i < r; ++i)
    for (int j = 0; j < c; ++j) t[j * r + i] = a[i * c + j];
}

/* axis_solve (ops/kernels.hpp:36-51) */
static void axis_solve(int n, const double *lu, const int *perm, int dim, const int *ext, int axis, double *x) {
  long inner = 1, outer = 1;
  for (int k = 0; k < axis; ++k) inner *= ext[k];
  for (int k = axis + 1; k < dim; ++k) outer *= ext[k];
  double fib[4 * MAXQ], sol[4 * MAXQ];
  for (long o = 0; o < outer; ++o)
    for (long i = 0; i < inner; ++i) {
      double *base = x + o * n * inner + i;
      for (int k = 0; k < n; ++k) fib[k] = base[k * inner];
      or_lu_solve(n, lu, perm, fib, sol);
      for (int k = 0; k < n; ++k) base[k * inner] = sol[k];
    }
}

/* rotate, Sylvester, rotate back on one n1 x n2 slice (precond/ksvd.hpp:121-128) */
static int schur_sylvester(int n1, int n2, const double *sq, double *x) {
  const double *q1 = sq, *t1 = sq + n1 * n1, *q2 = sq + 2 * n1 * n1, *t2 = q2 + n2 * n2;
  const size_t big = (size_t)n1 * (n1 > n2 ? n1 : n2);
  double *q1t = (double *)xcalloc(big, sizeof(double));
  double *q2t = (double *)xcalloc(big, sizeof(double));
  double *tmp = (double *)xcalloc(big, sizeof(double));
  double *mm = (double *)xcalloc(big, sizeof(double));
  double *y = (double *)xcalloc(big, sizeof(double));
  transpose(n1, n1, q1, q1t);
  transpose(n2, n2, q2, q2t);
  matmul(n1, n1, n2, q1t, x, tmp);
  matmul(n1, n2, n2, tmp, q2, mm);
  const int st = or_sylvester(n1, n2, t1, t2, mm, y);
  matmul(n1, n1, n2, q1, y, tmp);
  matmul(n1, n2, n2, tmp, q2t, x);
  free(q1t); free(q2t); free(tmp); free(mm); free(y);
  return st;
}

static int apply_block(const or_pc *pc, int idx, double *x) {
  if (!pc->has[idx]) {
    const int n = pc->blk_len;
    double *tmp = (double *)xcalloc((size_t)n, sizeof(double));
    memcpy(tmp, x, sizeof(double) * n);
    or_lu_solve(n, pc->fb_lu[idx], pc->fb_perm[idx], tmp, x);
    free(tmp);
    return OR_OK;
  }
  const double *lu = pc->lu + (size_t)idx * pc_lu_len(pc);
  const int *perm = pc->perm + (size_t)idx * pc_perm_len(pc);
  const double *sq = pc->sq + (size_t)idx * pc_sq_len(pc);
  const int n1 = pc->n1, q = pc->q;
  if (pc->dim == 2) {
    /* apply_factors_2d (precond/ksvd.hpp:112-129) */
    int ext[2] = {q, n1};
    axis_solve(n1, lu, perm, 2, ext, 1, x);
    axis_solve(q, lu + n1 * n1, perm + n1, 2, ext, 0, x);
    return schur_sylvester(n1, q, sq, x);
  }
  /* apply_factors_3d (precond/ksvd.hpp:132-153) */
  int ext[3] = {q, q, n1};
  axis_solve(n1, lu, perm, 3, ext, 2, x);
  axis_solve(q, lu + n1 * n1, perm + n1, 3, ext, 1, x);
  axis_solve(q, lu + n1 * n1 + q * q, perm + n1 + q, 3, ext, 0, x);
  int st = OR_OK;
  for (int sl = 0; sl < n1; ++sl) {
    const int r = schur_sylvester(q, q, sq, x + (size_t)sl * q * q);
    if (r != OR_OK) st = r;
  }
  return st;
}

/* KsvdPC2D/3D::apply (precond/ksvd.hpp:172-233) */
void or_pc_apply(const or_pc *pc, const double *in, double *out) {
  const size_t total = (size_t)pc->nblk * pc->blk_len;
  memcpy(out, in, sizeof(double) * total);
  for (int idx = 0; idx < pc->nblk; ++idx) apply_block(pc, idx, out + (size_t)idx * pc->blk_len);
}

int or_apply_factors_2d(int n1, int n2, const double *a1, const double *b1, const double *a2, const double *b2,
                        double *x) {
  double *lu = (double *)xcalloc((size_t)n1 * n1 + n2 * n2, sizeof(double));
  int *perm = (int *)xcalloc((size_t)n1 + n2, sizeof(int));
  double *sq = (double *)xcalloc((size_t)2 * n1 * n1 + 2 * n2 * n2, sizeof(double));
  int st = make_factors_2d(n1, n2, a1, b1, a2, b2, lu, perm, sq);
  if (st == OR_OK) {
    int ext[2] = {n2, n1};
    axis_solve(n1, lu, perm, 2, ext, 1, x);
    axis_solve(n2, lu + n1 * n1, perm + n1, 2, ext, 0, x);
    st = schur_sylvester(n1, n2, sq, x);
  }
  free(lu); free(perm); free(sq);
  return st;
}

/* ======================================================================
 * GMRES (solve/gmres.hpp:52-179)
 * ====================================================================== */
typedef struct {
  const or_sys *s;
  double a, b;
  int small_mode;
  const or_pc *pc;
} gm_ctx;

static void gm_op(const gm_ctx *c, const double *in, double *out) { or_jv(c->s, c->a, c->b, c->small_mode, in, out); }
static void gm_pc(const gm_ctx *c, const double *in, double *out) { or_pc_apply(c->pc, in, out); }

int or_gmres(const or_sys *s, double a, double b, int small_mode, const or_pc *pc, const double *rhs, double tol,
             int restart, int max_it, int left, double *x, int *iterations, double *hist, int hist_cap,
             int *converged) {
  gm_ctx ctx = {s, a, b, small_mode, pc};
  const long n = (long)s->n_elements * s->n_c * npe_of(s);
  const int m = restart;
  double *tmp = (double *)xcalloc((size_t)n, sizeof(double));
  double *tmp2 = (double *)xcalloc((size_t)n, sizeof(double));
  double *r = (double *)xcalloc((size_t)n, sizeof(double));
  double *v = (double *)xcalloc((size_t)(m + 1) * n, sizeof(double));
  double *h = (double *)xcalloc((size_t)(m + 1) * m, sizeof(double));
  double *cs = (double *)xcalloc((size_t)m, sizeof(double));
  double *sn = (double *)xcalloc((size_t)m, sizeof(double));
  double *g = (double *)xcalloc((size_t)m + 1, sizeof(double));
  double *y = (double *)xcalloc((size_t)m, sizeof(double));
  int its = 0, nh = 0, conv = 0;
  for (long i = 0; i < n; ++i) x[i] = 0.0;
  double target;
  if (!left) {
    target = tol * norm2(rhs, n);
  } else {
    gm_pc(&ctx, rhs, r);
    target = tol * norm2(r, n);
  }
  if (target == 0.0) {
    conv = 1;
    goto done;
  }
  while (its < max_it) {
    gm_op(&ctx, x, tmp);
    for (long i = 0; i < n; ++i) tmp[i] = rhs[i] - tmp[i];
    if (!left) memcpy(r, tmp, sizeof(double) * n); else gm_pc(&ctx, tmp, r);
    const double beta = norm2(r, n);
    if (beta <= target) {
      conv = 1;
      goto done;
    }
    for (long i = 0; i < n; ++i) v[i] = r[i] / beta;
    for (int i = 0; i <= m; ++i) g[i] = 0.0;
    g[0] = beta;
    for (long i = 0; i < (long)(m + 1) * m; ++i) h[i] = 0.0;
    int k = 0;
    for (; k < m && its < max_it; ++k) {
      ++its;
      double *vk = v + (size_t)k * n, *vk1 = v + (size_t)(k + 1) * n;
      if (!left) {
        gm_pc(&ctx, vk, tmp2);
        gm_op(&ctx, tmp2, vk1);
      } else {
        gm_op(&ctx, vk, tmp);
        gm_pc(&ctx, tmp, vk1);
      }
      for (int j = 0; j <= k; ++j) {
        const double *vj = v + (size_t)j * n;
        double dot = 0.0;
        for (long i = 0; i < n; ++i) dot += vj[i] * vk1[i];
        h[j * m + k] = dot;
        for (long i = 0; i < n; ++i) vk1[i] -= dot * vj[i];
      }
      const double hkk = norm2(vk1, n);
      h[(k + 1) * m + k] = hkk;
      if (hkk > 0.0)
        for (long i = 0; i < n; ++i) vk1[i] /= hkk;
      for (int j = 0; j < k; ++j) {
        const double t1 = h[j * m + k], t2 = h[(j + 1) * m + k];
        h[j * m + k] = cs[j] * t1 + sn[j] * t2;
        h[(j + 1) * m + k] = -sn[j] * t1 + cs[j] * t2;
      }
      const double t1 = h[k * m + k], t2 = h[(k + 1) * m + k];
      const double den = hypot(t1, t2);
      cs[k] = den == 0.0 ? 1.0 : t1 / den;
      sn[k] = den == 0.0 ? 0.0 : t2 / den;
      h[k * m + k] = den;
      h[(k + 1) * m + k] = 0.0;
      const double gk = g[k];
      g[k] = cs[k] * gk;
      g[k + 1] = -sn[k] * gk;
      if (nh < hist_cap) hist[nh] = fabs(g[k + 1]);
      ++nh;
      if (fabs(g[k + 1]) <= target) {
        ++k;
        break;
      }
    }
    for (int i = k - 1; i >= 0; --i) {
      double sacc = g[i];
      for (int j = i + 1; j < k; ++j) sacc -= h[i * m + j] * y[j];
      y[i] = sacc / h[i * m + i];
    }
    for (long i = 0; i < n; ++i) tmp[i] = 0.0;
    for (int j = 0; j < k; ++j)
      for (long i = 0; i < n; ++i) tmp[i] += y[j] * v[(size_t)j * n + i];
    if (!left) {
      gm_pc(&ctx, tmp, tmp2);
      for (long i = 0; i < n; ++i) x[i] += tmp2[i];
    } else {
      for (long i = 0; i < n; ++i) x[i] += tmp[i];
    }
    if (nh > 0 && fabs(g[k]) <= target) {
      /* residual_history.back() is |g[k]| of the last completed iteration */
      conv = 1;
      goto done;
    }
  }
  gm_op(&ctx, x, tmp);
  for (long i = 0; i < n; ++i) tmp[i] = rhs[i] - tmp[i];
  if (!left) memcpy(r, tmp, sizeof(double) * n); else gm_pc(&ctx, tmp, r);
  conv = norm2(r, n) <= target;
done:
  *iterations = its;
  *converged = conv;
  free(tmp); free(tmp2); free(r); free(v); free(h); free(cs); free(sn); free(g); free(y);
  return nh;
}
