// Matrix-free shuffled products of one element's diagonal block (device, CTA-cooperative).
//
// Restates kernels::ElementShuffled (reference ops/shuffled.hpp:22-505): apply_2d (:65-147),
// apply_t_2d (:149-234), apply_3d (:238-367), apply_t_3d (:369-503). Compiled with -fmad=false:
// every accumulator is summed in the reference's order by one thread, parallelism is over
// independent accumulators, so results equal the reference's bit for bit.
//
// Scratch `ws` is global memory (L2 resident) private to the calling CTA.
#pragma once

#include "tpdg_internal.hpp"

namespace tpdg_gpu {

// Cooperating thread groups: a whole CTA or one warp works on one block.
struct CtaGroup {
  __device__ __forceinline__ int rank() const { return threadIdx.x; }
  __device__ __forceinline__ int size() const { return blockDim.x; }
  __device__ __forceinline__ void sync() const { __syncthreads(); }
};
struct WarpGroup {
  __device__ __forceinline__ int rank() const { return threadIdx.x & 31; }
  __device__ __forceinline__ int size() const { return 32; }
  __device__ __forceinline__ void sync() const { __syncwarp(); }
};

struct ShufCtx {
  DevSys s;
  int e, comp, ncb;  // element (local), component (small mode), components in the block
};

__device__ __forceinline__ double sh_dft(const ShufCtx& k, int dir, int qv, int r, int c) {
  const int nc = k.s.n_c;
  const int rr = k.s.small ? k.comp : r, cc = k.s.small ? k.comp : c;
  return k.s.dft[((size_t(k.e) * k.s.dim + dir) * k.s.nqv + qv) * nc * nc + rr * nc + cc];
}
__device__ __forceinline__ double sh_dfm(const ShufCtx& k, int f, int qf, int r, int c) {
  const int nc = k.s.n_c;
  const int rr = k.s.small ? k.comp : r, cc = k.s.small ? k.comp : c;
  return k.s.dfm[((size_t(k.e) * 2 * k.s.dim + f) * k.s.nqf + qf) * nc * nc + rr * nc + cc];
}

#define SG(a, j) (S.g[(a) * q + (j)])
#define SD(a, j) (S.d[(a) * q + (j)])

// u = Atilde v (2D). ws >= 2*mu + mu + 2*nc*nc*mu
template <class Grp>
__device__ void shuf_apply_2d_dev(const Grp& g, const ShufCtx& k, const double* v, double* u, double* ws) {
  const DevSys& S = k.s;
  const int q = S.q, mu = S.mu, nc = k.ncb, m1 = nc * q, tid = g.rank(), nt = g.size();
  const double a = S.a, b = S.b;
  double* tgg = ws;
  double* tdg = tgg + mu;
  double* sm = tdg + mu;
  double* r1 = sm + mu;
  double* r2 = r1 + nc * nc * mu;
  const double* jd = S.jdet + size_t(k.e) * mu * mu;
  for (int al = tid; al < mu; al += nt) {
    double sg = 0.0, sd = 0.0;
    for (int ec = 0; ec < q; ++ec) {
      double cg = 0.0, cd = 0.0;
      for (int ar = 0; ar < q; ++ar) {
        cg += SG(al, ar) * v[ec * q + ar];
        cd += SD(al, ar) * v[ec * q + ar];
      }
      sg += SG(al, ec) * cg;
      sd += SG(al, ec) * cd;
    }
    tgg[al] = sg;
    tdg[al] = sd;
  }
  g.sync();
  for (int t = tid; t < mu * (1 + nc * nc); t += nt) {
    const int be = t % mu, rc = t / mu;  // rc == 0: sm ; rc-1 = cr*nc + cc
    if (rc == 0) {
      double acc = 0.0;
      for (int al = 0; al < mu; ++al) acc += S.w[al] * jd[be * mu + al] * tgg[al];
      sm[be] = acc;
    } else if (b != 0.0) {
      const int cr = (rc - 1) / nc, cc = (rc - 1) % nc;
      double x1 = 0.0, x2 = 0.0;
      for (int al = 0; al < mu; ++al) {
        const int qv = be * mu + al;
        x1 += S.w[al] * sh_dft(k, 0, qv, cr, cc) * tdg[al];
        x2 += S.w[al] * sh_dft(k, 1, qv, cr, cc) * tgg[al];
      }
      r1[(cr * nc + cc) * mu + be] = x1;
      r2[(cr * nc + cc) * mu + be] = x2;
    }
  }
  g.sync();
  for (int t = tid; t < m1 * m1; t += nt) {
    const int br = t % q, cr = (t / q) % nc, dc = (t / m1) % q, cc = t / (m1 * q);
    double acc = 0.0;
    for (int be = 0; be < mu; ++be) {
      const double wb = S.w[be];
      double val = 0.0;
      if (cr == cc && a != 0.0) val += a * sm[be];
      if (b != 0.0) val += b * r1[(cr * nc + cc) * mu + be];
      acc += wb * SG(be, br) * SG(be, dc) * val;
      if (b != 0.0) acc += wb * SD(be, br) * SG(be, dc) * b * r2[(cr * nc + cc) * mu + be];
    }
    if (b != 0.0)
      for (int f = 0; f < 4; ++f) {
        const double* fw = S.face_w + (size_t(k.e) * 4 + f) * mu;
        const int layer = (f % 2) == 0 ? 0 : q - 1;
        if (f / 2 == 0) {
          const double vc = v[layer * q + layer];
          double s = 0.0;
          for (int be = 0; be < mu; ++be) s += fw[be] * sh_dfm(k, f, be, cr, cc) * SG(be, br) * SG(be, dc);
          acc -= b * s * vc;
        } else if (dc == layer && br == layer) {
          double s = 0.0;
          for (int al = 0; al < mu; ++al) s += fw[al] * sh_dfm(k, f, al, cr, cc) * tgg[al];
          acc -= b * s;
        }
      }
    u[t] = acc;  // index (cc*q + dc)*m1 + cr*q + br
  }
  g.sync();
}

// v = Atilde^T u (2D). ws >= 2*nc*nc*mu + 3*mu + 4*mu
template <class Grp>
__device__ void shuf_apply_t_2d_dev(const Grp& g, const ShufCtx& k, const double* u, double* v, double* ws) {
  const DevSys& S = k.s;
  const int q = S.q, mu = S.mu, nc = k.ncb, m1 = nc * q, tid = g.rank(), nt = g.size();
  const double a = S.a, b = S.b;
#define UU(cr, br, cc, dc) u[((cc) * q + (dc)) * m1 + (cr) * q + (br)]
  double* hgg = ws;
  double* hdg = hgg + nc * nc * mu;
  double* km = hdg + nc * nc * mu;
  double* k1 = km + mu;
  double* k2 = k1 + mu;
  double* fs = k2 + mu;  // axis-0 face sums [2] ; axis-1 coefs [2][mu]
  const double* jd = S.jdet + size_t(k.e) * mu * mu;
  for (int t = tid; t < nc * nc * mu; t += nt) {
    const int be = t % mu, cc = (t / mu) % nc, cr = t / (mu * nc);
    double sg = 0.0, sd = 0.0;
    for (int dc = 0; dc < q; ++dc) {
      double cg = 0.0, cd = 0.0;
      for (int br = 0; br < q; ++br) {
        cg += SG(be, br) * UU(cr, br, cc, dc);
        cd += SD(be, br) * UU(cr, br, cc, dc);
      }
      sg += SG(be, dc) * cg;
      sd += SG(be, dc) * cd;
    }
    hgg[t] = sg;
    hdg[t] = sd;
  }
  g.sync();
  for (int al = tid; al < mu; al += nt) {
    double xm = 0.0, x1 = 0.0, x2 = 0.0;
    for (int be = 0; be < mu; ++be) {
      const double wb = S.w[be];
      const int qv = be * mu + al;
      const double w = S.w[al] * wb;
      double smass = 0.0;
      for (int c = 0; c < nc; ++c) smass += hgg[(c * nc + c) * mu + be];
      xm += w * jd[qv] * smass;
      if (b != 0.0) {
        double s1 = 0.0, s2 = 0.0;
        for (int cr = 0; cr < nc; ++cr)
          for (int cc = 0; cc < nc; ++cc) {
            s1 += sh_dft(k, 0, qv, cr, cc) * hgg[(cr * nc + cc) * mu + be];
            s2 += sh_dft(k, 1, qv, cr, cc) * hdg[(cr * nc + cc) * mu + be];
          }
        x1 += w * s1;
        x2 += w * s2;
      }
    }
    km[al] = xm;
    k1[al] = x1;
    k2[al] = x2;
  }
  // face pre-sums: axis-0 faces (f=0,1) -> scalar ; axis-1 faces (f=2,3) -> coef[al]
  for (int t = tid; t < 2 + 2 * mu; t += nt) {
    if (b == 0.0) break;
    if (t < 2) {
      const int f = t;
      const double* fw = S.face_w + (size_t(k.e) * 4 + f) * mu;
      double s = 0.0;
      for (int be = 0; be < mu; ++be) {
        double sc = 0.0;
        for (int cr = 0; cr < nc; ++cr)
          for (int cc = 0; cc < nc; ++cc) sc += sh_dfm(k, f, be, cr, cc) * hgg[(cr * nc + cc) * mu + be];
        s += fw[be] * sc;
      }
      fs[f] = s;
    } else {
      const int f = 2 + (t - 2) / mu, al = (t - 2) % mu;
      const double* fw = S.face_w + (size_t(k.e) * 4 + f) * mu;
      const int layer = (f % 2) == 0 ? 0 : q - 1;
      double sc = 0.0;
      for (int cr = 0; cr < nc; ++cr)
        for (int cc = 0; cc < nc; ++cc) sc += sh_dfm(k, f, al, cr, cc) * UU(cr, layer, cc, layer);
      fs[t] = b * fw[al] * sc;
    }
  }
  g.sync();
  for (int t = tid; t < q * q; t += nt) {
    const int ar = t % q, ec = t / q;
    double acc = 0.0;
    for (int al = 0; al < mu; ++al) {
      acc += SG(al, ar) * SG(al, ec) * (a * km[al] + b * k2[al]);
      acc += SD(al, ar) * SG(al, ec) * b * k1[al];
    }
    if (b != 0.0)
      for (int f = 0; f < 4; ++f) {
        const int layer = (f % 2) == 0 ? 0 : q - 1;
        if (f / 2 == 0) {
          if (ec == layer && ar == layer) acc -= b * fs[f];
        } else {
          const double* coef = fs + 2 + (f - 2) * mu;
          for (int al = 0; al < mu; ++al) acc -= coef[al] * SG(al, ar) * SG(al, ec);
        }
      }
    v[t] = acc;
  }
  g.sync();
#undef UU
}

// u = Atilde v (3D, O(p^5)).
template <class Grp>
__device__ void shuf_apply_3d_dev(const Grp& g, const ShufCtx& k, const double* v, double* u, double* ws) {
  const DevSys& S = k.s;
  const int q = S.q, mu = S.mu, nc = k.ncb, m1 = nc * q, q2 = q * q, tid = g.rank(), nt = g.size();
  const double a = S.a, b = S.b;
#define VV(a1, a2, e1, e2) v[((e2) * q + (e1)) * q2 + (a2) * q + (a1)]
  const int n4 = mu * q * q * q;
  double* a1g = ws;
  double* a1d = a1g + n4;
  double* t4x = a1d + n4;
  double* t4y = t4x + mu * mu;
  double* t4g = t4y + mu * mu;
  double* rm = t4g + mu * mu;
  double* r1 = rm + mu;
  double* r2 = r1 + nc * nc * mu;
  double* r3 = r2 + nc * nc * mu;
  double* wbuf = r3 + nc * nc * mu;          // [4][mu]
  double* inner = wbuf + 4 * mu;             // [4][nc][nc][mu]
  double* s2f = inner + 4 * nc * nc * mu;    // [2][nc][nc]
  for (int t = tid; t < n4; t += nt) {
    const int e2 = t % q, e1 = (t / q) % q, a2 = (t / q2) % q, al = t / (q2 * q);
    double sg = 0.0, sd = 0.0;
    for (int ar = 0; ar < q; ++ar) {
      sg += SG(al, ar) * VV(ar, a2, e1, e2);
      sd += SD(al, ar) * VV(ar, a2, e1, e2);
    }
    a1g[t] = sg;
    a1d[t] = sd;
  }
  // wbuf for x/y faces (only needs v)
  for (int t = tid; t < 4 * mu; t += nt) {
    if (b == 0.0) break;
    const int f = t / mu, al = t % mu, axis = f / 2, layer = (f % 2) == 0 ? 0 : q - 1;
    double s = 0.0;
    for (int ej = 0; ej < q; ++ej)
      for (int aj = 0; aj < q; ++aj) {
        const double vv = axis == 0 ? VV(layer, aj, layer, ej) : VV(aj, layer, ej, layer);
        s += SG(al, ej) * SG(al, aj) * vv;
      }
    wbuf[t] = s;
  }
  g.sync();
  for (int t = tid; t < mu * mu; t += nt) {
    const int be = t % mu, al = t / mu;
    double sx = 0.0, sy = 0.0, sg = 0.0;
    for (int e2 = 0; e2 < q; ++e2)
      for (int e1 = 0; e1 < q; ++e1) {
        double cx = 0.0, cy = 0.0, cg = 0.0;
        for (int a2 = 0; a2 < q; ++a2) {
          const int idg = ((al * q + a2) * q + e1) * q + e2;
          cx += SG(be, a2) * a1d[idg];
          cy += SD(be, a2) * a1g[idg];
          cg += SG(be, a2) * a1g[idg];
        }
        const double gee = SG(al, e1) * SG(be, e2);
        sx += gee * cx;
        sy += gee * cy;
        sg += gee * cg;
      }
    t4x[t] = sx;
    t4y[t] = sy;
    t4g[t] = sg;
  }
  // inner sums of the x/y faces: inner[f][cr][cc][be] = sum_al fw dfm wbuf
  for (int t = tid; t < 4 * nc * nc * mu; t += nt) {
    if (b == 0.0) break;
    const int be = t % mu, cc = (t / mu) % nc, cr = (t / (mu * nc)) % nc, f = t / (mu * nc * nc);
    const double* fw = S.face_w + (size_t(k.e) * 6 + f) * mu * mu;
    double s = 0.0;
    for (int al = 0; al < mu; ++al) s += fw[be * mu + al] * sh_dfm(k, f, be * mu + al, cr, cc) * wbuf[f * mu + al];
    inner[t] = s;
  }
  g.sync();
  const double* jd = S.jdet + size_t(k.e) * mu * mu * mu;
  for (int t = tid; t < mu * (1 + nc * nc) + 2 * nc * nc; t += nt) {
    if (t < mu * (1 + nc * nc)) {
      const int ga = t % mu, rc = t / mu;
      if (rc == 0) {
        double acc = 0.0;
        for (int be = 0; be < mu; ++be)
          for (int al = 0; al < mu; ++al) {
            const int qv = (ga * mu + be) * mu + al;
            acc += S.w[al] * S.w[be] * jd[qv] * t4g[al * mu + be];
          }
        rm[ga] = acc;
      } else if (b != 0.0) {
        const int cr = (rc - 1) / nc, cc = (rc - 1) % nc;
        double x1 = 0.0, x2 = 0.0, x3 = 0.0;
        for (int be = 0; be < mu; ++be)
          for (int al = 0; al < mu; ++al) {
            const int qv = (ga * mu + be) * mu + al;
            const double w = S.w[al] * S.w[be];
            x1 += w * sh_dft(k, 0, qv, cr, cc) * t4x[al * mu + be];
            x2 += w * sh_dft(k, 1, qv, cr, cc) * t4y[al * mu + be];
            x3 += w * sh_dft(k, 2, qv, cr, cc) * t4g[al * mu + be];
          }
        const int rc2 = (cr * nc + cc) * mu + ga;
        r1[rc2] = x1;
        r2[rc2] = x2;
        r3[rc2] = x3;
      }
    } else if (b != 0.0) {  // z faces: s2f[f-4][cr][cc]
      const int tt = t - mu * (1 + nc * nc);
      const int f = 4 + tt / (nc * nc), cr = (tt % (nc * nc)) / nc, cc = tt % nc;
      const double* fw = S.face_w + (size_t(k.e) * 6 + f) * mu * mu;
      double s = 0.0;
      for (int be = 0; be < mu; ++be)
        for (int al = 0; al < mu; ++al) s += fw[be * mu + al] * sh_dfm(k, f, be * mu + al, cr, cc) * t4g[al * mu + be];
      s2f[tt] = s;
    }
  }
  g.sync();
  for (int t = tid; t < m1 * m1; t += nt) {
    const int b3 = t % q, cr = (t / q) % nc, d3 = (t / m1) % q, cc = t / (m1 * q);
    double acc = 0.0;
    for (int ga = 0; ga < mu; ++ga) {
      const double wg = S.w[ga];
      double val = 0.0;
      if (cr == cc && a != 0.0) val += a * rm[ga];
      if (b != 0.0) val += b * (r1[(cr * nc + cc) * mu + ga] + r2[(cr * nc + cc) * mu + ga]);
      acc += wg * SG(ga, b3) * SG(ga, d3) * val;
      if (b != 0.0) acc += wg * SD(ga, b3) * SG(ga, d3) * b * r3[(cr * nc + cc) * mu + ga];
    }
    if (b != 0.0)
      for (int f = 0; f < 6; ++f) {
        const int layer = (f % 2) == 0 ? 0 : q - 1;
        if (f / 2 == 2) {
          if (d3 == layer && b3 == layer) acc -= b * s2f[((f - 4) * nc + cr) * nc + cc];
        } else {
          const double* in = inner + ((f * nc + cr) * nc + cc) * mu;
          double s = 0.0;
          for (int be = 0; be < mu; ++be) s += SG(be, b3) * SG(be, d3) * in[be];
          acc -= b * s;
        }
      }
    u[t] = acc;
  }
  g.sync();
#undef VV
}

// v = Atilde^T u (3D).
template <class Grp>
__device__ void shuf_apply_t_3d_dev(const Grp& g, const ShufCtx& k, const double* u, double* v, double* ws) {
  const DevSys& S = k.s;
  const int q = S.q, mu = S.mu, nc = k.ncb, m1 = nc * q, q2 = q * q, tid = g.rank(), nt = g.size();
  const double a = S.a, b = S.b;
#define UU(cr, b3, cc, d3) u[((cc) * q + (d3)) * m1 + (cr) * q + (b3)]
  double* hgg = ws;
  double* hdg = hgg + nc * nc * mu;
  double* kx = hdg + nc * nc * mu;
  double* ky = kx + mu * mu;
  double* kg = ky + mu * mu;
  double* p1x = kg + mu * mu;
  double* p1y = p1x + mu * q * q;
  double* p1g = p1y + mu * q * q;
  double* lbuf = p1g + mu * q * q;  // [4][mu]
  for (int t = tid; t < nc * nc * mu; t += nt) {
    const int ga = t % mu, cc = (t / mu) % nc, cr = t / (mu * nc);
    double sg = 0.0, sd = 0.0;
    for (int d3 = 0; d3 < q; ++d3) {
      double cg = 0.0, cd = 0.0;
      for (int b3 = 0; b3 < q; ++b3) {
        cg += SG(ga, b3) * UU(cr, b3, cc, d3);
        cd += SD(ga, b3) * UU(cr, b3, cc, d3);
      }
      sg += SG(ga, d3) * cg;
      sd += SG(ga, d3) * cd;
    }
    hgg[t] = sg;
    hdg[t] = sd;
  }
  g.sync();
  const double* jd = S.jdet + size_t(k.e) * mu * mu * mu;
  for (int t = tid; t < mu * mu + 4 * mu; t += nt) {
    if (t < mu * mu) {
      const int be = t % mu, al = t / mu;
      double xx = 0.0, xy = 0.0, xg = 0.0;
      for (int ga = 0; ga < mu; ++ga) {
        const double wg = S.w[ga];
        const int qv = (ga * mu + be) * mu + al;
        const double w = S.w[al] * S.w[be] * wg;
        double smass = 0.0;
        for (int c = 0; c < nc; ++c) smass += hgg[(c * nc + c) * mu + ga];
        xg += a * w * jd[qv] * smass;
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
          xx += b * w * s1;
          xy += b * w * s2;
          xg += b * w * s3;
        }
      }
      if (b != 0.0)  // z faces fold into kg (f = 4, 5 in order)
        for (int f = 4; f < 6; ++f) {
          const double* fw = S.face_w + (size_t(k.e) * 6 + f) * mu * mu;
          const int layer = (f % 2) == 0 ? 0 : q - 1;
          double sc = 0.0;
          for (int cr = 0; cr < nc; ++cr)
            for (int cc = 0; cc < nc; ++cc) sc += sh_dfm(k, f, be * mu + al, cr, cc) * UU(cr, layer, cc, layer);
          xg -= b * fw[be * mu + al] * sc;
        }
      kx[al * mu + be] = xx;
      ky[al * mu + be] = xy;
      kg[al * mu + be] = xg;
    } else if (b != 0.0) {
      const int tt = t - mu * mu, f = tt / mu, al = tt % mu;
      const double* fw = S.face_w + (size_t(k.e) * 6 + f) * mu * mu;
      double s = 0.0;
      for (int be = 0; be < mu; ++be) {
        double sc = 0.0;
        for (int cr = 0; cr < nc; ++cr)
          for (int cc = 0; cc < nc; ++cc) sc += sh_dfm(k, f, be * mu + al, cr, cc) * hgg[(cr * nc + cc) * mu + be];
        s += fw[be * mu + al] * sc;
      }
      lbuf[tt] = s;
    }
  }
  g.sync();
  for (int t = tid; t < mu * q * q; t += nt) {
    const int e2 = t % q, a2 = (t / q) % q, al = t / q2;
    double sx = 0.0, sy = 0.0, sg = 0.0;
    for (int be = 0; be < mu; ++be) {
      const double ge2 = SG(be, e2);
      sx += SG(be, a2) * ge2 * kx[al * mu + be];
      sy += SD(be, a2) * ge2 * ky[al * mu + be];
      sg += SG(be, a2) * ge2 * kg[al * mu + be];
    }
    p1x[t] = sx;
    p1y[t] = sy;
    p1g[t] = sg;
  }
  g.sync();
  for (int t = tid; t < q2 * q2; t += nt) {
    const int a1 = t % q, a2 = (t / q) % q, e1 = (t / q2) % q, e2 = t / (q2 * q);
    double acc = 0.0;
    for (int al = 0; al < mu; ++al) {
      const double ge1 = SG(al, e1);
      const int idx = (al * q + a2) * q + e2;
      acc += SD(al, a1) * ge1 * p1x[idx];
      acc += SG(al, a1) * ge1 * (p1y[idx] + p1g[idx]);
    }
    if (b != 0.0)
      for (int f = 0; f < 4; ++f) {
        const int layer = (f % 2) == 0 ? 0 : q - 1;
        int aj, ej;
        if (f / 2 == 0) {
          if (e1 != layer || a1 != layer) continue;
          aj = a2;
          ej = e2;
        } else {
          if (e2 != layer || a2 != layer) continue;
          aj = a1;
          ej = e1;
        }
        double s = 0.0;
        for (int al = 0; al < mu; ++al) s += SG(al, aj) * SG(al, ej) * lbuf[f * mu + al];
        acc -= b * s;
      }
    v[t] = acc;  // index ((e2*q + e1)*q2 + a2*q + a1)
  }
  g.sync();
#undef UU
}

#undef SG
#undef SD

__host__ __device__ inline size_t shuffled_ws_doubles(int dim, int q, int mu, int nc) {
  if (dim == 2) return size_t(3 * mu + 2 * nc * nc * mu + 2 * nc * nc * mu + 3 * mu + 2 + 2 * mu + 8);
  const size_t fwd = 2 * size_t(mu) * q * q * q + 3 * mu * mu + mu + 3 * nc * nc * mu + 4 * mu + 4 * nc * nc * mu + 2 * nc * nc;
  const size_t bwd = 2 * nc * nc * mu + 3 * mu * mu + 3 * size_t(mu) * q * q + 4 * mu;
  return (fwd > bwd ? fwd : bwd) + 8;
}

} // namespace tpdg_gpu
