/* TEST INFRASTRUCTURE ONLY -- the parity checker, never the product path.
 * See oracle.h for the contract. Every function restates the cited reference
 * lines with the same loop order, so that with -ffp-contract=off the results
 * are bitwise those of the reference on the same inputs.
 */
#include "oracle.h"

#include <math.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

static _Thread_local char g_err[256];
const char* or_last_error(void) { return g_err; }
static int fail(int code, const char* msg) {
  snprintf(g_err, sizeof g_err, "%s", msg);
  return code;
}

#define XMALLOC(T, n) ((T*)calloc((size_t)((n) > 0 ? (n) : 1), sizeof(T)))

/* ------------------------------------------------------------ sparse.cpp */

/* sparse.cpp:78-91 -- sequential per-row accumulation */
void or_spmv(const or_csr* m, const double* x, double* y) {
  for (int r = 0; r < m->nrows; ++r) {
    double acc = 0.0;
    for (int k = m->rp[r]; k < m->rp[r + 1]; ++k) acc += m->v[k] * x[m->ci[k]];
    y[r] = acc;
  }
}

/* sparse.cpp:217-221 */
double or_norm2(int n, const double* v) {
  double s = 0.0;
  for (int i = 0; i < n; ++i) s += v[i] * v[i];
  return sqrt(s);
}

/* sparse.cpp:223-227 */
double or_dot(int n, const double* a, const double* b) {
  double s = 0.0;
  for (int i = 0; i < n; ++i) s += a[i] * b[i];
  return s;
}

/* sparse.cpp:229-237 */
double or_norm_inf(const or_csr* m) {
  double best = 0.0;
  for (int r = 0; r < m->nrows; ++r) {
    double s = 0.0;
    for (int k = m->rp[r]; k < m->rp[r + 1]; ++k) s += fabs(m->v[k]);
    if (s > best) best = s;
  }
  return best;
}

/* sparse.cpp:310-341 -- partial pivoting on max |a_ik| (first max wins),
 * whole-row swaps, multiplier a_ik * (1/a_kk) */
int or_lu_factor(int n, double* a, int* piv) {
  for (int i = 0; i < n; ++i) piv[i] = i;
  for (int k = 0; k < n; ++k) {
    int p = k;
    double best = fabs(a[(size_t)k * n + k]);
    for (int i = k + 1; i < n; ++i) {
      const double v = fabs(a[(size_t)i * n + k]);
      if (v > best) {
        best = v;
        p = i;
      }
    }
    if (best == 0.0) return fail(OR_SINGULAR_MATRIX, "dense_lu_factor: singular pivot column");
    if (p != k) {
      for (int j = 0; j < n; ++j) {
        const double t = a[(size_t)k * n + j];
        a[(size_t)k * n + j] = a[(size_t)p * n + j];
        a[(size_t)p * n + j] = t;
      }
      const int t = piv[k];
      piv[k] = piv[p];
      piv[p] = t;
    }
    const double inv_piv = 1.0 / a[(size_t)k * n + k];
    for (int i = k + 1; i < n; ++i) {
      const double mult = a[(size_t)i * n + k] * inv_piv;
      a[(size_t)i * n + k] = mult;
      if (mult == 0.0) continue;
      for (int j = k + 1; j < n; ++j) a[(size_t)i * n + j] -= mult * a[(size_t)k * n + j];
    }
  }
  return OR_OK;
}

/* sparse.cpp:343-361 */
void or_lu_solve(int n, const double* lu, const int* piv, double* b) {
  double stackbuf[128];
  double* x = n <= 128 ? stackbuf : XMALLOC(double, n);
  for (int i = 0; i < n; ++i) x[i] = b[piv[i]];
  for (int i = 1; i < n; ++i) {
    double acc = x[i];
    for (int j = 0; j < i; ++j) acc -= lu[(size_t)i * n + j] * x[j];
    x[i] = acc;
  }
  for (int i = n - 1; i >= 0; --i) {
    double acc = x[i];
    for (int j = i + 1; j < n; ++j) acc -= lu[(size_t)i * n + j] * x[j];
    x[i] = acc / lu[(size_t)i * n + i];
  }
  for (int i = 0; i < n; ++i) b[i] = x[i];
  if (x != stackbuf) free(x);
}

/* ------------------------------------------------------------- vanka.cpp */

static int cmp_int(const void* a, const void* b) {
  const int x = *(const int*)a, y = *(const int*)b;
  return (x > y) - (x < y);
}

/* vanka.cpp:11-42 -- velocity set = sorted unique columns c < n_u of the seed
 * rows; nx = lower_bound(n_x); SV fine level seeds consecutive row triples */
int or_build_patches(const or_csr* k, int n_x, int n_y, int n_p, int sv_triples,
                     or_patches* out) {
  const int n_u = n_x + n_y;
  memset(out, 0, sizeof *out);
  if (k->nrows != n_u + n_p) return fail(OR_DIM, "build_patches: block sizes do not match K");
  if (sv_triples && n_p % 3 != 0)
    return fail(OR_DIM, "build_patches: triple seeding needs a multiple-of-3 pressure count");
  const int group = sv_triples ? 3 : 1;
  const int np = n_p / group;
  out->npatch = np;
  out->pptr = XMALLOC(int, np + 1);
  out->pidx = XMALLOC(int, n_p);
  out->vptr = XMALLOC(int, np + 1);
  out->nx = XMALLOC(int, np);
  int64_t cap = 0;
  for (int p0 = 0; p0 < n_p; ++p0) cap += k->rp[n_u + p0 + 1] - k->rp[n_u + p0];
  out->vidx = XMALLOC(int, cap);
  int pp = 0, vv = 0;
  for (int i = 0; i < np; ++i) {
    const int start = vv;
    for (int g = 0; g < group; ++g) {
      const int row = n_u + i * group + g;
      out->pidx[pp++] = row;
      for (int q = k->rp[row]; q < k->rp[row + 1]; ++q)
        if (k->ci[q] < n_u) out->vidx[vv++] = k->ci[q];
    }
    qsort(out->vidx + start, (size_t)(vv - start), sizeof(int), cmp_int);
    int u = start;
    for (int q = start; q < vv; ++q)
      if (q == start || out->vidx[q] != out->vidx[u - 1]) out->vidx[u++] = out->vidx[q];
    vv = u;
    if (vv == start) {
      or_patches_free(out);
      return fail(OR_SINGULAR_PATCH, "build_patches: pressure row couples to no velocity DoFs");
    }
    int nx = 0;
    while (start + nx < vv && out->vidx[start + nx] < n_x) ++nx;
    out->nx[i] = nx;
    out->pptr[i + 1] = pp;
    out->vptr[i + 1] = vv;
  }
  return OR_OK;
}

void or_patches_free(or_patches* p) {
  free(p->pptr);
  free(p->pidx);
  free(p->vptr);
  free(p->vidx);
  free(p->nx);
  memset(p, 0, sizeof *p);
}

static void copy_patches(const or_patches* in, or_patches* out) {
  const int np = in->npatch;
  out->npatch = np;
  out->pptr = XMALLOC(int, np + 1);
  out->vptr = XMALLOC(int, np + 1);
  out->nx = XMALLOC(int, np);
  out->pidx = XMALLOC(int, in->pptr[np]);
  out->vidx = XMALLOC(int, in->vptr[np]);
  memcpy(out->pptr, in->pptr, sizeof(int) * (np + 1));
  memcpy(out->vptr, in->vptr, sizeof(int) * (np + 1));
  memcpy(out->nx, in->nx, sizeof(int) * np);
  memcpy(out->pidx, in->pidx, sizeof(int) * in->pptr[np]);
  memcpy(out->vidx, in->vidx, sizeof(int) * in->vptr[np]);
}

/* vanka.cpp:47-60 -- dense restriction through a scatter map (assignment,
 * missing entries stay 0) */
static void gather_dense(const or_csr* k, const int* rows, int nr, const int* cols, int nc,
                         int* scatter, double* d) {
  memset(d, 0, sizeof(double) * (size_t)nr * nc);
  for (int c = 0; c < nc; ++c) scatter[cols[c]] = c;
  for (int r = 0; r < nr; ++r) {
    const int row = rows[r];
    for (int q = k->rp[row]; q < k->rp[row + 1]; ++q) {
      const int loc = scatter[k->ci[q]];
      if (loc >= 0) d[(size_t)r * nc + loc] = k->v[q];
    }
  }
  for (int c = 0; c < nc; ++c) scatter[cols[c]] = -1;
}

/* vanka.cpp:64-149 */
int or_factor_patches(const or_csr* k, const or_patches* p, int n_u, or_vanka* f) {
  (void)n_u;
  memset(f, 0, sizeof *f);
  const int np_ = p->npatch;
  const int n = k->nrows;
  copy_patches(p, &f->pat);
  f->n = n;
  f->weights = XMALLOC(double, n);
  /* vanka.cpp:67-73 */
  for (int i = 0; i < np_; ++i) {
    for (int q = p->vptr[i]; q < p->vptr[i + 1]; ++q) f->weights[p->vidx[q]] += 1.0;
    for (int q = p->pptr[i]; q < p->pptr[i + 1]; ++q) f->weights[p->pidx[q]] += 1.0;
  }
  for (int d = 0; d < n; ++d)
    if (f->weights[d] > 0.0) f->weights[d] = 1.0 / f->weights[d];

  f->lu_off = XMALLOC(int64_t, np_ + 1);
  f->piv_off = XMALLOC(int64_t, np_ + 1);
  f->aux_off = XMALLOC(int64_t, np_ + 1);
  f->s_off = XMALLOC(int64_t, np_ + 1);
  for (int i = 0; i < np_; ++i) {
    const int nv = p->vptr[i + 1] - p->vptr[i];
    const int npp = p->pptr[i + 1] - p->pptr[i];
    const int nx = p->nx[i], ny = nv - nx;
    f->lu_off[i + 1] = f->lu_off[i] + (int64_t)nx * nx + (int64_t)ny * ny;
    f->piv_off[i + 1] = f->piv_off[i] + nv;
    f->aux_off[i + 1] = f->aux_off[i] + (int64_t)nv * npp;
    f->s_off[i + 1] = f->s_off[i] + (int64_t)npp * npp;
  }
  f->lu = XMALLOC(double, f->lu_off[np_]);
  f->piv = XMALLOC(int, f->piv_off[np_]);
  f->uhat = XMALLOC(double, f->aux_off[np_]);
  f->bhat = XMALLOC(double, f->aux_off[np_]);
  f->sinv = XMALLOC(double, f->s_off[np_]);

  int* scatter = XMALLOC(int, n);
  for (int d = 0; d < n; ++d) scatter[d] = -1;
  int maxv = 1, maxp = 1;
  for (int i = 0; i < np_; ++i) {
    const int nv = p->vptr[i + 1] - p->vptr[i];
    const int npp = p->pptr[i + 1] - p->pptr[i];
    if (nv > maxv) maxv = nv;
    if (npp > maxp) maxp = npp;
  }
  double* b = XMALLOC(double, (size_t)maxp * maxv);
  double* col = XMALLOC(double, maxv > maxp ? maxv : maxp);
  double* s = XMALLOC(double, (size_t)maxp * maxp);
  int* spiv = XMALLOC(int, maxp);
  int rc = OR_OK;

  for (int i = 0; i < np_ && rc == OR_OK; ++i) {
    const int* vel = p->vidx + p->vptr[i];
    const int* pres = p->pidx + p->pptr[i];
    const int nv = p->vptr[i + 1] - p->vptr[i];
    const int npp = p->pptr[i + 1] - p->pptr[i];
    const int nx = p->nx[i], ny = nv - nx;
    double* lux = f->lu + f->lu_off[i];
    double* luy = lux + (size_t)nx * nx;
    int* pivx = f->piv + f->piv_off[i];
    int* pivy = pivx + nx;
    /* vanka.cpp:88-96 */
    if (nx > 0) {
      gather_dense(k, vel, nx, vel, nx, scatter, lux);
      if (or_lu_factor(nx, lux, pivx) != OR_OK) {
        rc = fail(OR_SINGULAR_PATCH, "factor_patches: singular velocity block");
        break;
      }
    }
    if (ny > 0) {
      gather_dense(k, vel + nx, ny, vel + nx, ny, scatter, luy);
      if (or_lu_factor(ny, luy, pivy) != OR_OK) {
        rc = fail(OR_SINGULAR_PATCH, "factor_patches: singular velocity block");
        break;
      }
    }
    gather_dense(k, pres, npp, vel, nv, scatter, b); /* np x nv, vanka.cpp:97 */
    double* uhat = f->uhat + f->aux_off[i];          /* nv x np */
    double* bhat = f->bhat + f->aux_off[i];          /* np x nv */
    double* sinv = f->sinv + f->s_off[i];            /* np x np */
    /* vanka.cpp:99-111: u_hat = -A^-1 B^T per component */
    for (int j = 0; j < npp; ++j) {
      for (int q = 0; q < nx; ++q) col[q] = -b[(size_t)j * nv + q];
      if (nx > 0) or_lu_solve(nx, lux, pivx, col);
      for (int q = 0; q < nx; ++q) uhat[(size_t)q * npp + j] = col[q];
      for (int q = 0; q < ny; ++q) col[q] = -b[(size_t)j * nv + nx + q];
      if (ny > 0) or_lu_solve(ny, luy, pivy, col);
      for (int q = 0; q < ny; ++q) uhat[(size_t)(nx + q) * npp + j] = col[q];
    }
    /* vanka.cpp:112-119: S = B u_hat */
    for (int a = 0; a < npp; ++a)
      for (int c = 0; c < npp; ++c) {
        double acc = 0.0;
        for (int m = 0; m < nv; ++m) acc += b[(size_t)a * nv + m] * uhat[(size_t)m * npp + c];
        s[a * npp + c] = acc;
      }
    if (or_lu_factor(npp, s, spiv) != OR_OK) {
      rc = fail(OR_SINGULAR_PATCH, "factor_patches: singular Schur block");
      break;
    }
    /* vanka.cpp:126-132: S^-1 from unit vectors */
    for (int j = 0; j < npp; ++j) {
      for (int q = 0; q < npp; ++q) col[q] = 0.0;
      col[j] = 1.0;
      or_lu_solve(npp, s, spiv, col);
      for (int q = 0; q < npp; ++q) sinv[q * npp + j] = col[q];
    }
    /* vanka.cpp:133-140: b_hat = S^-1 u_hat^T */
    for (int a = 0; a < npp; ++a)
      for (int c = 0; c < nv; ++c) {
        double acc = 0.0;
        for (int m = 0; m < npp; ++m) acc += sinv[a * npp + m] * uhat[(size_t)c * npp + m];
        bhat[(size_t)a * nv + c] = acc;
      }
    /* vanka.cpp:142-144 */
    f->a_factor_bytes += 8 * ((int64_t)nx * nx + (int64_t)ny * ny);
    f->aux_bytes += 8 * (2 * (int64_t)nv * npp + (int64_t)npp * npp);
    f->dense_inverse_bytes += 8 * (int64_t)(nv + npp) * (nv + npp);
  }
  free(scatter);
  free(b);
  free(col);
  free(s);
  free(spiv);
  if (rc != OR_OK) or_vanka_free(f);
  return rc;
}

void or_vanka_free(or_vanka* f) {
  or_patches_free(&f->pat);
  free(f->lu_off);
  free(f->aux_off);
  free(f->s_off);
  free(f->piv_off);
  free(f->lu);
  free(f->piv);
  free(f->uhat);
  free(f->bhat);
  free(f->sinv);
  free(f->weights);
  memset(f, 0, sizeof *f);
}

/* vanka.cpp:151-184 -- sequential patch order, delta += w * x */
void or_apply_vanka(const or_vanka* f, const double* r, double* delta) {
  const or_patches* p = &f->pat;
  memset(delta, 0, sizeof(double) * (size_t)f->n);
  int maxv = 1, maxp = 1;
  for (int i = 0; i < p->npatch; ++i) {
    if (p->vptr[i + 1] - p->vptr[i] > maxv) maxv = p->vptr[i + 1] - p->vptr[i];
    if (p->pptr[i + 1] - p->pptr[i] > maxp) maxp = p->pptr[i + 1] - p->pptr[i];
  }
  double* bu = XMALLOC(double, maxv);
  double* xu = XMALLOC(double, maxv);
  double* bp = XMALLOC(double, maxp);
  double* xp = XMALLOC(double, maxp);
  for (int i = 0; i < p->npatch; ++i) {
    const int* vel = p->vidx + p->vptr[i];
    const int* pres = p->pidx + p->pptr[i];
    const int nv = p->vptr[i + 1] - p->vptr[i];
    const int npp = p->pptr[i + 1] - p->pptr[i];
    const int nx = p->nx[i], ny = nv - nx;
    const double* lux = f->lu + f->lu_off[i];
    const double* luy = lux + (size_t)nx * nx;
    const int* pivx = f->piv + f->piv_off[i];
    const int* pivy = pivx + nx;
    const double* uhat = f->uhat + f->aux_off[i];
    const double* bhat = f->bhat + f->aux_off[i];
    const double* sinv = f->sinv + f->s_off[i];
    for (int q = 0; q < nv; ++q) bu[q] = r[vel[q]];
    for (int q = 0; q < npp; ++q) bp[q] = r[pres[q]];
    for (int q = 0; q < nv; ++q) xu[q] = bu[q];
    if (nx > 0) or_lu_solve(nx, lux, pivx, xu);
    if (ny > 0) or_lu_solve(ny, luy, pivy, xu + nx);
    for (int a = 0; a < npp; ++a) {
      double acc = 0.0;
      for (int j = 0; j < npp; ++j) acc += sinv[a * npp + j] * bp[j];
      for (int j = 0; j < nv; ++j) acc += bhat[(size_t)a * nv + j] * bu[j];
      xp[a] = acc;
    }
    for (int q = 0; q < nv; ++q) {
      double acc = xu[q];
      for (int j = 0; j < npp; ++j) acc += uhat[(size_t)q * npp + j] * xp[j];
      delta[vel[q]] += f->weights[vel[q]] * acc;
    }
    for (int a = 0; a < npp; ++a) delta[pres[a]] += f->weights[pres[a]] * xp[a];
  }
  free(bu);
  free(xu);
  free(bp);
  free(xp);
}

/* ------------------------------------------ 3 components (config 5) --- */
/* vanka.cpp:11-42 with one seed and three velocity blocks */
int or_build_patches3(const or_csr* k, int n_x, int n_y, int n_z, int n_p, or_patches3* out) {
  const int n_u = n_x + n_y + n_z;
  memset(out, 0, sizeof *out);
  if (n_p < 0 || k->nrows != n_u + n_p)
    return fail(OR_DIM, "build_patches3: block sizes do not match K");
  out->npatch = n_p;
  out->pptr = XMALLOC(int, n_p + 1);
  out->pidx = XMALLOC(int, n_p);
  out->vptr = XMALLOC(int, n_p + 1);
  out->cnt = XMALLOC(int, 3 * (int64_t)n_p);
  int64_t cap = 0;
  for (int p0 = 0; p0 < n_p; ++p0) cap += k->rp[n_u + p0 + 1] - k->rp[n_u + p0];
  out->vidx = XMALLOC(int, cap > 0 ? cap : 1);
  int vv = 0;
  for (int i = 0; i < n_p; ++i) {
    const int row = n_u + i, start = vv;
    out->pptr[i] = i;
    out->pidx[i] = row;
    for (int q = k->rp[row]; q < k->rp[row + 1]; ++q)  /* canonical row: sorted, unique */
      if (k->ci[q] < n_u) out->vidx[vv++] = k->ci[q];
    if (vv == start) {
      or_patches3_free(out);
      return fail(OR_SINGULAR_PATCH, "build_patches3: pressure row couples to no velocity DoFs");
    }
    int cx = 0, cy = 0;
    while (start + cx < vv && out->vidx[start + cx] < n_x) ++cx;
    while (start + cx + cy < vv && out->vidx[start + cx + cy] < n_x + n_y) ++cy;
    out->cnt[3 * i] = cx;
    out->cnt[3 * i + 1] = cy;
    out->cnt[3 * i + 2] = vv - start - cx - cy;
    out->vptr[i + 1] = vv;
  }
  out->pptr[n_p] = n_p;
  return OR_OK;
}

void or_patches3_free(or_patches3* p) {
  free(p->pptr);
  free(p->pidx);
  free(p->vptr);
  free(p->vidx);
  free(p->cnt);
  memset(p, 0, sizeof *p);
}

/* vanka.cpp:64-149 with three velocity blocks */
int or_factor_patches3(const or_csr* k, const or_patches3* p, or_vanka3* f) {
  memset(f, 0, sizeof *f);
  const int np_ = p->npatch, n = k->nrows;
  f->n = n;
  f->pat.npatch = np_;
  f->pat.pptr = XMALLOC(int, np_ + 1);
  f->pat.pidx = XMALLOC(int, np_ > 0 ? np_ : 1);
  f->pat.vptr = XMALLOC(int, np_ + 1);
  f->pat.vidx = XMALLOC(int, p->vptr[np_] > 0 ? p->vptr[np_] : 1);
  f->pat.cnt = XMALLOC(int, 3 * (size_t)(np_ > 0 ? np_ : 1));
  memcpy(f->pat.pptr, p->pptr, sizeof(int) * (np_ + 1));
  memcpy(f->pat.pidx, p->pidx, sizeof(int) * np_);
  memcpy(f->pat.vptr, p->vptr, sizeof(int) * (np_ + 1));
  memcpy(f->pat.vidx, p->vidx, sizeof(int) * p->vptr[np_]);
  memcpy(f->pat.cnt, p->cnt, sizeof(int) * 3 * np_);
  f->weights = XMALLOC(double, n);
  for (int i = 0; i < np_; ++i) {
    for (int q = p->vptr[i]; q < p->vptr[i + 1]; ++q) f->weights[p->vidx[q]] += 1.0;
    for (int q = p->pptr[i]; q < p->pptr[i + 1]; ++q) f->weights[p->pidx[q]] += 1.0;
  }
  for (int d = 0; d < n; ++d)
    if (f->weights[d] > 0.0) f->weights[d] = 1.0 / f->weights[d];
  f->lu_off = XMALLOC(int64_t, np_ + 1);
  f->piv_off = XMALLOC(int64_t, np_ + 1);
  f->aux_off = XMALLOC(int64_t, np_ + 1);
  f->s_off = XMALLOC(int64_t, np_ + 1);
  int maxv = 1, maxp = 1;
  for (int i = 0; i < np_; ++i) {
    const int nv = p->vptr[i + 1] - p->vptr[i], npp = p->pptr[i + 1] - p->pptr[i];
    int64_t sq = 0;
    for (int c = 0; c < 3; ++c) sq += (int64_t)p->cnt[3 * i + c] * p->cnt[3 * i + c];
    f->lu_off[i + 1] = f->lu_off[i] + sq;
    f->piv_off[i + 1] = f->piv_off[i] + nv;
    f->aux_off[i + 1] = f->aux_off[i] + (int64_t)nv * npp;
    f->s_off[i + 1] = f->s_off[i] + (int64_t)npp * npp;
    if (nv > maxv) maxv = nv;
    if (npp > maxp) maxp = npp;
  }
  f->lu = XMALLOC(double, f->lu_off[np_] > 0 ? f->lu_off[np_] : 1);
  f->piv = XMALLOC(int, f->piv_off[np_] > 0 ? f->piv_off[np_] : 1);
  f->uhat = XMALLOC(double, f->aux_off[np_] > 0 ? f->aux_off[np_] : 1);
  f->bhat = XMALLOC(double, f->aux_off[np_] > 0 ? f->aux_off[np_] : 1);
  f->sinv = XMALLOC(double, f->s_off[np_] > 0 ? f->s_off[np_] : 1);
  int* scatter = XMALLOC(int, n);
  for (int d = 0; d < n; ++d) scatter[d] = -1;
  double* b = XMALLOC(double, (size_t)maxp * maxv);
  double* col = XMALLOC(double, maxv > maxp ? maxv : maxp);
  double* s = XMALLOC(double, (size_t)maxp * maxp);
  int* spiv = XMALLOC(int, maxp);
  int rc = OR_OK;
  for (int i = 0; i < np_ && rc == OR_OK; ++i) {
    const int* vel = p->vidx + p->vptr[i];
    const int* pres = p->pidx + p->pptr[i];
    const int nv = p->vptr[i + 1] - p->vptr[i], npp = p->pptr[i + 1] - p->pptr[i];
    const int* cnt = p->cnt + 3 * i;
    double* lu[3];
    int* piv[3];
    int off[3] = {0, cnt[0], cnt[0] + cnt[1]};
    lu[0] = f->lu + f->lu_off[i];
    lu[1] = lu[0] + (size_t)cnt[0] * cnt[0];
    lu[2] = lu[1] + (size_t)cnt[1] * cnt[1];
    piv[0] = f->piv + f->piv_off[i];
    piv[1] = piv[0] + cnt[0];
    piv[2] = piv[1] + cnt[1];
    for (int c = 0; c < 3 && rc == OR_OK; ++c) {
      if (cnt[c] == 0) continue;
      gather_dense(k, vel + off[c], cnt[c], vel + off[c], cnt[c], scatter, lu[c]);
      if (or_lu_factor(cnt[c], lu[c], piv[c]) != OR_OK)
        rc = fail(OR_SINGULAR_PATCH, "factor_patches3: singular velocity block");
    }
    if (rc != OR_OK) break;
    gather_dense(k, pres, npp, vel, nv, scatter, b);
    double* uhat = f->uhat + f->aux_off[i];
    double* bhat = f->bhat + f->aux_off[i];
    double* sinv = f->sinv + f->s_off[i];
    for (int j = 0; j < npp; ++j)
      for (int c = 0; c < 3; ++c) {
        for (int q = 0; q < cnt[c]; ++q) col[q] = -b[(size_t)j * nv + off[c] + q];
        if (cnt[c] > 0) or_lu_solve(cnt[c], lu[c], piv[c], col);
        for (int q = 0; q < cnt[c]; ++q) uhat[(size_t)(off[c] + q) * npp + j] = col[q];
      }
    for (int a = 0; a < npp; ++a)
      for (int c = 0; c < npp; ++c) {
        double acc = 0.0;
        for (int m = 0; m < nv; ++m) acc += b[(size_t)a * nv + m] * uhat[(size_t)m * npp + c];
        s[a * npp + c] = acc;
      }
    if (or_lu_factor(npp, s, spiv) != OR_OK) {
      rc = fail(OR_SINGULAR_PATCH, "factor_patches3: singular Schur block");
      break;
    }
    for (int j = 0; j < npp; ++j) {
      for (int q = 0; q < npp; ++q) col[q] = 0.0;
      col[j] = 1.0;
      or_lu_solve(npp, s, spiv, col);
      for (int q = 0; q < npp; ++q) sinv[q * npp + j] = col[q];
    }
    for (int a = 0; a < npp; ++a)
      for (int c = 0; c < nv; ++c) {
        double acc = 0.0;
        for (int m = 0; m < npp; ++m) acc += sinv[a * npp + m] * uhat[(size_t)c * npp + m];
        bhat[(size_t)a * nv + c] = acc;
      }
  }
  free(scatter);
  free(b);
  free(col);
  free(s);
  free(spiv);
  if (rc != OR_OK) or_vanka3_free(f);
  return rc;
}

void or_vanka3_free(or_vanka3* f) {
  or_patches3_free(&f->pat);
  free(f->lu_off);
  free(f->piv_off);
  free(f->aux_off);
  free(f->s_off);
  free(f->lu);
  free(f->piv);
  free(f->uhat);
  free(f->bhat);
  free(f->sinv);
  free(f->weights);
  memset(f, 0, sizeof *f);
}

/* vanka.cpp:151-184 with three blocks, patch order, delta += w x */
void or_apply_vanka3(const or_vanka3* f, const double* r, double* delta) {
  const or_patches3* p = &f->pat;
  memset(delta, 0, sizeof(double) * (size_t)f->n);
  int maxv = 1, maxp = 1;
  for (int i = 0; i < p->npatch; ++i) {
    if (p->vptr[i + 1] - p->vptr[i] > maxv) maxv = p->vptr[i + 1] - p->vptr[i];
    if (p->pptr[i + 1] - p->pptr[i] > maxp) maxp = p->pptr[i + 1] - p->pptr[i];
  }
  double* bu = XMALLOC(double, maxv);
  double* xu = XMALLOC(double, maxv);
  double* bp = XMALLOC(double, maxp);
  double* xp = XMALLOC(double, maxp);
  for (int i = 0; i < p->npatch; ++i) {
    const int* vel = p->vidx + p->vptr[i];
    const int* pres = p->pidx + p->pptr[i];
    const int nv = p->vptr[i + 1] - p->vptr[i], npp = p->pptr[i + 1] - p->pptr[i];
    const int* cnt = p->cnt + 3 * i;
    const double* lu = f->lu + f->lu_off[i];
    const int* piv = f->piv + f->piv_off[i];
    const double* uhat = f->uhat + f->aux_off[i];
    const double* bhat = f->bhat + f->aux_off[i];
    const double* sinv = f->sinv + f->s_off[i];
    for (int q = 0; q < nv; ++q) bu[q] = r[vel[q]];
    for (int q = 0; q < npp; ++q) bp[q] = r[pres[q]];
    for (int q = 0; q < nv; ++q) xu[q] = bu[q];
    int off = 0;
    for (int c = 0; c < 3; ++c) {
      if (cnt[c] > 0) or_lu_solve(cnt[c], lu, piv, xu + off);
      lu += (size_t)cnt[c] * cnt[c];
      piv += cnt[c];
      off += cnt[c];
    }
    for (int a = 0; a < npp; ++a) {
      double acc = 0.0;
      for (int j = 0; j < npp; ++j) acc += sinv[a * npp + j] * bp[j];
      for (int j = 0; j < nv; ++j) acc += bhat[(size_t)a * nv + j] * bu[j];
      xp[a] = acc;
    }
    for (int q = 0; q < nv; ++q) {
      double acc = xu[q];
      for (int j = 0; j < npp; ++j) acc += uhat[(size_t)q * npp + j] * xp[j];
      delta[vel[q]] += f->weights[vel[q]] * acc;
    }
    for (int a = 0; a < npp; ++a) delta[pres[a]] += f->weights[pres[a]] * xp[a];
  }
  free(bu);
  free(xu);
  free(bp);
  free(xp);
}

/* ------------------------------------------------------------ krylov.cpp */

/* krylov.cpp:17-121 -- right-preconditioned FGMRES, MGS + Givens */
int or_fgmres(int n, or_op a, void* actx, const double* b, double* x, or_op prec, void* pctx,
              const or_fgmres_opts* opt, or_report* rep, double* hist, int cap) {
  int hlen = 0;
#define PUSH(v)                   \
  do {                            \
    if (hist && hlen < cap) hist[hlen] = (v); \
    ++hlen;                       \
  } while (0)
  or_report R = {0, 0, 0.0, 0};
  const double bnorm = or_norm2(n, b);
  const double ref = bnorm > 0.0 ? bnorm : 1.0;
  double* ax = XMALLOC(double, n);
  double* r = XMALLOC(double, n);
  a(actx, x, ax);
  for (int i = 0; i < n; ++i) r[i] = b[i] - ax[i];
  double rnorm = or_norm2(n, r);
  PUSH(rnorm);
  if (rnorm / ref <= opt->tol) {
    R.converged = 1;
    R.final_relative_residual = rnorm / ref;
    R.history_len = hlen;
    if (rep) *rep = R;
    free(ax);
    free(r);
    return OR_OK;
  }
  const int m = opt->restart;
  double** v = XMALLOC(double*, m + 1);
  double** z = XMALLOC(double*, m);
  for (int i = 0; i <= m; ++i) v[i] = XMALLOC(double, n);
  for (int i = 0; i < m; ++i) z[i] = XMALLOC(double, n);
  double* w = XMALLOC(double, n);
  double* h = XMALLOC(double, (size_t)(m + 1) * m);
  double* cs = XMALLOC(double, m);
  double* sn = XMALLOC(double, m);
  double* g = XMALLOC(double, m + 1);
  double* y = XMALLOC(double, m);

  while (R.iterations < opt->max_iters) {
    a(actx, x, ax);
    for (int i = 0; i < n; ++i) r[i] = b[i] - ax[i];
    rnorm = or_norm2(n, r);
    if (rnorm / ref <= opt->tol) {
      R.converged = 1;
      break;
    }
    for (int i = 0; i < n; ++i) v[0][i] = r[i] / rnorm;
    for (int i = 0; i <= m; ++i) g[i] = 0.0;
    g[0] = rnorm;
    int j = 0;
    for (; j < m && R.iterations < opt->max_iters; ++j) {
      for (int i = 0; i < n; ++i) z[j][i] = 0.0;
      prec(pctx, v[j], z[j]);
      a(actx, z[j], w);
      for (int i = 0; i <= j; ++i) {
        const double hij = or_dot(n, w, v[i]);
        h[i * m + j] = hij;
        for (int k = 0; k < n; ++k) w[k] -= hij * v[i][k];
      }
      const double wnorm = or_norm2(n, w);
      h[(j + 1) * m + j] = wnorm;
      const int breakdown = wnorm < opt->breakdown;
      if (!breakdown)
        for (int k = 0; k < n; ++k) v[j + 1][k] = w[k] / wnorm;
      for (int i = 0; i < j; ++i) {
        const double t = cs[i] * h[i * m + j] + sn[i] * h[(i + 1) * m + j];
        h[(i + 1) * m + j] = -sn[i] * h[i * m + j] + cs[i] * h[(i + 1) * m + j];
        h[i * m + j] = t;
      }
      const double denom = hypot(h[j * m + j], h[(j + 1) * m + j]);
      if (denom > 0.0) {
        cs[j] = h[j * m + j] / denom;
        sn[j] = h[(j + 1) * m + j] / denom;
      } else {
        cs[j] = 1.0;
        sn[j] = 0.0;
      }
      h[j * m + j] = cs[j] * h[j * m + j] + sn[j] * h[(j + 1) * m + j];
      h[(j + 1) * m + j] = 0.0;
      g[j + 1] = -sn[j] * g[j];
      g[j] = cs[j] * g[j];
      ++R.iterations;
      rnorm = fabs(g[j + 1]);
      PUSH(rnorm);
      if (rnorm / ref <= opt->tol || breakdown) {
        ++j;
        break;
      }
    }
    for (int i = j - 1; i >= 0; --i) {
      double s = g[i];
      for (int k = i + 1; k < j; ++k) s -= h[i * m + k] * y[k];
      y[i] = s / h[i * m + i];
    }
    for (int i = 0; i < j; ++i)
      for (int k = 0; k < n; ++k) x[k] += y[i] * z[i][k];
    if (rnorm / ref <= opt->tol) {
      R.converged = 1;
      break;
    }
  }
  a(actx, x, ax);
  for (int i = 0; i < n; ++i) r[i] = b[i] - ax[i];
  R.final_relative_residual = or_norm2(n, r) / ref;
  if (R.final_relative_residual <= opt->tol) R.converged = 1;
  R.history_len = hlen;
  if (rep) *rep = R;
  for (int i = 0; i <= m; ++i) free(v[i]);
  for (int i = 0; i < m; ++i) free(z[i]);
  free(v);
  free(z);
  free(w);
  free(h);
  free(cs);
  free(sn);
  free(g);
  free(y);
  free(ax);
  free(r);
  return OR_OK;
#undef PUSH
}

static void op_spmv(void* ctx, const double* x, double* y) { or_spmv((const or_csr*)ctx, x, y); }
static void op_vanka(void* ctx, const double* x, double* y) {
  or_apply_vanka((const or_vanka*)ctx, x, y);
}

/* vanka.cpp:186-209 */
int or_vanka_relax(const or_csr* k, const or_vanka* f, double* x, const double* b, int mode,
                   int sweeps, double omega) {
  const int n = k->nrows;
  double* r = XMALLOC(double, n);
  if (mode == 1) {
    double* d = XMALLOC(double, n);
    for (int s = 0; s < sweeps; ++s) {
      or_spmv(k, x, r);
      for (int i = 0; i < n; ++i) r[i] = b[i] - r[i];
      or_apply_vanka(f, r, d);
      for (int i = 0; i < n; ++i) x[i] += omega * d[i];
    }
    free(d);
    free(r);
    return OR_OK;
  }
  or_spmv(k, x, r);
  for (int i = 0; i < n; ++i) r[i] = b[i] - r[i];
  double* corr = XMALLOC(double, n);
  or_fgmres_opts opt = {0.0, sweeps, sweeps, 1e-30};
  or_fgmres(n, op_spmv, (void*)k, r, corr, op_vanka, (void*)f, &opt, NULL, NULL, 0);
  for (int i = 0; i < n; ++i) x[i] += corr[i];
  free(corr);
  free(r);
  return OR_OK;
}

/* ---------------------------------------------------- preconditioner.cpp */

/* transpose (sparse.cpp:93-111), built once instead of per call (:72) */
typedef struct {
  or_csr m;
  int *rp, *ci;
  double* v;
} own_csr;

static void transpose_csr(const or_csr* a, own_csr* t) {
  const int nnz = a->rp[a->nrows];
  t->rp = XMALLOC(int, a->ncols + 1);
  t->ci = XMALLOC(int, nnz);
  t->v = XMALLOC(double, nnz);
  for (int q = 0; q < nnz; ++q) t->rp[a->ci[q] + 1]++;
  for (int c = 0; c < a->ncols; ++c) t->rp[c + 1] += t->rp[c];
  int* next = XMALLOC(int, a->ncols + 1);
  memcpy(next, t->rp, sizeof(int) * a->ncols);
  for (int r = 0; r < a->nrows; ++r)
    for (int q = a->rp[r]; q < a->rp[r + 1]; ++q) {
      const int c = a->ci[q];
      t->ci[next[c]] = r;
      t->v[next[c]] = a->v[q];
      ++next[c];
    }
  free(next);
  t->m.nrows = a->ncols;
  t->m.ncols = a->nrows;
  t->m.rp = t->rp;
  t->m.ci = t->ci;
  t->m.v = t->v;
}

/* preconditioner.cpp:40-55 */
int or_mono_setup(or_mono* m, int nlevels, const or_csr* ks, const or_csr* ps, const int* nxyz,
                  int enclosed) {
  memset(m, 0, sizeof *m);
  m->nlevels = nlevels;
  m->k = XMALLOC(or_csr, nlevels);
  m->p = XMALLOC(or_csr, nlevels);
  m->nxyz = XMALLOC(int, 3 * nlevels);
  m->vanka = XMALLOC(or_vanka, nlevels);
  memcpy(m->k, ks, sizeof(or_csr) * nlevels);
  if (nlevels > 1) memcpy(m->p, ps, sizeof(or_csr) * (nlevels - 1));
  memcpy(m->nxyz, nxyz, sizeof(int) * 3 * nlevels);
  for (int l = 0; l + 1 < nlevels; ++l) {
    or_patches pt;
    int rc = or_build_patches(&ks[l], nxyz[3 * l], nxyz[3 * l + 1], nxyz[3 * l + 2], 0, &pt);
    if (rc != OR_OK) return rc;
    rc = or_factor_patches(&ks[l], &pt, nxyz[3 * l] + nxyz[3 * l + 1], &m->vanka[l]);
    or_patches_free(&pt);
    if (rc != OR_OK) return rc;
  }
  const or_csr* bot = &ks[nlevels - 1];
  const int nc = bot->nrows;
  m->nc = nc;
  m->coarse_lu = XMALLOC(double, (size_t)nc * nc);
  m->coarse_piv = XMALLOC(int, nc);
  for (int r = 0; r < nc; ++r)
    for (int q = bot->rp[r]; q < bot->rp[r + 1]; ++q)
      m->coarse_lu[(size_t)r * nc + bot->ci[q]] += bot->v[q]; /* to_dense, sparse.cpp:269-277 */
  if (enclosed) {
    const int row = nxyz[3 * (nlevels - 1)] + nxyz[3 * (nlevels - 1) + 1];
    m->coarse_lu[(size_t)row * nc + row] += 1e-12 * or_norm_inf(&ks[0]);
  }
  return or_lu_factor(nc, m->coarse_lu, m->coarse_piv);
}

void or_mono_free(or_mono* m) {
  for (int l = 0; l + 1 < m->nlevels; ++l) or_vanka_free(&m->vanka[l]);
  free(m->k);
  free(m->p);
  free(m->nxyz);
  free(m->vanka);
  free(m->coarse_lu);
  free(m->coarse_piv);
  memset(m, 0, sizeof *m);
}

/* preconditioner.cpp:57-81 */
static void cycle_level(const or_mono* m, int level, const double* b, double* x, int nu1,
                        int nu2, int skip_finest) {
  if (level == m->nlevels - 1) {
    memcpy(x, b, sizeof(double) * m->nc);
    or_lu_solve(m->nc, m->coarse_lu, m->coarse_piv, x);
    return;
  }
  const or_csr* k = &m->k[level];
  const or_csr* p = &m->p[level];
  const int n = k->nrows;
  const int relax_here = !(level == 0 && skip_finest);
  if (relax_here && nu1 > 0) or_vanka_relax(k, &m->vanka[level], x, b, 0, nu1, 1.0);
  double* r = XMALLOC(double, n);
  or_spmv(k, x, r);
  for (int i = 0; i < n; ++i) r[i] = b[i] - r[i];
  own_csr pt;
  transpose_csr(p, &pt);
  double* rc = XMALLOC(double, p->ncols);
  double* xc = XMALLOC(double, p->ncols);
  or_spmv(&pt.m, r, rc);
  cycle_level(m, level + 1, rc, xc, nu1, nu2, skip_finest);
  double* corr = XMALLOC(double, n);
  or_spmv(p, xc, corr);
  for (int i = 0; i < n; ++i) x[i] += corr[i];
  if (relax_here && nu2 > 0) or_vanka_relax(k, &m->vanka[level], x, b, 0, nu2, 1.0);
  free(pt.rp);
  free(pt.ci);
  free(pt.v);
  free(r);
  free(rc);
  free(xc);
  free(corr);
}

static int vcycle_impl(const or_mono* m, const double* b, double* x, int nu1, int nu2,
                       int skip_finest) {
  memset(x, 0, sizeof(double) * m->k[0].nrows);
  cycle_level(m, 0, b, x, nu1, nu2, skip_finest);
  return OR_OK;
}

/* preconditioner.cpp:83-88 */
int or_vcycle(const or_mono* m, const double* b, double* x, int nu1, int nu2) {
  return vcycle_impl(m, b, x, nu1, nu2, 0);
}

/* preconditioner.cpp:90-105 (TH transfer only: transfer.cpp:70-80) */
int or_dc_setup(or_dc* d, const or_csr* k0, int n_x0, int n_y0, int n_p0, int sv, int nlevels,
                const or_csr* ks, const or_csr* ps, const int* nxyz, const or_config* cfg) {
  memset(d, 0, sizeof *d);
  if (sv) return fail(OR_ERROR, "oracle: SV mass-projection transfer is not restated");
  d->k0 = *k0;
  d->n_x0 = n_x0;
  d->n_y0 = n_y0;
  d->n_p0 = n_p0;
  d->stationary_fine = sv;
  d->cfg = *cfg;
  or_patches pt;
  int rc = or_build_patches(k0, n_x0, n_y0, n_p0, sv, &pt);
  if (rc != OR_OK) return rc;
  rc = or_factor_patches(k0, &pt, n_x0 + n_y0, &d->fine);
  or_patches_free(&pt);
  if (rc != OR_OK) return rc;
  return or_mono_setup(&d->mono, nlevels, ks, ps, nxyz, cfg->enclosed_flow);
}

void or_dc_free(or_dc* d) {
  or_vanka_free(&d->fine);
  or_mono_free(&d->mono);
}

/* preconditioner.cpp:114-153 */
int or_dc_apply(const or_dc* d, const double* r, double* z) {
  const int n = d->k0.nrows;
  const int n_u0 = d->n_x0 + d->n_y0;
  const or_config* c = &d->cfg;
  double* x = z;
  memset(x, 0, sizeof(double) * n);
  const int relax_fine = c->variant != 1;
  const int mode = d->stationary_fine ? 1 : 0;
  if (relax_fine && c->nu1 > 0) or_vanka_relax(&d->k0, &d->fine, x, r, mode, c->nu1, c->omega0);
  double* r1 = XMALLOC(double, n);
  if (relax_fine && c->nu1 > 0) {
    or_spmv(&d->k0, x, r1);
    for (int i = 0; i < n; ++i) r1[i] = r[i] - r1[i];
  } else {
    memcpy(r1, r, sizeof(double) * n);
  }
  /* transfer.cpp:127-135 then TH injection restrict_ (transfer.cpp:112-125) */
  double* rc = XMALLOC(double, n);
  for (int i = 0; i < n_u0; ++i) rc[i] = c->eta_u * r1[i];
  for (int i = n_u0; i < n; ++i) rc[i] = c->eta_p * r1[i];
  const or_csr* k1 = &d->mono.k[0];
  const int n1 = k1->nrows;
  double* e = XMALLOC(double, n1);
  double* res = XMALLOC(double, n1);
  double* de = XMALLOC(double, n1);
  const int skip_finest = c->variant == 2;
  for (int g = 0; g < c->gamma; ++g) {
    memcpy(res, rc, sizeof(double) * n1);
    if (g > 0) {
      or_spmv(k1, e, de);
      for (int i = 0; i < n1; ++i) res[i] -= de[i];
    }
    vcycle_impl(&d->mono, res, de, c->nu1, c->nu2, skip_finest);
    for (int i = 0; i < n1; ++i) e[i] += de[i];
  }
  /* prolong (transfer.cpp:97-110, TH copy) */
  for (int i = 0; i < n; ++i) x[i] += e[i];
  if (relax_fine && c->nu2 > 0) or_vanka_relax(&d->k0, &d->fine, x, r, mode, c->nu2, c->omega0);
  free(r1);
  free(rc);
  free(e);
  free(res);
  free(de);
  return OR_OK;
}

typedef struct {
  const or_dc* d;
  double* rp;
} prec_ctx;

static void project_pressure(const or_dc* d, double* v) {
  const int n_u = d->n_x0 + d->n_y0, n_p = d->n_p0;
  double mean = 0.0;
  for (int i = 0; i < n_p; ++i) mean += v[n_u + i];
  mean /= n_p;
  for (int i = 0; i < n_p; ++i) v[n_u + i] -= mean;
}

/* preconditioner.cpp:241-250 */
static void op_prec(void* ctx, const double* r, double* z) {
  prec_ctx* p = (prec_ctx*)ctx;
  const or_dc* d = p->d;
  if (d->cfg.enclosed_flow) {
    memcpy(p->rp, r, sizeof(double) * d->k0.nrows);
    project_pressure(d, p->rp);
    or_dc_apply(d, p->rp, z);
    project_pressure(d, z);
  } else {
    or_dc_apply(d, r, z);
  }
}

/* preconditioner.cpp:229-259 */
int or_solve_stokes(const or_dc* d, const double* rhs, double* x, or_report* rep, double* hist,
                    int cap) {
  const int n = d->k0.nrows;
  prec_ctx pc = {d, XMALLOC(double, n)};
  or_fgmres_opts opt = {d->cfg.tol, d->cfg.max_iters, d->cfg.restart, 1e-30};
  memset(x, 0, sizeof(double) * n);
  int rc = or_fgmres(n, op_spmv, (void*)&d->k0, rhs, x, op_prec, &pc, &opt, rep, hist, cap);
  free(pc.rp);
  return rc;
}
