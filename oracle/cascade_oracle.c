/*
 * cascade_oracle.c -- plain-C restatement of the reference EAM hot path.
 *
 * TEST INFRASTRUCTURE ONLY (see cascade_oracle.h).  Serial, worker count 1.
 * Every function restates a reference function in the same floating-point
 * operation order so that results are bit-identical to the reference built
 * with -ffp-contract=off (oracle/Makefile builds both that way and
 * tests/test_oracle_vs_ref.py pins the two against each other).
 *
 * Data layout differs on purpose: records live in a flat slot array plus a
 * key-sorted array of buckets instead of std::map, and ghost links are
 * (site, bucket index) pairs.
 *
 * Reference paths are relative to /root/reference/proj.
 */
#define _POSIX_C_SOURCE 200809L
#include "cascade_oracle.h"

#include <math.h>
#include <stdarg.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

/* ------------------------------------------------------------------ units */
/* core/include/cascademd/units.h:11-27 (same constant expressions) */
static const double ev_si = 1.602176634e-19;
static const double amu_si = 1.66053906660e-27;
static const double boltzmann_si = 1.380649e-23;
static const double angstrom_si = 1e-10;
static const double picosecond_si = 1e-12;
#define ACCEL_FACTOR ((ev_si / angstrom_si / amu_si) * (picosecond_si * picosecond_si) / angstrom_si)
static const double speed_factor = 98.22694750253277;
#define MV2_TO_EV (1.0 / ACCEL_FACTOR)
#define BOLTZMANN_EV (boltzmann_si / ev_si)

/* ------------------------------------------------------------------ types */
typedef struct { double x, y, z; } v3;
typedef struct {
  v3 pos, vel, force;
  double rho, df;
  uint64_t tag;
  uint16_t species;
  uint8_t valid, ghost;
} rec_t; /* AtomRecord, store.h:16-26 */

typedef struct { int64_t key; int n, cap; rec_t* r; } bucket_t;
typedef struct { int64_t id; int idx; } aref_t; /* AtomRef, store.h:30-33 */
typedef struct { aref_t image, source; } glink_t;

typedef struct {
  long bx, by, bz, g;
  double a0;
} box_t; /* BoxSpec, lattice.h:21-42 */

typedef struct { double x0, h; long nseg; double* seg; /* 7 per segment */ } spline_t;
typedef struct { double value, deriv; } seval_t;

typedef struct {
  int atomic_number;
  double mass, lattice_const, cutoff;
  spline_t embed, zr, dens;
  unsigned long long r_underflow, rho_clamp;
} pot_t;

typedef struct {
  double cutoff;
  long z_reach;
  int64_t *ef, *of, *eh, *oh;
  long nef, nof, neh, noh;
} offsets_t;

typedef struct { long z_lo, z_hi; } cblock_t;

struct orc_ctx {
  orc_config cfg;
  pot_t pot;
  box_t box;
  double index_cutoff;
  offsets_t idx;
  cblock_t blocks[2]; /* W = 1 colour partition: red, blue */
  rec_t* slots;
  long nslots;
  bucket_t* bk;
  int nbk, capbk;
  glink_t* links;
  long nlinks, caplinks;
  int64_t* ghost_ids;
  long nghost_ids;
  orc_state st;
  char err[512];
  /* defect series of the last orc_run (sim.h:69, series_) */
  double* ser_t;
  long* ser_d;
  long nser, capser;
};

static char g_create_err[512];

static int fail(orc_ctx* c, int code, const char* fmt, ...) {
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(c->err, sizeof c->err, fmt, ap);
  va_end(ap);
  return code;
}

static inline v3 v3sub(v3 a, v3 b) { v3 r = {a.x - b.x, a.y - b.y, a.z - b.z}; return r; }
static inline double norm2(v3 a) { return a.x * a.x + a.y * a.y + a.z * a.z; } /* vec3.h:14 */

/* ---------------------------------------------------------------- lattice */
static long total_x(const box_t* b) { return b->bx + 2 * b->g; }
static long total_y(const box_t* b) { return b->by + 2 * b->g; }
static long total_z(const box_t* b) { return b->bz + 2 * b->g; }
static long slot_count(const box_t* b) { return 2 * total_x(b) * total_y(b) * total_z(b); }
static double len_x(const box_t* b) { return b->bx * b->a0; }
static double len_y(const box_t* b) { return b->by * b->a0; }
static double len_z(const box_t* b) { return b->bz * b->a0; }

typedef struct { long x, y, z; } lc_t;

/* lattice.cpp:10-15 */
static int64_t coord_to_id(lc_t c, const box_t* b) {
  const long tx2 = 2 * total_x(b);
  return (int64_t)tx2 * total_y(b) * c.z + (int64_t)tx2 * c.y + c.x;
}
/* lattice.cpp:17-26 */
static lc_t id_to_coord(int64_t id, const box_t* b) {
  const long tx2 = 2 * total_x(b);
  lc_t c;
  c.x = (long)(id % tx2);
  id /= tx2;
  c.y = (long)(id % total_y(b));
  c.z = (long)(id / total_y(b));
  return c;
}
/* lattice.cpp:28-32 */
static int coord_in_box(lc_t c, const box_t* b) {
  return c.x >= 0 && c.x < 2 * total_x(b) && c.y >= 0 && c.y < total_y(b) && c.z >= 0 &&
         c.z < total_z(b);
}
/* lattice.cpp:34-43 */
static int is_ghost_c(lc_t c, const box_t* b) {
  const long g = b->g;
  return c.x < 2 * g || c.x >= 2 * (g + b->bx) || c.y < g || c.y >= g + b->by || c.z < g ||
         c.z >= g + b->bz;
}
static int is_ghost_id(int64_t id, const box_t* b) { return is_ghost_c(id_to_coord(id, b), b); }

/* lattice.cpp:45-52 */
static v3 site_position(lc_t c, const box_t* b) {
  const double a = b->a0;
  v3 p;
  if (c.x % 2 == 0) {
    p.x = 0.5 * c.x * a;
    p.y = c.y * a;
    p.z = c.z * a;
  } else {
    p.x = 0.5 * (c.x - 1) * a + 0.5 * a;
    p.y = c.y * a + 0.5 * a;
    p.z = c.z * a + 0.5 * a;
  }
  return p;
}

/* lattice.cpp:58-62: halves round toward -inf */
static inline long rhd(double t) { return (long)ceil(t - 0.5); }
static inline double sq(double v) { return v * v; }
static inline long clampl(long v, long lo, long hi) { return v < lo ? lo : (v > hi ? hi : v); }

/* lattice.cpp:66-89 (unclamped) */
static lc_t nearest_site_coord(v3 p, double a0) {
  const double fx = p.x / a0, fy = p.y / a0, fz = p.z / a0;
  const long ci = rhd(fx), cj = rhd(fy), ck = rhd(fz);
  const double dc = sq(fx - ci) + sq(fy - cj) + sq(fz - ck);
  const long bi = rhd(fx - 0.5), bj = rhd(fy - 0.5), bk = rhd(fz - 0.5);
  const double db = sq(fx - bi - 0.5) + sq(fy - bj - 0.5) + sq(fz - bk - 0.5);
  lc_t corner = {2 * ci, cj, ck}, center = {2 * bi + 1, bj, bk};
  if (dc < db) return corner;
  if (db < dc) return center;
  if (corner.z != center.z) return corner.z < center.z ? corner : center;
  if (corner.y != center.y) return corner.y < center.y ? corner : center;
  return corner.x < center.x ? corner : center;
}

/* lattice.cpp:99-131 (clamped; -1 = domain error) */
static int64_t nearest_site(v3 p, const box_t* b) {
  const double a = b->a0;
  if (p.x < 0.0 || p.x >= total_x(b) * a || p.y < 0.0 || p.y >= total_y(b) * a ||
      p.z < 0.0 || p.z >= total_z(b) * a)
    return -1;
  const double fx = p.x / a, fy = p.y / a, fz = p.z / a;
  const long ci = clampl(rhd(fx), 0, total_x(b) - 1);
  const long cj = clampl(rhd(fy), 0, total_y(b) - 1);
  const long ck = clampl(rhd(fz), 0, total_z(b) - 1);
  const double dc = sq(fx - ci) + sq(fy - cj) + sq(fz - ck);
  const long bi = clampl(rhd(fx - 0.5), 0, total_x(b) - 1);
  const long bj = clampl(rhd(fy - 0.5), 0, total_y(b) - 1);
  const long bk = clampl(rhd(fz - 0.5), 0, total_z(b) - 1);
  const double db = sq(fx - bi - 0.5) + sq(fy - bj - 0.5) + sq(fz - bk - 0.5);
  lc_t corner = {2 * ci, cj, ck}, center = {2 * bi + 1, bj, bk};
  if (dc < db) return coord_to_id(corner, b);
  if (db < dc) return coord_to_id(center, b);
  const int64_t a1 = coord_to_id(corner, b), a2 = coord_to_id(center, b);
  return a1 < a2 ? a1 : a2;
}

static int domain_fail(orc_ctx* c, v3 p) {
  return fail(c, ORC_DOMAIN,
              "nearest_site: position (%f, %f, %f) outside the ghost-inclusive box volume", p.x,
              p.y, p.z);
}

/* ------------------------------------------------------------ offsets */
typedef struct { int64_t off; long dz; } cand_t;
static int cand_cmp(const void* a, const void* b) {
  const int64_t x = ((const cand_t*)a)->off, y = ((const cand_t*)b)->off;
  return x < y ? -1 : (x > y ? 1 : 0);
}

/* neighbors.cpp:11-87 */
static int build_offsets(orc_ctx* c, double cutoff) {
  const box_t* b = &c->box;
  if (!(cutoff > 0.0)) return fail(c, ORC_INVALID, "build_offsets: cutoff must be positive");
  if (cutoff > (double)b->g * b->a0)
    return fail(c, ORC_INVALID,
                "build_offsets: cutoff %f A exceeds the ghost reach ghost_width*a0 = %f A",
                cutoff, b->g * b->a0);
  offsets_t* ix = &c->idx;
  ix->cutoff = cutoff;
  ix->z_reach = 0;
  const long reach = (long)ceil(cutoff / b->a0) + 1;
  const double c2 = cutoff * cutoff;
  const long tx2 = 2 * total_x(b);
  const int64_t sy = tx2, sz = (int64_t)tx2 * total_y(b);
  const long w = 2 * reach + 1;
  cand_t* ev = malloc(sizeof(cand_t) * 2 * w * w * w);
  cand_t* od = malloc(sizeof(cand_t) * 2 * w * w * w);
  long ne = 0, no = 0;
  for (long dz = -reach; dz <= reach; ++dz)
    for (long dy = -reach; dy <= reach; ++dy)
      for (long dx = -reach; dx <= reach; ++dx) {
        {
          const double d2 = (double)(dx * dx + dy * dy + dz * dz) * b->a0 * b->a0;
          if (d2 <= c2 && !(dx == 0 && dy == 0 && dz == 0)) {
            const int64_t off = sz * dz + sy * dy + 2 * dx;
            ev[ne].off = off; ev[ne++].dz = dz;
            od[no].off = off; od[no++].dz = dz;
          }
        }
        {
          const double hx = dx + 0.5, hy = dy + 0.5, hz = dz + 0.5;
          const double d2 = (hx * hx + hy * hy + hz * hz) * b->a0 * b->a0;
          if (d2 <= c2) { ev[ne].off = sz * dz + sy * dy + (2 * dx + 1); ev[ne++].dz = dz; }
        }
        {
          const double hx = dx - 0.5, hy = dy - 0.5, hz = dz - 0.5;
          const double d2 = (hx * hx + hy * hy + hz * hz) * b->a0 * b->a0;
          if (d2 <= c2) { od[no].off = sz * dz + sy * dy + (2 * dx - 1); od[no++].dz = dz; }
        }
      }
  qsort(ev, ne, sizeof(cand_t), cand_cmp);
  qsort(od, no, sizeof(cand_t), cand_cmp);
  ix->ef = malloc(sizeof(int64_t) * (ne + 1)); ix->eh = malloc(sizeof(int64_t) * (ne + 1));
  ix->of = malloc(sizeof(int64_t) * (no + 1)); ix->oh = malloc(sizeof(int64_t) * (no + 1));
  ix->nef = ix->neh = ix->nof = ix->noh = 0;
  for (long i = 0; i < ne; ++i) {
    ix->ef[ix->nef++] = ev[i].off;
    if (ev[i].off > 0) {
      ix->eh[ix->neh++] = ev[i].off;
      if (ev[i].dz > ix->z_reach) ix->z_reach = ev[i].dz;
    }
  }
  for (long i = 0; i < no; ++i) {
    ix->of[ix->nof++] = od[i].off;
    if (od[i].off > 0) {
      ix->oh[ix->noh++] = od[i].off;
      if (od[i].dz > ix->z_reach) ix->z_reach = od[i].dz;
    }
  }
  free(ev);
  free(od);
  return ORC_OK;
}

/* ------------------------------------------------------------- splines */
/* spline.cpp:14-77 */
static int build_spline(orc_ctx* c, double x0, double h, const double* y, long n, spline_t* s) {
  if (n < 4) return fail(c, ORC_INVALID, "build_spline: need at least 4 knots, got %ld", n);
  if (!(h > 0.0) || !isfinite(h) || !isfinite(x0))
    return fail(c, ORC_INVALID, "build_spline: non-finite or non-positive grid");
  for (long i = 0; i < n; ++i)
    if (!isfinite(y[i])) return fail(c, ORC_INVALID, "build_spline: non-finite knot value");
  double* r = calloc(n, sizeof(double));
  double* m = calloc(n, sizeof(double));
  const double inv_h2 = 1.0 / (h * h);
  for (long i = 1; i + 1 < n; ++i) r[i] = 6.0 * (y[i + 1] - 2.0 * y[i] + y[i - 1]) * inv_h2;
  m[1] = r[1] / 6.0;
  m[n - 2] = r[n - 2] / 6.0;
  if (n > 4) {
    const long lo = 2, hi = n - 3, cnt = hi - lo + 1;
    double* diag = malloc(sizeof(double) * cnt);
    double* rhs = malloc(sizeof(double) * cnt);
    for (long k = 0; k < cnt; ++k) { diag[k] = 4.0; rhs[k] = r[lo + k]; }
    rhs[0] -= m[1];
    rhs[cnt - 1] -= m[n - 2];
    for (long k = 1; k < cnt; ++k) {
      const double w = 1.0 / diag[k - 1];
      diag[k] -= w;
      rhs[k] -= w * rhs[k - 1];
    }
    m[lo + cnt - 1] = rhs[cnt - 1] / diag[cnt - 1];
    for (long k = cnt - 1; k-- > 0;) m[lo + k] = (rhs[k] - m[lo + k + 1]) / diag[k];
    free(diag);
    free(rhs);
  }
  m[0] = 2.0 * m[1] - m[2];
  m[n - 1] = 2.0 * m[n - 2] - m[n - 3];
  s->x0 = x0;
  s->h = h;
  s->nseg = n - 1;
  s->seg = malloc(sizeof(double) * 7 * (n - 1));
  for (long i = 0; i + 1 < n; ++i) {
    double* g = s->seg + 7 * i;
    g[0] = (m[i + 1] - m[i]) / (6.0 * h);
    g[1] = 0.5 * m[i];
    g[2] = (y[i + 1] - y[i]) / h - h * (2.0 * m[i] + m[i + 1]) / 6.0;
    g[3] = y[i];
    g[4] = 3.0 * g[0];
    g[5] = 2.0 * g[1];
    g[6] = g[2];
  }
  free(r);
  free(m);
  return ORC_OK;
}

static double x_last(const spline_t* s) { return s->x0 + s->h * (double)s->nseg; }

/* spline.cpp:79-93 */
static seval_t spline_eval(const spline_t* s, double x) {
  const double last = x_last(s);
  if (x < s->x0) x = s->x0;
  if (x > last) x = last;
  const double u = (x - s->x0) / s->h;
  long i = (long)u;
  if (i < 0) i = 0;
  if (i >= s->nseg) i = s->nseg - 1;
  const double t = x - (s->x0 + s->h * (double)i);
  const double* g = s->seg + 7 * i;
  seval_t e = {((g[0] * t + g[1]) * t + g[2]) * t + g[3], (g[4] * t + g[5]) * t + g[6]};
  return e;
}

/* potential.cpp:11-17 */
static seval_t pot_density(pot_t* p, double r) {
  if (r < p->dens.x0) { p->r_underflow++; r = p->dens.x0; }
  return spline_eval(&p->dens, r);
}
/* potential.cpp:19-31 (r > 0 guaranteed by the overlap check of every caller) */
static seval_t pot_pair(pot_t* p, double r) {
  if (r < p->zr.x0) { p->r_underflow++; r = p->zr.x0; }
  else if (r > p->cutoff) r = p->cutoff;
  const seval_t z = spline_eval(&p->zr, r);
  seval_t e = {z.value / r, (z.deriv * r - z.value) / (r * r)};
  return e;
}
/* potential.cpp:33-38 */
static seval_t pot_embedding(pot_t* p, double rho) {
  if (rho < p->embed.x0 || rho > x_last(&p->embed)) p->rho_clamp++;
  return spline_eval(&p->embed, rho);
}

/* ------------------------------------------------------- potential file */
/* potential.cpp:40-185: funcfl tokenizer with line-numbered errors */
typedef struct {
  FILE* f;
  const char* path;
  int line;
  char buf[1 << 16];
  char* tok;
  char* save;
} reader_t;

static int rd_line(reader_t* r, char* out, size_t n) {
  if (!fgets(out, (int)n, r->f)) return 0;
  r->line++;
  return 1;
}
static int rd_token(reader_t* r, char** tok) {
  for (;;) {
    if (r->tok) {
      char* t = r->tok;
      r->tok = strtok_r(NULL, " \t\r\n", &r->save);
      *tok = t;
      return 1;
    }
    if (!fgets(r->buf, sizeof r->buf, r->f)) return 0;
    r->line++;
    r->tok = strtok_r(r->buf, " \t\r\n", &r->save);
  }
}

static int read_block(orc_ctx* c, reader_t* r, long n, const char* what, double** out) {
  double* v = malloc(sizeof(double) * n);
  for (long i = 0; i < n; ++i) {
    char* tok;
    if (!rd_token(r, &tok)) {
      free(v);
      return fail(c, ORC_RUNTIME, "%s:%d: table %s ends early: expected %ld values, found %ld",
                  r->path, r->line, what, n, i);
    }
    char* end;
    const double x = strtod(tok, &end);
    if (*end != '\0' || !isfinite(x)) {
      free(v);
      return fail(c, ORC_RUNTIME, "%s:%d: non-numeric entry in %s table: '%s'", r->path,
                  r->line, what, tok);
    }
    v[i] = x;
  }
  *out = v;
  return ORC_OK;
}

static int parse_potential(orc_ctx* c, const char* path) {
  reader_t r;
  memset(&r, 0, sizeof r);
  r.path = path;
  r.f = fopen(path, "r");
  if (!r.f) return fail(c, ORC_RUNTIME, "cannot open potential file '%s'", path);
  pot_t* p = &c->pot;
  char line[4096];
  int rc = ORC_OK;
  double *fv = NULL, *zv = NULL, *dv = NULL;
  if (!rd_line(&r, line, sizeof line)) { rc = fail(c, ORC_RUNTIME, "%s:%d: unexpected end of file", path, r.line); goto out; }
  if (!rd_line(&r, line, sizeof line)) { rc = fail(c, ORC_RUNTIME, "%s:%d: unexpected end of file", path, r.line); goto out; }
  {
    double z, mass, a0;
    char name[256];
    if (sscanf(line, "%lf %lf %lf %255s", &z, &mass, &a0, name) != 4) {
      rc = fail(c, ORC_RUNTIME, "%s:%d: element line needs: atomic-number mass lattice-constant name", path, r.line);
      goto out;
    }
    if (z < 1.0 || z != floor(z)) { rc = fail(c, ORC_RUNTIME, "%s:%d: atomic number must be a positive integer", path, r.line); goto out; }
    if (!(mass > 0.0)) { rc = fail(c, ORC_RUNTIME, "%s:%d: mass must be positive", path, r.line); goto out; }
    if (!(a0 > 0.0)) { rc = fail(c, ORC_RUNTIME, "%s:%d: lattice constant must be positive", path, r.line); goto out; }
    p->atomic_number = (int)z;
    p->mass = mass;
    p->lattice_const = a0;
  }
  long nrho, nr;
  double drho, dr;
  if (!rd_line(&r, line, sizeof line)) { rc = fail(c, ORC_RUNTIME, "%s:%d: unexpected end of file", path, r.line); goto out; }
  if (sscanf(line, "%ld %lf %ld %lf %lf", &nrho, &drho, &nr, &dr, &p->cutoff) != 5) {
    rc = fail(c, ORC_RUNTIME, "%s:%d: grid line needs: Nrho drho Nr dr cutoff", path, r.line);
    goto out;
  }
  if (nrho < 4 || nr < 4) { rc = fail(c, ORC_RUNTIME, "%s:%d: node counts must be at least 4 (cubic spline)", path, r.line); goto out; }
  if (!(drho > 0.0) || !(dr > 0.0)) { rc = fail(c, ORC_RUNTIME, "%s:%d: grid spacings must be positive", path, r.line); goto out; }
  if (!(p->cutoff > 0.0)) { rc = fail(c, ORC_RUNTIME, "%s:%d: cutoff must be positive", path, r.line); goto out; }
  if (fabs((double)nr * dr - p->cutoff) > 1e-9) { rc = fail(c, ORC_RUNTIME, "%s:%d: cutoff does not match the r-table extent Nr*dr", path, r.line); goto out; }
  if ((rc = read_block(c, &r, nrho, "embedding", &fv))) goto out;
  if ((rc = read_block(c, &r, nr, "pair z(r)", &zv))) goto out;
  if ((rc = read_block(c, &r, nr, "density", &dv))) goto out;
  {
    char* extra;
    if (rd_token(&r, &extra)) { rc = fail(c, ORC_RUNTIME, "%s:%d: trailing data after the tables: '%s'", path, r.line, extra); goto out; }
  }
  if ((rc = build_spline(c, 0.0, drho, fv, nrho, &p->embed))) goto out;
  if ((rc = build_spline(c, dr, dr, zv, nr, &p->zr))) goto out;
  if ((rc = build_spline(c, dr, dr, dv, nr, &p->dens))) goto out;
out:
  free(fv);
  free(zv);
  free(dv);
  fclose(r.f);
  return rc;
}

/* ----------------------------------------------------------- the store */
static bucket_t* bk_find(orc_ctx* c, int64_t key) {
  int lo = 0, hi = c->nbk - 1;
  while (lo <= hi) {
    const int mid = (lo + hi) / 2;
    if (c->bk[mid].key == key) return &c->bk[mid];
    if (c->bk[mid].key < key) lo = mid + 1; else hi = mid - 1;
  }
  return NULL;
}
static bucket_t* bk_get(orc_ctx* c, int64_t key) {
  int lo = 0, hi = c->nbk;
  while (lo < hi) {
    const int mid = (lo + hi) / 2;
    if (c->bk[mid].key < key) lo = mid + 1; else hi = mid;
  }
  if (lo < c->nbk && c->bk[lo].key == key) return &c->bk[lo];
  if (c->nbk == c->capbk) {
    c->capbk = c->capbk ? 2 * c->capbk : 16;
    c->bk = realloc(c->bk, sizeof(bucket_t) * c->capbk);
  }
  memmove(&c->bk[lo + 1], &c->bk[lo], sizeof(bucket_t) * (c->nbk - lo));
  c->nbk++;
  c->bk[lo].key = key;
  c->bk[lo].n = c->bk[lo].cap = 0;
  c->bk[lo].r = NULL;
  return &c->bk[lo];
}
static int bk_push(bucket_t* b, const rec_t* r) {
  if (b->n == b->cap) {
    b->cap = b->cap ? 2 * b->cap : 4;
    b->r = realloc(b->r, sizeof(rec_t) * b->cap);
  }
  b->r[b->n] = *r;
  return b->n++;
}
static void bk_clear_all(orc_ctx* c) {
  for (int i = 0; i < c->nbk; ++i) free(c->bk[i].r);
  c->nbk = 0;
}
static void bk_compact(orc_ctx* c) { /* drop empty buckets */
  int w = 0;
  for (int i = 0; i < c->nbk; ++i) {
    if (c->bk[i].n > 0) c->bk[w++] = c->bk[i];
    else free(c->bk[i].r);
  }
  c->nbk = w;
}

static rec_t* at_ref(orc_ctx* c, aref_t r) {
  if (r.idx < 0) return &c->slots[r.id];
  return &bk_find(c, r.id)->r[r.idx];
}

#define FOR_INTERIOR(b, ID)                                                        \
  for (long z_ = (b)->g; z_ < (b)->g + (b)->bz; ++z_)                              \
    for (long y_ = (b)->g; y_ < (b)->g + (b)->by; ++y_)                            \
      for (int64_t row_ = ((int64_t)z_ * total_y(b) + y_) * (2 * total_x(b)),      \
                   x_ = 2 * (b)->g;                                                \
           x_ < 2 * ((b)->g + (b)->bx); ++x_)                                      \
        for (int64_t ID = row_ + x_, once_ = 1; once_; once_ = 0)

/* store.cpp:29-42 */
static int store_insert(orc_ctx* c, const rec_t* in) {
  const int64_t id = nearest_site(in->pos, &c->box);
  if (id < 0) return domain_fail(c, in->pos);
  rec_t r = *in;
  r.valid = 1;
  r.ghost = 0;
  if (!c->slots[id].valid) { c->slots[id] = r; return ORC_OK; }
  bk_push(bk_get(c, id), &r);
  return ORC_OK;
}

/* store.cpp:44-76 */
typedef struct { int64_t key; long seq; rec_t r; } keep_t;
static int keep_cmp(const void* a, const void* b) {
  const keep_t *x = a, *y = b;
  if (x->key != y->key) return x->key < y->key ? -1 : 1;
  return x->seq < y->seq ? -1 : (x->seq > y->seq ? 1 : 0);
}
static int store_update_hash(orc_ctx* c) {
  const box_t* b = &c->box;
  FOR_INTERIOR(b, id) {
    rec_t* r = &c->slots[id];
    if (!r->valid || r->ghost) continue;
    const int64_t real = nearest_site(r->pos, b);
    if (real < 0) return domain_fail(c, r->pos);
    if (real != id) {
      bk_push(bk_get(c, real), r);
      r->valid = 0;
    }
  }
  long total = 0;
  for (int i = 0; i < c->nbk; ++i) total += c->bk[i].n;
  keep_t* keep = malloc(sizeof(keep_t) * (total + 1));
  long nk = 0;
  for (int i = 0; i < c->nbk; ++i) {
    bucket_t* bk = &c->bk[i];
    for (int j = 0; j < bk->n; ++j) {
      rec_t* r = &bk->r[j];
      if (r->ghost) { keep[nk].key = bk->key; keep[nk].seq = nk; keep[nk].r = *r; nk++; continue; }
      const int64_t real = nearest_site(r->pos, b);
      if (real < 0) { free(keep); return domain_fail(c, r->pos); }
      rec_t* slot = &c->slots[real];
      if (!slot->valid && !is_ghost_id(real, b)) *slot = *r;
      else { keep[nk].key = real; keep[nk].seq = nk; keep[nk].r = *r; nk++; }
    }
  }
  qsort(keep, nk, sizeof(keep_t), keep_cmp);
  bk_clear_all(c);
  for (long i = 0; i < nk; ++i) bk_push(bk_get(c, keep[i].key), &keep[i].r);
  free(keep);
  return ORC_OK;
}

static inline long floor_div(long a, long b) { /* store.cpp:80-84 */
  long q = a / b;
  if ((a % b != 0) && ((a < 0) != (b < 0))) --q;
  return q;
}

/* store.cpp:88-118 */
static int wrap_rec(orc_ctx* c, rec_t* r) {
  const box_t* b = &c->box;
  for (int pass = 0; pass < 4; ++pass) {
    const lc_t q = nearest_site_coord(r->pos, b->a0);
    const long kx = floor_div(q.x - 2 * b->g, 2 * b->bx);
    const long ky = floor_div(q.y - b->g, b->by);
    const long kz = floor_div(q.z - b->g, b->bz);
    if (kx == 0 && ky == 0 && kz == 0) return ORC_OK;
    r->pos.x -= (double)kx * len_x(b);
    r->pos.y -= (double)ky * len_y(b);
    r->pos.z -= (double)kz * len_z(b);
  }
  return fail(c, ORC_LOGIC, "canonicalize_positions: wrap did not converge");
}
static int store_canonicalize(orc_ctx* c) {
  const box_t* b = &c->box;
  int rc;
  FOR_INTERIOR(b, id) {
    rec_t* r = &c->slots[id];
    if (r->valid && !r->ghost && (rc = wrap_rec(c, r))) return rc;
  }
  for (int i = 0; i < c->nbk; ++i)
    for (int j = 0; j < c->bk[i].n; ++j)
      if (!c->bk[i].r[j].ghost && (rc = wrap_rec(c, &c->bk[i].r[j]))) return rc;
  return ORC_OK;
}

static void push_link(orc_ctx* c, aref_t img, aref_t src) {
  if (c->nlinks == c->caplinks) {
    c->caplinks = c->caplinks ? 2 * c->caplinks : 1024;
    c->links = realloc(c->links, sizeof(glink_t) * c->caplinks);
  }
  c->links[c->nlinks].image = img;
  c->links[c->nlinks].source = src;
  c->nlinks++;
}

/* store.cpp:160-182 */
static void emit_images(orc_ctx* c, const rec_t* rec, aref_t source, lc_t q, long kxm, long kym,
                        long kzm) {
  const box_t* b = &c->box;
  for (long kz = -kzm; kz <= kzm; ++kz)
    for (long ky = -kym; ky <= kym; ++ky)
      for (long kx = -kxm; kx <= kxm; ++kx) {
        if (kx == 0 && ky == 0 && kz == 0) continue;
        lc_t ci = {q.x + 2 * b->bx * kx, q.y + b->by * ky, q.z + b->bz * kz};
        if (!coord_in_box(ci, b)) continue;
        rec_t img = *rec;
        img.ghost = 1;
        img.pos.x += (double)kx * len_x(b);
        img.pos.y += (double)ky * len_y(b);
        img.pos.z += (double)kz * len_z(b);
        const int64_t iid = coord_to_id(ci, b);
        rec_t* slot = &c->slots[iid];
        aref_t ir;
        if (!slot->valid) {
          *slot = img;
          ir.id = iid; ir.idx = -1;
        } else {
          ir.id = iid;
          ir.idx = bk_push(bk_get(c, iid), &img);
        }
        push_link(c, ir, source);
      }
}

/* store.cpp:120-195 */
static int store_fill_ghosts(orc_ctx* c) {
  const box_t* b = &c->box;
  for (long i = 0; i < c->nghost_ids; ++i) c->slots[c->ghost_ids[i]].valid = 0;
  for (int i = 0; i < c->nbk; ++i) {
    bucket_t* bk = &c->bk[i];
    int w = 0;
    for (int j = 0; j < bk->n; ++j)
      if (!bk->r[j].ghost) bk->r[w++] = bk->r[j];
    bk->n = w;
  }
  bk_compact(c);
  c->nlinks = 0;
  const long g = b->g;
  if (g == 0) return ORC_OK;
  const long kxm = (g + b->bx - 1) / b->bx, kym = (g + b->by - 1) / b->by,
             kzm = (g + b->bz - 1) / b->bz;
  FOR_INTERIOR(b, id) {
    const rec_t* r = &c->slots[id];
    if (r->valid && !r->ghost) {
      aref_t src = {id, -1};
      rec_t copy = *r;
      emit_images(c, &copy, src, id_to_coord(id, b), kxm, kym, kzm);
    }
  }
  /* snapshot of (key, index) of interior buckets */
  long n = 0;
  for (int i = 0; i < c->nbk; ++i)
    if (!is_ghost_id(c->bk[i].key, b)) n += c->bk[i].n;
  aref_t* snap = malloc(sizeof(aref_t) * (n + 1));
  n = 0;
  for (int i = 0; i < c->nbk; ++i) {
    if (is_ghost_id(c->bk[i].key, b)) continue;
    for (int j = 0; j < c->bk[i].n; ++j) { snap[n].id = c->bk[i].key; snap[n].idx = j; n++; }
  }
  for (long i = 0; i < n; ++i) {
    const rec_t r = bk_find(c, snap[i].id)->r[snap[i].idx];
    if (!r.ghost) emit_images(c, &r, snap[i], id_to_coord(snap[i].id, b), kxm, kym, kzm);
  }
  free(snap);
  return ORC_OK;
}

/* store.cpp:197-210 */
static long store_atom_count(const orc_ctx* c) {
  const box_t* b = &c->box;
  long n = 0;
  FOR_INTERIOR(b, id) if (c->slots[id].valid && !c->slots[id].ghost) ++n;
  for (int i = 0; i < c->nbk; ++i) {
    if (is_ghost_id(c->bk[i].key, b)) continue;
    for (int j = 0; j < c->bk[i].n; ++j) if (!c->bk[i].r[j].ghost) ++n;
  }
  return n;
}

/* ------------------------------------------------------- force engine */
typedef struct {
  int hit;
  char detail[160];
} fatal_t; /* forces.cpp:17-38 */

static void fatal_report(fatal_t* f, const rec_t* a, const rec_t* b, double r2) {
  if (f->hit) return;
  f->hit = 1;
  snprintf(f->detail, sizeof f->detail, "atoms %llu and %llu overlap (separation %.3e A)",
           (unsigned long long)a->tag, (unsigned long long)b->tag, sqrt(r2));
}

static const double overlap_r2 = 1e-12; /* forces.cpp:14 */

static int check_cutoffs(orc_ctx* c) { /* forces.cpp:48-53 */
  if (c->idx.cutoff < c->pot.cutoff)
    return fail(c, ORC_INVALID, "offset index cutoff is smaller than the potential cutoff");
  return ORC_OK;
}

static void zero_rho(orc_ctx* c) { /* forces.cpp:87-94 */
  for (long i = 0; i < c->nslots; ++i) if (c->slots[i].valid) c->slots[i].rho = 0.0;
  for (int i = 0; i < c->nbk; ++i) for (int j = 0; j < c->bk[i].n; ++j) c->bk[i].r[j].rho = 0.0;
}
static void zero_force(orc_ctx* c) { /* forces.cpp:96-103 */
  const v3 z = {0, 0, 0};
  for (long i = 0; i < c->nslots; ++i) if (c->slots[i].valid) c->slots[i].force = z;
  for (int i = 0; i < c->nbk; ++i) for (int j = 0; j < c->bk[i].n; ++j) c->bk[i].r[j].force = z;
}

static const int64_t* half_list(const orc_ctx* c, int odd, long* n) {
  *n = odd ? c->idx.noh : c->idx.neh;
  return odd ? c->idx.oh : c->idx.eh;
}
static const int64_t* full_list(const orc_ctx* c, int odd, long* n) {
  *n = odd ? c->idx.nof : c->idx.nef;
  return odd ? c->idx.of : c->idx.ef;
}

/* forces.cpp:109-137 */
static void density_slots(orc_ctx* c, fatal_t* fat, long z_lo, long z_hi) {
  const box_t* b = &c->box;
  const long g = b->g, tx2 = 2 * total_x(b);
  const double cut2 = c->pot.cutoff * c->pot.cutoff;
  for (long z = z_lo; z < z_hi; ++z)
    for (long y = g; y < g + b->by; ++y) {
      const int64_t row = ((int64_t)z * total_y(b) + y) * tx2;
      for (long x = 2 * g; x < 2 * (g + b->bx); ++x) {
        const int64_t id = row + x;
        rec_t* a = &c->slots[id];
        if (!a->valid) continue;
        long nh;
        const int64_t* hl = half_list(c, (int)(x & 1), &nh);
        for (long k = 0; k < nh; ++k) {
          rec_t* p = &c->slots[id + hl[k]];
          if (!p->valid) continue;
          const v3 d = v3sub(a->pos, p->pos);
          const double r2 = norm2(d);
          if (r2 > cut2) continue;
          if (r2 < overlap_r2) { fatal_report(fat, a, p, r2); continue; }
          const double rho = pot_density(&c->pot, sqrt(r2)).value;
          a->rho += rho;
          p->rho += rho;
        }
      }
    }
}

/* forces.cpp:139-174 */
static double pair_slots(orc_ctx* c, fatal_t* fat, long z_lo, long z_hi) {
  const box_t* b = &c->box;
  const long g = b->g, tx2 = 2 * total_x(b);
  const double cut2 = c->pot.cutoff * c->pot.cutoff;
  double energy = 0.0;
  for (long z = z_lo; z < z_hi; ++z)
    for (long y = g; y < g + b->by; ++y) {
      const int64_t row = ((int64_t)z * total_y(b) + y) * tx2;
      for (long x = 2 * g; x < 2 * (g + b->bx); ++x) {
        const int64_t id = row + x;
        rec_t* a = &c->slots[id];
        if (!a->valid) continue;
        long nh;
        const int64_t* hl = half_list(c, (int)(x & 1), &nh);
        for (long k = 0; k < nh; ++k) {
          rec_t* p = &c->slots[id + hl[k]];
          if (!p->valid) continue;
          const v3 d = v3sub(a->pos, p->pos);
          const double r2 = norm2(d);
          if (r2 > cut2) continue;
          if (r2 < overlap_r2) { fatal_report(fat, a, p, r2); continue; }
          const double r = sqrt(r2);
          const seval_t ph = pot_pair(&c->pot, r);
          const seval_t de = pot_density(&c->pot, r);
          const double fp = -((a->df + p->df) * de.deriv + ph.deriv) / r;
          const v3 f = {d.x * fp, d.y * fp, d.z * fp};
          a->force.x += f.x; a->force.y += f.y; a->force.z += f.z;
          p->force.x -= f.x; p->force.y -= f.y; p->force.z -= f.z;
          energy += ph.value;
        }
      }
    }
  return energy;
}

/* forces.cpp:185-225: every pair with >= 1 clash atom, from the clash side.
 * mode 0: density, mode 1: force (returns energy) */
static double visit_clash(orc_ctx* c, fatal_t* fat, int mode) {
  const box_t* b = &c->box;
  const double cut2 = c->pot.cutoff * c->pot.cutoff;
  double energy = 0.0;
  for (int bi = 0; bi < c->nbk; ++bi) {
    const int64_t id = c->bk[bi].key;
    if (is_ghost_id(id, b)) continue;
    const int odd = (id_to_coord(id, b).x & 1) != 0;
    long nf;
    const int64_t* offs = full_list(c, odd, &nf);
    for (int i = 0; i < c->bk[bi].n; ++i) {
/* bucket storage never reallocates during the visit (no pushes) */
#define TRY_PAIR(P, SYM)                                                             \
  do {                                                                               \
    rec_t* atom = &c->bk[bi].r[i];                                                   \
    rec_t* pp = (P);                                                                 \
    const v3 d = v3sub(atom->pos, pp->pos);                                          \
    const double r2 = norm2(d);                                                      \
    if (r2 > cut2) break;                                                            \
    if (r2 < overlap_r2) { fatal_report(fat, atom, pp, r2); break; }                 \
    if (mode == 0) {                                                                 \
      const double rho = pot_density(&c->pot, sqrt(r2)).value;                       \
      atom->rho += rho;                                                              \
      if (SYM) pp->rho += rho;                                                       \
    } else {                                                                         \
      const double r = sqrt(r2);                                                     \
      const seval_t ph = pot_pair(&c->pot, r);                                       \
      const seval_t de = pot_density(&c->pot, r);                                    \
      const double fp = -((atom->df + pp->df) * de.deriv + ph.deriv) / r;            \
      const v3 f = {d.x * fp, d.y * fp, d.z * fp};                                   \
      atom->force.x += f.x; atom->force.y += f.y; atom->force.z += f.z;              \
      if (SYM) {                                                                     \
        pp->force.x -= f.x; pp->force.y -= f.y; pp->force.z -= f.z;                  \
        energy += ph.value;                                                          \
      } else {                                                                       \
        energy += 0.5 * ph.value;                                                    \
      }                                                                              \
    }                                                                                \
  } while (0)
      rec_t* own = &c->slots[id];
      if (own->valid) TRY_PAIR(own, 1);
      for (int j = i + 1; j < c->bk[bi].n; ++j) TRY_PAIR(&c->bk[bi].r[j], 1);
      for (long k = 0; k < nf; ++k) {
        const int64_t nid = id + offs[k];
        rec_t* slot = &c->slots[nid];
        if (slot->valid) TRY_PAIR(slot, 1);
        bucket_t* nb = bk_find(c, nid);
        if (!nb) continue;
        if (is_ghost_id(nid, b)) {
          for (int j = 0; j < nb->n; ++j) TRY_PAIR(&nb->r[j], 0);
        } else if (nid > id) {
          for (int j = 0; j < nb->n; ++j) TRY_PAIR(&nb->r[j], 1);
        }
      }
#undef TRY_PAIR
    }
  }
  return energy;
}

/* forces.cpp:256-275 */
static double embed_slots(orc_ctx* c, long z_lo, long z_hi) {
  const box_t* b = &c->box;
  const long g = b->g, tx2 = 2 * total_x(b);
  double energy = 0.0;
  for (long z = z_lo; z < z_hi; ++z)
    for (long y = g; y < g + b->by; ++y) {
      const int64_t row = ((int64_t)z * total_y(b) + y) * tx2;
      for (long x = 2 * g; x < 2 * (g + b->bx); ++x) {
        rec_t* a = &c->slots[row + x];
        if (!a->valid) continue;
        const seval_t em = pot_embedding(&c->pot, a->rho);
        a->df = em.deriv;
        energy += em.value;
      }
    }
  return energy;
}
/* forces.cpp:277-288 */
static double embed_clash(orc_ctx* c) {
  double energy = 0.0;
  for (int i = 0; i < c->nbk; ++i) {
    if (is_ghost_id(c->bk[i].key, &c->box)) continue;
    for (int j = 0; j < c->bk[i].n; ++j) {
      rec_t* a = &c->bk[i].r[j];
      const seval_t em = pot_embedding(&c->pot, a->rho);
      a->df = em.deriv;
      energy += em.value;
    }
  }
  return energy;
}
/* forces.cpp:290-309 */
static void fold_rho(orc_ctx* c) {
  for (long i = 0; i < c->nlinks; ++i)
    at_ref(c, c->links[i].source)->rho += at_ref(c, c->links[i].image)->rho;
}
static void refresh_ghosts(orc_ctx* c) {
  for (long i = 0; i < c->nlinks; ++i) {
    const rec_t* s = at_ref(c, c->links[i].source);
    rec_t* im = at_ref(c, c->links[i].image);
    im->rho = s->rho;
    im->df = s->df;
  }
}
static void fold_force(orc_ctx* c) {
  for (long i = 0; i < c->nlinks; ++i) {
    rec_t* s = at_ref(c, c->links[i].source);
    const rec_t* im = at_ref(c, c->links[i].image);
    s->force.x += im->force.x; s->force.y += im->force.y; s->force.z += im->force.z;
  }
}

/* forces.cpp:343-366 with workers = 1: two blocks, red then blue */
static void build_partition(orc_ctx* c) {
  const box_t* b = &c->box;
  const long nb = 2, base = b->bz / nb, rem = b->bz % nb;
  long z = b->g;
  for (long k = 0; k < nb; ++k) {
    const long t = base + (k < rem ? 1 : 0);
    c->blocks[k].z_lo = z;
    c->blocks[k].z_hi = z + t;
    z += t;
  }
}

/* forces.cpp:368-379 */
int orc_compute_density(orc_ctx* c) {
  int rc;
  if ((rc = check_cutoffs(c))) return rc;
  fatal_t fat = {0};
  zero_rho(c);
  density_slots(c, &fat, c->box.g, c->box.g + c->box.bz);
  visit_clash(c, &fat, 0);
  fold_rho(c);
  if (fat.hit) return fail(c, ORC_RUNTIME, "%s", fat.detail);
  return ORC_OK;
}
/* forces.cpp:381-388 */
int orc_compute_embedding(orc_ctx* c, double* e) {
  const double en = embed_slots(c, c->box.g, c->box.g + c->box.bz) + embed_clash(c);
  refresh_ghosts(c);
  if (e) *e = en;
  return ORC_OK;
}
/* forces.cpp:390-402 */
int orc_compute_pair(orc_ctx* c, double* e) {
  int rc;
  if ((rc = check_cutoffs(c))) return rc;
  fatal_t fat = {0};
  zero_force(c);
  double energy = pair_slots(c, &fat, c->box.g, c->box.g + c->box.bz);
  energy += visit_clash(c, &fat, 1);
  fold_force(c);
  if (fat.hit) return fail(c, ORC_RUNTIME, "%s", fat.detail);
  if (e) *e = energy;
  return ORC_OK;
}
/* forces.cpp:414-447 (W = 1 schedule: identical visit order, block-wise sums) */
int orc_eval_forces(orc_ctx* c, double* e_emb, double* e_pair) {
  int rc;
  if ((rc = check_cutoffs(c))) return rc;
  fatal_t fat = {0};
  zero_rho(c);
  for (int k = 0; k < 2; ++k) density_slots(c, &fat, c->blocks[k].z_lo, c->blocks[k].z_hi);
  visit_clash(c, &fat, 0);
  fold_rho(c);
  if (fat.hit) return fail(c, ORC_RUNTIME, "%s", fat.detail);
  double partial[2];
  for (int k = 0; k < 2; ++k) partial[k] = embed_slots(c, c->blocks[k].z_lo, c->blocks[k].z_hi);
  double emb = 0.0;
  for (int k = 0; k < 2; ++k) emb += partial[k];
  emb += embed_clash(c);
  refresh_ghosts(c);
  zero_force(c);
  for (int k = 0; k < 2; ++k) partial[k] = pair_slots(c, &fat, c->blocks[k].z_lo, c->blocks[k].z_hi);
  double pair = 0.0;
  for (int k = 0; k < 2; ++k) pair += partial[k];
  pair += visit_clash(c, &fat, 1);
  fold_force(c);
  if (fat.hit) return fail(c, ORC_RUNTIME, "%s", fat.detail);
  if (e_emb) *e_emb = emb;
  if (e_pair) *e_pair = pair;
  return ORC_OK;
}

/* --------------------------------------------------------- simulation */
/* mt19937_64 (the C++ standard's published parameters), sim.cpp:17-39 */
typedef struct { uint64_t mt[312]; int i; double spare; int have; } gauss_t;
static void mt_seed(gauss_t* g, uint64_t seed) {
  g->mt[0] = seed;
  for (int i = 1; i < 312; ++i)
    g->mt[i] = 6364136223846793005ULL * (g->mt[i - 1] ^ (g->mt[i - 1] >> 62)) + (uint64_t)i;
  g->i = 312;
  g->have = 0;
}
static uint64_t mt_next(gauss_t* g) {
  const uint64_t upper = ~0ULL << 31, lower = ~upper;
  if (g->i >= 312) {
    for (int k = 0; k < 312; ++k) {
      const uint64_t y = (g->mt[k] & upper) | (g->mt[(k + 1) % 312] & lower);
      g->mt[k] = g->mt[(k + 156) % 312] ^ (y >> 1) ^ ((y & 1ULL) ? 0xb5026f5aa96619e9ULL : 0ULL);
    }
    g->i = 0;
  }
  uint64_t y = g->mt[g->i++];
  y ^= (y >> 29) & 0x5555555555555555ULL;
  y ^= (y << 17) & 0x71d67fffeda60000ULL;
  y ^= (y << 37) & 0xfff7eee000000000ULL;
  y ^= y >> 43;
  return y;
}
static double uniform01(gauss_t* g) {
  return (double)((mt_next(g) >> 11) + 1) * (1.0 / 9007199254740993.0);
}
static double gauss_next(gauss_t* g) {
  if (g->have) { g->have = 0; return g->spare; }
  const double r = sqrt(-2.0 * log(uniform01(g)));
  const double a = 6.283185307179586476925286766559 * uniform01(g);
  g->spare = r * sin(a);
  g->have = 1;
  return r * cos(a);
}

/* sim.cpp:100-130 */
static int init_bcc(orc_ctx* c, double temperature, uint64_t seed) {
  const box_t* b = &c->box;
  const double mass = c->pot.mass;
  const double sigma =
      temperature > 0.0 ? sqrt(BOLTZMANN_EV * temperature * ACCEL_FACTOR / mass) : 0.0;
  gauss_t* g = malloc(sizeof(gauss_t));
  mt_seed(g, seed);
  uint64_t tag = 0;
  int rc = ORC_OK;
  FOR_INTERIOR(b, id) {
    rec_t r;
    memset(&r, 0, sizeof r);
    r.pos = site_position(id_to_coord(id, b), b);
    r.vel.x = sigma * gauss_next(g);
    r.vel.y = sigma * gauss_next(g);
    r.vel.z = sigma * gauss_next(g);
    r.tag = tag++;
    r.species = (uint16_t)c->pot.atomic_number;
    r.valid = 1;
    if ((rc = store_insert(c, &r))) { free(g); return rc; }
  }
  free(g);
  if (c->nbk) return fail(c, ORC_LOGIC, "perfect lattice produced a hash clash");
  const long n = (long)tag;
  v3 mean = {0, 0, 0};
  FOR_INTERIOR(b, id) {
    if (!c->slots[id].valid) continue;
    mean.x += c->slots[id].vel.x; mean.y += c->slots[id].vel.y; mean.z += c->slots[id].vel.z;
  }
  const double inv = 1.0 / (double)n;
  mean.x *= inv; mean.y *= inv; mean.z *= inv;
  FOR_INTERIOR(b, id) {
    if (!c->slots[id].valid) continue;
    c->slots[id].vel.x -= mean.x; c->slots[id].vel.y -= mean.y; c->slots[id].vel.z -= mean.z;
  }
  return ORC_OK;
}

/* sim.cpp:43-53: slots by id, then interior clash buckets in key order */
#define FOR_ATOM(c, R, BODY)                                                         \
  do {                                                                               \
    FOR_INTERIOR(&(c)->box, id__) {                                                  \
      rec_t* R = &(c)->slots[id__];                                                  \
      if (R->valid) { BODY; }                                                        \
    }                                                                                \
    for (int bi__ = 0; bi__ < (c)->nbk; ++bi__) {                                    \
      if (is_ghost_id((c)->bk[bi__].key, &(c)->box)) continue;                       \
      for (int j__ = 0; j__ < (c)->bk[bi__].n; ++j__) {                              \
        rec_t* R = &(c)->bk[bi__].r[j__];                                            \
        BODY;                                                                        \
      }                                                                              \
    }                                                                                \
  } while (0)

int orc_refresh_forces(orc_ctx* c) { /* sim.cpp:223-235 */
  double emb = 0, pair = 0;
  const int rc = orc_eval_forces(c, &emb, &pair);
  if (rc) {
    char tmp[1024];
    snprintf(tmp, sizeof tmp, "step %ld: %s", c->st.step, c->err);
    snprintf(c->err, sizeof c->err, "%s", tmp);
    return rc == ORC_INVALID ? ORC_RUNTIME : rc;
  }
  c->st.pair = pair;
  c->st.embedding = emb;
  c->st.r_underflow = c->pot.r_underflow;
  c->st.rho_clamp = c->pot.rho_clamp;
  return ORC_OK;
}

int orc_measure(orc_ctx* c) { /* sim.cpp:237-246 */
  double sum = 0.0, mx = 0.0;
  FOR_ATOM(c, a, {
    const double v2 = norm2(a->vel);
    sum += v2;
    if (v2 > mx) mx = v2;
  });
  c->st.kinetic = 0.5 * c->pot.mass * sum * MV2_TO_EV;
  c->st.max_speed = sqrt(mx);
  return ORC_OK;
}

double orc_pka_speed(double e, double m) { /* sim.cpp:88-92 */
  return sqrt(2.0 * e / m) * speed_factor;
}
double orc_adaptive_dt(double vmax, double dt_max, double max_disp) { /* sim.cpp:94-98 */
  double dt = dt_max;
  if (vmax > 0.0) { const double q = max_disp / vmax; if (q < dt) dt = q; }
  return dt > 1e-7 ? dt : 1e-7;
}

static int step_once(orc_ctx* c, double dt) { /* sim.cpp:248-273 */
  if (!(dt > 0.0)) return fail(c, ORC_INVALID, "dt must be positive");
  const double hk = 0.5 * dt * ACCEL_FACTOR / c->pot.mass;
  FOR_ATOM(c, a, {
    a->vel.x += a->force.x * hk; a->vel.y += a->force.y * hk; a->vel.z += a->force.z * hk;
    a->pos.x += a->vel.x * dt; a->pos.y += a->vel.y * dt; a->pos.z += a->vel.z * dt;
  });
  int rc;
  if ((rc = store_canonicalize(c))) return rc;
  if ((rc = store_update_hash(c))) return rc;
  if ((rc = store_fill_ghosts(c))) return rc;
  ++c->st.step;
  if ((rc = orc_refresh_forces(c))) return rc;
  double sum = 0.0, mx = 0.0;
  FOR_ATOM(c, a, {
    a->vel.x += a->force.x * hk; a->vel.y += a->force.y * hk; a->vel.z += a->force.z * hk;
    const double v2 = norm2(a->vel);
    sum += v2;
    if (v2 > mx) mx = v2;
  });
  c->st.kinetic = 0.5 * c->pot.mass * sum * MV2_TO_EV;
  c->st.max_speed = sqrt(mx);
  c->st.t += dt;
  c->st.dt = dt;
  return ORC_OK;
}

int orc_step(orc_ctx* c, double dt, long nsteps) {
  for (long i = 0; i < nsteps; ++i) {
    const double d = dt > 0.0 ? dt : orc_adaptive_dt(c->st.max_speed, c->cfg.dt_max, c->cfg.max_disp);
    const int rc = step_once(c, d);
    if (rc) return rc;
  }
  return ORC_OK;
}

int orc_inject_pka(orc_ctx* c) { /* sim.cpp:163-186 */
  const orc_config* f = &c->cfg;
  const box_t* b = &c->box;
  const long cx = f->pka_site[0] >= 0 ? f->pka_site[0] : b->bx / 2;
  const long cy = f->pka_site[1] >= 0 ? f->pka_site[1] : b->by / 2;
  const long cz = f->pka_site[2] >= 0 ? f->pka_site[2] : b->bz / 2;
  const lc_t q = {2 * (b->g + cx), b->g + cy, b->g + cz};
  const int64_t id = coord_to_id(q, b);
  rec_t* a = &c->slots[id];
  if (!a->valid) return fail(c, ORC_INVALID, "pka.site: no atom at cell (%ld,%ld,%ld)", cx, cy, cz);
  const v3 dir = {(double)f->pka_dir[0], (double)f->pka_dir[1], (double)f->pka_dir[2]};
  const double len = sqrt(norm2(dir));
  if (!(len > 0.0)) return fail(c, ORC_INVALID, "pka.direction: must not be the zero vector");
  const double v = orc_pka_speed(f->pka_energy_kev * 1000.0, c->pot.mass);
  const double s = v / len;
  a->vel.x = dir.x * s; a->vel.y = dir.y * s; a->vel.z = dir.z * s;
  return orc_measure(c);
}

int orc_count_defects(const orc_ctx* c, long out[3]) { /* analysis.cpp:40-56 */
  const box_t* b = &c->box;
  long vac = 0, inter = 0;
  FOR_INTERIOR(b, id) if (!c->slots[id].valid) ++vac;
  for (int i = 0; i < c->nbk; ++i) {
    const int64_t k = c->bk[i].key;
    if (is_ghost_id(k, b)) continue;
    const long extra = c->bk[i].n;
    if (extra == 0) continue;
    const long occ = (c->slots[k].valid ? 1 : 0) + extra;
    if (!c->slots[k].valid) --vac;
    inter += occ - 1;
  }
  out[0] = vac;
  out[1] = inter;
  out[2] = vac > inter ? vac : inter;
  return ORC_OK;
}

/* ------------------------------------------------------- construction */
const char* orc_create_error(void) { return g_create_err; }

orc_ctx* orc_create(const char* path, const orc_config* cfg, int init_lattice) {
  orc_ctx* c = calloc(1, sizeof(orc_ctx));
  c->cfg = *cfg;
  int rc = parse_potential(c, path);
  if (rc) goto bad;
  /* make_box, sim.cpp:62-78 (validate_config is the host config layer's job) */
  if (cfg->box_x <= 0 || cfg->box_y <= 0 || cfg->box_z <= 0) {
    fail(c, ORC_INVALID, "box: dimensions must be positive");
    goto bad;
  }
  {
    const double a0 = cfg->a0 > 0.0 ? cfg->a0 : c->pot.lattice_const;
    if (cfg->max_disp >= a0 / 2.0) {
      fail(c, ORC_INVALID, "max_disp: must stay below half the lattice constant");
      goto bad;
    }
    const double ic = c->pot.cutoff + 0.3 * a0;
    c->box.bx = cfg->box_x; c->box.by = cfg->box_y; c->box.bz = cfg->box_z;
    c->box.a0 = a0;
    c->box.g = cfg->ghost_width > 0 ? cfg->ghost_width : (long)ceil(ic / a0);
    c->index_cutoff = c->pot.cutoff + 0.3 * c->box.a0; /* sim.cpp:80-84 */
  }
  c->nslots = slot_count(&c->box);
  c->slots = calloc(c->nslots, sizeof(rec_t));
  c->ghost_ids = malloc(sizeof(int64_t) * c->nslots);
  for (int64_t id = 0; id < c->nslots; ++id)
    if (is_ghost_id(id, &c->box)) c->ghost_ids[c->nghost_ids++] = id;
  if ((rc = build_offsets(c, c->index_cutoff))) goto bad;
  build_partition(c);
  if (init_lattice) {
    if ((rc = init_bcc(c, cfg->temperature, cfg->seed))) goto bad;
    if ((rc = store_fill_ghosts(c))) goto bad;
    if ((rc = orc_refresh_forces(c))) goto bad;
    orc_measure(c);
  }
  return c;
bad:
  snprintf(g_create_err, sizeof g_create_err, "%s", c->err);
  orc_destroy(c);
  return NULL;
}

void orc_destroy(orc_ctx* c) {
  if (c) { free(c->ser_t); free(c->ser_d); }
  if (!c) return;
  free(c->pot.embed.seg); free(c->pot.zr.seg); free(c->pot.dens.seg);
  free(c->idx.ef); free(c->idx.of); free(c->idx.eh); free(c->idx.oh);
  free(c->slots);
  bk_clear_all(c);
  free(c->bk);
  free(c->links);
  free(c->ghost_ids);
  free(c);
}

const char* orc_error(const orc_ctx* c) { return c->err; }
void orc_box(const orc_ctx* c, long d[4], double* a0) {
  d[0] = c->box.bx; d[1] = c->box.by; d[2] = c->box.bz; d[3] = c->box.g;
  *a0 = c->box.a0;
}
double orc_index_cutoff(const orc_ctx* c) { return c->index_cutoff; }
double orc_potential_cutoff(const orc_ctx* c) { return c->pot.cutoff; }
double orc_mass(const orc_ctx* c) { return c->pot.mass; }

int orc_insert(orc_ctx* c, const double p[3], const double v[3], unsigned long long tag) {
  rec_t r;
  memset(&r, 0, sizeof r);
  r.pos.x = p[0]; r.pos.y = p[1]; r.pos.z = p[2];
  if (v) { r.vel.x = v[0]; r.vel.y = v[1]; r.vel.z = v[2]; }
  r.tag = tag;
  r.species = (uint16_t)c->pot.atomic_number;
  return store_insert(c, &r);
}
int orc_set_atom(orc_ctx* c, long long site, int idx, const double p[3], const double v[3]) {
  if (site < 0 || site >= c->nslots) return fail(c, ORC_INVALID, "site out of range");
  rec_t* r;
  if (idx < 0) r = &c->slots[site];
  else {
    bucket_t* b = bk_find(c, site);
    if (!b || idx >= b->n) return fail(c, ORC_INVALID, "no clash record (%lld, %d)", site, idx);
    r = &b->r[idx];
  }
  if (p) { r->pos.x = p[0]; r->pos.y = p[1]; r->pos.z = p[2]; }
  if (v) { r->vel.x = v[0]; r->vel.y = v[1]; r->vel.z = v[2]; }
  return ORC_OK;
}
long orc_displace_interior(orc_ctx* c, const double* disp, long n) {
  long i = 0;
  FOR_INTERIOR(&c->box, id) {
    rec_t* r = &c->slots[id];
    if (!r->valid || i >= n) continue;
    r->pos.x += disp[3 * i]; r->pos.y += disp[3 * i + 1]; r->pos.z += disp[3 * i + 2];
    ++i;
  }
  return i;
}
int orc_canonicalize(orc_ctx* c) { return store_canonicalize(c); }
int orc_update_hash(orc_ctx* c) { return store_update_hash(c); }
int orc_fill_ghosts(orc_ctx* c) { return store_fill_ghosts(c); }
int orc_rehash(orc_ctx* c) {
  int rc;
  if ((rc = store_canonicalize(c))) return rc;
  if ((rc = store_update_hash(c))) return rc;
  return store_fill_ghosts(c);
}
long orc_atom_count(const orc_ctx* c) { return store_atom_count(c); }
long long orc_nearest_site(orc_ctx* c, const double p[3]) {
  const v3 q = {p[0], p[1], p[2]};
  const int64_t id = nearest_site(q, &c->box);
  if (id < 0) domain_fail(c, q);
  return id;
}
void orc_guards(const orc_ctx* c, unsigned long long out[2]) {
  out[0] = c->pot.r_underflow;
  out[1] = c->pot.rho_clamp;
}
void orc_get_state(const orc_ctx* c, orc_state* st) { *st = c->st; }

long orc_slot_count(const orc_ctx* c) { return c->nslots; }
void orc_get_slots(const orc_ctx* c, double* pos, double* vel, double* force, double* rho,
                   double* df, unsigned long long* tag, unsigned char* valid,
                   unsigned char* ghost) {
  for (long i = 0; i < c->nslots; ++i) {
    const rec_t* r = &c->slots[i];
    if (pos) { pos[3 * i] = r->pos.x; pos[3 * i + 1] = r->pos.y; pos[3 * i + 2] = r->pos.z; }
    if (vel) { vel[3 * i] = r->vel.x; vel[3 * i + 1] = r->vel.y; vel[3 * i + 2] = r->vel.z; }
    if (force) { force[3 * i] = r->force.x; force[3 * i + 1] = r->force.y; force[3 * i + 2] = r->force.z; }
    if (rho) rho[i] = r->rho;
    if (df) df[i] = r->df;
    if (tag) tag[i] = r->tag;
    if (valid) valid[i] = r->valid;
    if (ghost) ghost[i] = r->ghost;
  }
}
long orc_clash_count(const orc_ctx* c) {
  long n = 0;
  for (int i = 0; i < c->nbk; ++i) n += c->bk[i].n;
  return n;
}
void orc_get_clash(const orc_ctx* c, long long* key, int* idx, double* pos, double* vel,
                   double* force, double* rho, double* df, unsigned long long* tag,
                   unsigned char* ghost) {
  long n = 0;
  for (int i = 0; i < c->nbk; ++i)
    for (int j = 0; j < c->bk[i].n; ++j, ++n) {
      const rec_t* r = &c->bk[i].r[j];
      if (key) key[n] = c->bk[i].key;
      if (idx) idx[n] = j;
      if (pos) { pos[3 * n] = r->pos.x; pos[3 * n + 1] = r->pos.y; pos[3 * n + 2] = r->pos.z; }
      if (vel) { vel[3 * n] = r->vel.x; vel[3 * n + 1] = r->vel.y; vel[3 * n + 2] = r->vel.z; }
      if (force) { force[3 * n] = r->force.x; force[3 * n + 1] = r->force.y; force[3 * n + 2] = r->force.z; }
      if (rho) rho[n] = r->rho;
      if (df) df[n] = r->df;
      if (tag) tag[n] = r->tag;
      if (ghost) ghost[n] = r->ghost;
    }
}

void orc_offsets(const orc_ctx* c, long counts[4], long long* ef, long long* of, long long* eh,
                 long long* oh, long* z_reach) {
  const offsets_t* ix = &c->idx;
  counts[0] = ix->nef; counts[1] = ix->nof; counts[2] = ix->neh; counts[3] = ix->noh;
  if (ef) for (long i = 0; i < ix->nef; ++i) ef[i] = ix->ef[i];
  if (of) for (long i = 0; i < ix->nof; ++i) of[i] = ix->of[i];
  if (eh) for (long i = 0; i < ix->neh; ++i) eh[i] = ix->eh[i];
  if (oh) for (long i = 0; i < ix->noh; ++i) oh[i] = ix->oh[i];
  if (z_reach) *z_reach = ix->z_reach;
}

int orc_potential_eval(orc_ctx* c, int which, double x, double out[2]) {
  seval_t e;
  if (which == 0) e = pot_density(&c->pot, x);
  else if (which == 1) {
    if (x <= 0.0) return fail(c, ORC_DOMAIN, "EamPotential::pair: r <= 0");
    e = pot_pair(&c->pot, x);
  } else e = pot_embedding(&c->pot, x);
  out[0] = e.value;
  out[1] = e.deriv;
  return ORC_OK;
}

long orc_spline(const orc_ctx* c, int which, double* x0, double* h, double* seg) {
  const spline_t* s = which == 0 ? &c->pot.embed : (which == 1 ? &c->pot.zr : &c->pot.dens);
  if (x0) *x0 = s->x0;
  if (h) *h = s->h;
  if (seg) memcpy(seg, s->seg, sizeof(double) * 7 * s->nseg);
  return s->nseg;
}

/* ------------------------------------------- synthetic table (tests) */
/* synthetic.h:17-32 constants, synthetic.cpp:10-98 closed forms + writer */
#define SYN_MASS 55.845
#define SYN_A0 2.8553
#define SYN_CUT 5.6
#define SYN_RNN 2.4727640449591856
#define SYN_RHO_RC 4.1
#define SYN_RHO_AMP 0.02171868164588797
#define SYN_PAIR_SLOPE 6.5
#define SYN_PAIR_AMP 0.5123847826890735
#define SYN_EMBED_AMP 9.053882773088201
#define SYN_EMBED_REG 0.09
#define SYN_RHO_TABLE_MAX 4.0
static double syn_density(double r) {
  if (r >= SYN_RHO_RC) return 0.0;
  const double t = SYN_RHO_RC - r;
  return SYN_RHO_AMP * t * t * t;
}
static double syn_phi(double r) {
  if (r >= SYN_CUT) return 0.0;
  const double damp = (SYN_CUT - r) / (SYN_CUT - SYN_RNN);
  return SYN_PAIR_AMP * exp(-SYN_PAIR_SLOPE * (r / SYN_RNN - 1.0)) * damp * damp * damp;
}
static double syn_embedding(double rho) {
  return -SYN_EMBED_AMP * (sqrt(rho + SYN_EMBED_REG) - sqrt(SYN_EMBED_REG));
}
static void write_block(FILE* f, const double* v, long n) {
  for (long i = 0; i < n; ++i) fprintf(f, "%.17g%c", v[i], (i % 4 == 3) ? '\n' : ' ');
  if (n % 4 != 0) fputc('\n', f);
}
int orc_write_synthetic_table(const char* path, long nrho, long nr) {
  if (nrho < 4 || nr < 4) return ORC_INVALID;
  FILE* f = fopen(path, "w");
  if (!f) return ORC_RUNTIME;
  fprintf(f,
          "synthetic Fe-like EAM: rho=%.17g*(%.17g-r)^3; "
          "phi=%.17g*exp(-%.17g*(r/%.17g-1))*((%.17g-r)/(%.17g-%.17g))^3; "
          "F=-%.17g*(sqrt(rho+%.17g)-sqrt(%.17g))\n",
          SYN_RHO_AMP, SYN_RHO_RC, SYN_PAIR_AMP, SYN_PAIR_SLOPE, SYN_RNN, SYN_CUT, SYN_CUT,
          SYN_RNN, SYN_EMBED_AMP, SYN_EMBED_REG, SYN_EMBED_REG);
  fprintf(f, "%d %.17g %.17g bcc\n", 26, SYN_MASS, SYN_A0);
  const double drho = SYN_RHO_TABLE_MAX / (double)(nrho - 1);
  const double dr = SYN_CUT / (double)nr;
  fprintf(f, "%ld %.17g %ld %.17g %.17g\n", nrho, drho, nr, dr, SYN_CUT);
  long n = nrho > nr ? nrho : nr;
  double* v = malloc(sizeof(double) * n);
  for (long k = 0; k < nrho; ++k) v[k] = syn_embedding(drho * (double)k);
  write_block(f, v, nrho);
  for (long k = 0; k < nr; ++k) { const double r = dr * (double)(k + 1); v[k] = r * syn_phi(r); }
  write_block(f, v, nr);
  for (long k = 0; k < nr; ++k) v[k] = syn_density(dr * (double)(k + 1));
  write_block(f, v, nr);
  free(v);
  return fclose(f) == 0 ? ORC_OK : ORC_RUNTIME;
}


/* ------------------------------------------------------------- run loop */
static int in_band(const orc_ctx* c, int64_t id, long band) { /* sim.cpp:190-197 */
  if (band <= 0) return 1;
  const box_t* b = &c->box;
  const int64_t tx2 = 2 * total_x(b), ty = total_y(b);
  const long cz = (long)(id / (tx2 * ty)), cy = (long)((id / tx2) % ty), x = (long)(id % tx2);
  const long cx = x >> 1, g = b->g;
  return cx - g < band || (g + b->bx - 1) - cx < band || cy - g < band ||
         (g + b->by - 1) - cy < band || cz - g < band || (g + b->bz - 1) - cz < band;
}

int orc_thermostat_rescale(orc_ctx* c) { /* sim.cpp:188-221 */
  const long band = c->cfg.thermostat_boundary_cells;
  const box_t* b = &c->box;
  double sum_v2 = 0.0;
  long n = 0;
  FOR_INTERIOR(b, id) {
    const rec_t* a = &c->slots[id];
    if (!a->valid || !in_band(c, id, band)) continue;
    sum_v2 += norm2(a->vel);
    ++n;
  }
  for (int i = 0; i < c->nbk; ++i) {
    if (is_ghost_id(c->bk[i].key, b) || !in_band(c, c->bk[i].key, band)) continue;
    for (int j = 0; j < c->bk[i].n; ++j) {
      sum_v2 += norm2(c->bk[i].r[j].vel);
      ++n;
    }
  }
  const double measured =
      n > 0 ? c->pot.mass * sum_v2 * MV2_TO_EV / (3.0 * (double)n * BOLTZMANN_EV) : 0.0;
  if (!(measured > 0.0)) {
    fprintf(stderr, "thermostat: measured temperature is zero, skipping\n");
    return ORC_OK;
  }
  const double f = sqrt(c->cfg.temperature / measured);
  FOR_INTERIOR(b, id) {
    rec_t* a = &c->slots[id];
    if (!a->valid || !in_band(c, id, band)) continue;
    a->vel.x *= f; a->vel.y *= f; a->vel.z *= f;
  }
  for (int i = 0; i < c->nbk; ++i) {
    if (is_ghost_id(c->bk[i].key, b) || !in_band(c, c->bk[i].key, band)) continue;
    for (int j = 0; j < c->bk[i].n; ++j) {
      rec_t* a = &c->bk[i].r[j];
      a->vel.x *= f; a->vel.y *= f; a->vel.z *= f;
    }
  }
  return orc_measure(c);
}

static const char* const k_symbols[] = { /* analysis.cpp:11-19 */
    "X",  "H",  "He", "Li", "Be", "B",  "C",  "N",  "O",  "F",  "Ne", "Na", "Mg", "Al", "Si",
    "P",  "S",  "Cl", "Ar", "K",  "Ca", "Sc", "Ti", "V",  "Cr", "Mn", "Fe", "Co", "Ni", "Cu",
    "Zn", "Ga", "Ge", "As", "Se", "Br", "Kr", "Rb", "Sr", "Y",  "Zr", "Nb", "Mo", "Tc", "Ru",
    "Rh", "Pd", "Ag", "Cd", "In", "Sn", "Sb", "Te", "I",  "Xe", "Cs", "Ba", "La", "Ce", "Pr",
    "Nd", "Pm", "Sm", "Eu", "Gd", "Tb", "Dy", "Ho", "Er", "Tm", "Yb", "Lu", "Hf", "Ta", "W",
    "Re", "Os", "Ir", "Pt", "Au", "Hg", "Tl", "Pb", "Bi", "Po", "At", "Rn", "Fr", "Ra", "Ac",
    "Th", "Pa", "U"};

static const char* symbol_for(unsigned z) {
  return z < sizeof(k_symbols) / sizeof(k_symbols[0]) ? k_symbols[z] : "X";
}

static void csv_time(double t, char out[48]) { /* analysis.cpp:66-75 */
  snprintf(out, 48, "%.9g", t);
  if (!strpbrk(out, ".eE") && strspn(out, "-0123456789") == strlen(out)) strcat(out, ".0");
}

int orc_write_snapshot(const orc_ctx* c, const char* path) { /* analysis.cpp:90-116 */
  const box_t* b = &c->box;
  const double shift = b->g * b->a0;
  FILE* f = fopen(path, "w");
  if (!f) return fail((orc_ctx*)c, ORC_RUNTIME, "cannot open %s for writing", path);
  char tb[48];
  csv_time(c->st.t, tb);
  fprintf(f, "%ld\n", store_atom_count(c));
  fprintf(f,
          "Lattice=\"%.10g 0 0 0 %.10g 0 0 0 %.10g\" "
          "Properties=species:S:1:pos:R:3:tag:I:1 Time=%s\n",
          b->bx * b->a0, b->by * b->a0, b->bz * b->a0, tb);
#define EMIT(a)                                                                         \
  fprintf(f, "%s %.10g %.10g %.10g %llu\n", symbol_for((a)->species), (a)->pos.x - shift, \
          (a)->pos.y - shift, (a)->pos.z - shift, (unsigned long long)(a)->tag)
  FOR_INTERIOR(b, id) {
    if (c->slots[id].valid) EMIT(&c->slots[id]);
  }
  for (int i = 0; i < c->nbk; ++i) {
    if (is_ghost_id(c->bk[i].key, b)) continue;
    for (int j = 0; j < c->bk[i].n; ++j) EMIT(&c->bk[i].r[j]);
  }
#undef EMIT
  const int bad = ferror(f);
  fclose(f);
  return bad ? fail((orc_ctx*)c, ORC_RUNTIME, "write failed: %s", path) : ORC_OK;
}

int orc_write_timeseries(const char* path, long n, const double* t, const long* d) {
  FILE* f = fopen(path, "w"); /* analysis.cpp:77-88 */
  if (!f) return ORC_RUNTIME;
  fputs("t_ps,vacancies,interstitials,frenkel_pairs\n", f);
  char tb[48];
  for (long i = 0; i < n; ++i) {
    csv_time(t[i], tb);
    fprintf(f, "%s,%ld,%ld,%ld\n", tb, d[3 * i], d[3 * i + 1], d[3 * i + 2]);
  }
  const int bad = ferror(f);
  fclose(f);
  return bad ? ORC_RUNTIME : ORC_OK;
}

static void sample_defects(orc_ctx* c) { /* sim.cpp:275-277 */
  if (c->nser == c->capser) {
    c->capser = c->capser ? 2 * c->capser : 64;
    c->ser_t = (double*)realloc(c->ser_t, c->capser * sizeof(double));
    c->ser_d = (long*)realloc(c->ser_d, 3 * c->capser * sizeof(long));
  }
  c->ser_t[c->nser] = c->st.t;
  orc_count_defects(c, c->ser_d + 3 * c->nser);
  ++c->nser;
}

long orc_series(const orc_ctx* c, double* t, long* d) {
  if (t) memcpy(t, c->ser_t, c->nser * sizeof(double));
  if (d) memcpy(d, c->ser_d, 3 * c->nser * sizeof(long));
  return c->nser;
}

static int nonempty(const char* s) { return s && s[0]; }

static int snapshot_file(orc_ctx* c, const orc_run_spec* r, const char* suffix) {
  if (!nonempty(r->snapshot_prefix)) return ORC_OK; /* sim.cpp:279-282 */
  char path[1024];
  snprintf(path, sizeof path, "%s%s", r->snapshot_prefix, suffix);
  return orc_write_snapshot(c, path);
}

int orc_run(orc_ctx* c, const orc_run_spec* r, const char* log_path) { /* sim.cpp:289-360 */
  c->cfg.thermostat_boundary_cells = r->thermostat_boundary_cells;
  FILE* log = NULL;
  if (nonempty(log_path)) log = strcmp(log_path, "-") == 0 ? stdout : fopen(log_path, "w");
  c->nser = 0;
  sample_defects(c);
  int rc = ORC_OK;
  if (r->snapshot_interval > 0 && (rc = snapshot_file(c, r, "_000000.xyz"))) goto out;
#define LOG_LINE()                                                                       \
  do {                                                                                   \
    if (log) {                                                                           \
      char tb_[48];                                                                      \
      csv_time(c->st.t, tb_);                                                            \
      const long n_ = store_atom_count(c);                                               \
      const double T_ = n_ == 0 ? 0.0 : 2.0 * c->st.kinetic / (3.0 * (double)n_ * BOLTZMANN_EV); \
      fprintf(log, "step %ld  t=%s ps  dt=%.4g  E=%.6f eV  T=%.1f K  FP=%ld\n", c->st.step, \
              tb_, c->st.dt, c->st.kinetic + c->st.pair + c->st.embedding, T_,             \
              c->ser_d[3 * (c->nser - 1) + 2]);                                         \
    }                                                                                    \
  } while (0)
#define GUARDED_STEP()                                                                   \
  do {                                                                                   \
    rc = orc_step(c, -1.0, 1);                                                           \
    if (rc) {                                                                            \
      if (nonempty(r->snapshot_prefix)) {                                                \
        char pm_[1024];                                                                  \
        snprintf(pm_, sizeof pm_, "%s_postmortem.xyz", r->snapshot_prefix);              \
        orc_write_snapshot(c, pm_);                                                      \
      }                                                                                  \
      if (nonempty(r->timeseries)) orc_write_timeseries(r->timeseries, c->nser, c->ser_t, c->ser_d); \
      goto out;                                                                          \
    }                                                                                    \
  } while (0)
  for (long i = 0; i < r->equilibration_steps; ++i) {
    GUARDED_STEP();
    if (r->thermostat_enabled && (i + 1) % r->thermostat_interval == 0)
      orc_thermostat_rescale(c);
  }
  if (c->cfg.pka_energy_kev > 0.0 && (rc = orc_inject_pka(c))) goto out;
  {
    long done = 0;
    int sampled_last = 1;
    for (;;) {
      const int step_cap = r->steps > 0 && done >= r->steps;
      const int time_cap = r->max_time > 0.0 && c->st.t >= r->max_time;
      const int no_budget = r->steps == 0 && r->max_time == 0.0;
      if (step_cap || time_cap || no_budget) break;
      GUARDED_STEP();
      ++done;
      if (r->thermostat_enabled && done % r->thermostat_interval == 0)
        orc_thermostat_rescale(c);
      sampled_last = 0;
      if (r->defect_interval > 0 && done % r->defect_interval == 0) {
        sample_defects(c);
        sampled_last = 1;
        LOG_LINE();
      }
      if (r->snapshot_interval > 0 && done % r->snapshot_interval == 0) {
        char suffix[32];
        snprintf(suffix, sizeof suffix, "_%06ld.xyz", done);
        if ((rc = snapshot_file(c, r, suffix))) goto out;
      }
    }
    if (!sampled_last) {
      sample_defects(c);
      LOG_LINE();
    }
  }
  if (nonempty(r->timeseries) &&
      orc_write_timeseries(r->timeseries, c->nser, c->ser_t, c->ser_d))
    rc = fail(c, ORC_RUNTIME, "write failed: %s", r->timeseries);
  if (!rc) rc = snapshot_file(c, r, "_final.xyz");
#undef LOG_LINE
#undef GUARDED_STEP
out:
  if (log && log != stdout) fclose(log);
  if (log == stdout) fflush(stdout);
  return rc;
}
