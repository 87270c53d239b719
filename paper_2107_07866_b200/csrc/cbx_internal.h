// cbx_internal.h -- shared definitions of the B200 EAM library (host + device).
//
// Site indexing.  The reference numbers lattice sites over the ghost-inclusive
// box as id = (z*ty + y)*2tx + x with a doubled x axis (even x = corner
// sublattice, odd x = body centre; core/src/lattice.cpp:10-15).  Writing
// x = 2*cx + par gives id = 2*cell + par with cell = (z*ty + y)*tx + cx.
// On the device every per-site array is split by sublattice:
//     dev = par*NC + cell          (NC = tx*ty*tz cells)
// so a warp of 32 consecutive cells of one parity reads 32 consecutive
// records (one 1 KB run for a double4 array) and shares one offset list.
#pragma once

#include <cstdint>
#include <cmath>
#include <cstdlib>

#if defined(__CUDACC__)
#define CBX_HD __host__ __device__ __forceinline__
#else
#define CBX_HD inline
#endif

namespace cbx {

// A/B switches of the experiment build (nvcc -DCBX_AB): read from the
// environment there (each restores an earlier design for a same-box
// comparison); the release library compiles every one to its default, so no
// environment variable can change its physics, layout or timing.
inline int ab_flag(const char* name, int dflt) {
#ifdef CBX_AB
  const char* e = std::getenv(name);
  return e ? std::atoi(e) : dflt;
#else
  (void)name;
  return dflt;
#endif
}

// Invalid (vacant) slots carry this x/y/z so that any distance to them
// exceeds every cutoff: no separate validity load in the stencil loops.
constexpr double kVacant = 1.0e30;
constexpr double kVacantTest = 1.0e29;
constexpr float kVacantF = 1.0e18f;  // fp32 shadow of a vacant site
constexpr double kOverlapR2 = 1e-12;  // forces.cpp:14
constexpr int kMaxOffsets = 1024;     // per list, constant memory
constexpr int kMaxOverlapRecords = 64;

// --- exact IEEE arithmetic, no FMA contraction (the reference builds with
// contraction off; lattice hashing and r^2 must be bit-identical) ----------
#if defined(__CUDA_ARCH__)
CBX_HD double xadd(double a, double b) { return __dadd_rn(a, b); }
CBX_HD double xsub(double a, double b) { return __dsub_rn(a, b); }
CBX_HD double xmul(double a, double b) { return __dmul_rn(a, b); }
CBX_HD double xdiv(double a, double b) { return __ddiv_rn(a, b); }
#else
CBX_HD double xadd(double a, double b) { return a + b; }
CBX_HD double xsub(double a, double b) { return a - b; }
CBX_HD double xmul(double a, double b) { return a * b; }
CBX_HD double xdiv(double a, double b) { return a / b; }
#endif

struct Geo {
  int bx, by, bz, g;  // interior cells per axis, ghost width (cells)
  int tx, ty, tz;     // ghost-inclusive cells per axis
  int txy;            // tx*ty
  long long NC;       // tx*ty*tz
  long long NI;       // bx*by*bz interior cells
  double a0;
  double lx, ly, lz;  // periodic lengths, BoxSpec::len_x = box_x * a0 (lattice.h:35-37)
  int kmx, kmy, kmz;  // fill_ghosts k_max per axis (store.cpp:139-141)
  // z-slab decomposition (multi-GPU).  Positions and hashes stay in the
  // global frame; this store covers global ghost-inclusive z cells
  // [zoff, zoff + tz).  One rank: zoff = 0, gbz = bz.
  int zoff;    // global ghost-inclusive z cell of local z cell 0
  int gbz;     // global interior z cells
  int gtz;     // global ghost-inclusive z cells (gbz + 2g)
  double glz;  // global periodic z length (gbz * a0)
  int slab;    // 1 when z ghosts come from neighbour ranks
  // n / bx and n / by for n < 2^31 as (n * m) >> sh (Granlund-Montgomery:
  // sh = 31 + ceil(log2 d), m = ceil(2^sh / d)); device site mapping
  unsigned long long mbx, mby;
  int sbx, sby;
  // stencil-pass work units walk columns of strips along y when rows hold
  // whole strips (unit_strip, stencil_fast.cuh); 0 keeps the row order
  int col_units;
};

// exact floor(n / d) for 0 <= n < 2^31 from the constants of make_magic
CBX_HD unsigned magic_div(unsigned n, unsigned long long m, int sh) {
  return (unsigned)(((unsigned long long)n * m) >> sh);
}

CBX_HD long long ref_id(long long cell, int par) { return 2 * cell + par; }
CBX_HD long long dev_of_ref(long long id, long long NC) { return (id & 1) * NC + (id >> 1); }
CBX_HD long long ref_of_dev(long long d, long long NC) {
  const int par = d >= NC;
  return 2 * (d - par * NC) + par;
}

// cell coordinates (ghost-inclusive, cell units) of a cell index
CBX_HD void cell_xyz(long long cell, const Geo& G, int& cx, int& cy, int& cz) {
  if (cell < (1ll << 31)) {  // 32-bit division (every box that fits one GPU)
    const unsigned c = (unsigned)cell, r = c / (unsigned)G.tx;
    cx = (int)(c - r * (unsigned)G.tx);
    cy = (int)(r % (unsigned)G.ty);
    cz = (int)(r / (unsigned)G.ty);
    return;
  }
  cx = (int)(cell % G.tx);
  const long long r = cell / G.tx;
  cy = (int)(r % G.ty);
  cz = (int)(r / G.ty);
}
CBX_HD long long cell_of(int cx, int cy, int cz, const Geo& G) {
  return ((long long)cz * G.ty + cy) * G.tx + cx;
}
CBX_HD bool cell_is_ghost(int cx, int cy, int cz, const Geo& G) {
  return cx < G.g || cx >= G.g + G.bx || cy < G.g || cy >= G.g + G.by || cz < G.g ||
         cz >= G.g + G.bz;
}
// interior enumeration e in [0, NI) -> cell, x fastest (matches for_each_interior_id order)
CBX_HD long long interior_cell(long long e, const Geo& G) {
  if (e < (1ll << 31)) {
    const unsigned u = (unsigned)e, r = u / (unsigned)G.bx;
    const int cx = (int)(u - r * (unsigned)G.bx);
    const int cy = (int)(r % (unsigned)G.by);
    const int cz = (int)(r / (unsigned)G.by);
    return cell_of(cx + G.g, cy + G.g, cz + G.g, G);
  }
  const int cx = (int)(e % G.bx);
  const long long r = e / G.bx;
  const int cy = (int)(r % G.by);
  const int cz = (int)(r / G.by);
  return cell_of(cx + G.g, cy + G.g, cz + G.g, G);
}

// lattice.cpp:58-62 round half toward -inf
CBX_HD long rhd(double t) { return (long)ceil(xsub(t, 0.5)); }
CBX_HD double xsq(double v) { return xmul(v, v); }
CBX_HD long clampl(long v, long lo, long hi) { return v < lo ? lo : (v > hi ? hi : v); }

// lattice.cpp:66-89: nearest site coordinate in doubled-x lattice units,
// unclamped (used by the periodic wrap)
CBX_HD void nearest_site_coord(double px, double py, double pz, double a0, long& ox, long& oy,
                               long& oz) {
  const double fx = xdiv(px, a0), fy = xdiv(py, a0), fz = xdiv(pz, a0);
  const long ci = rhd(fx), cj = rhd(fy), ck = rhd(fz);
  const double dc = xadd(xadd(xsq(xsub(fx, (double)ci)), xsq(xsub(fy, (double)cj))),
                         xsq(xsub(fz, (double)ck)));
  const long bi = rhd(xsub(fx, 0.5)), bj = rhd(xsub(fy, 0.5)), bk = rhd(xsub(fz, 0.5));
  const double db = xadd(xadd(xsq(xsub(xsub(fx, (double)bi), 0.5)),
                              xsq(xsub(xsub(fy, (double)bj), 0.5))),
                         xsq(xsub(xsub(fz, (double)bk), 0.5)));
  const long c_x = 2 * ci, c_y = cj, c_z = ck;
  const long b_x = 2 * bi + 1, b_y = bj, b_z = bk;
  bool corner;
  if (dc < db) corner = true;
  else if (db < dc) corner = false;
  else if (c_z != b_z) corner = c_z < b_z;
  else if (c_y != b_y) corner = c_y < b_y;
  else corner = c_x < b_x;
  ox = corner ? c_x : b_x;
  oy = corner ? c_y : b_y;
  oz = corner ? c_z : b_z;
}

// lattice.cpp:99-131: hash of a position to the reference site id, clamped to
// the box; returns -1 when the position lies outside the ghost-inclusive volume
CBX_HD long long nearest_site(double px, double py, double pz, const Geo& G) {
  const double a = G.a0;
  if (px < 0.0 || px >= xmul((double)G.tx, a) || py < 0.0 || py >= xmul((double)G.ty, a) ||
      pz < 0.0 || pz >= xmul((double)G.gtz, a))
    return -1;
  const double fx = xdiv(px, a), fy = xdiv(py, a), fz = xdiv(pz, a);
  const long ci = clampl(rhd(fx), 0, G.tx - 1);
  const long cj = clampl(rhd(fy), 0, G.ty - 1);
  const long ck = clampl(rhd(fz), 0, G.gtz - 1) - G.zoff;
  const double dc = xadd(xadd(xsq(xsub(fx, (double)ci)), xsq(xsub(fy, (double)cj))),
                         xsq(xsub(fz, (double)(ck + G.zoff))));
  const long bi = clampl(rhd(xsub(fx, 0.5)), 0, G.tx - 1);
  const long bj = clampl(rhd(xsub(fy, 0.5)), 0, G.ty - 1);
  const long bk = clampl(rhd(xsub(fz, 0.5)), 0, G.gtz - 1) - G.zoff;
  const double db = xadd(xadd(xsq(xsub(xsub(fx, (double)bi), 0.5)),
                              xsq(xsub(xsub(fy, (double)bj), 0.5))),
                         xsq(xsub(xsub(fz, (double)(bk + G.zoff)), 0.5)));
  const long long idc = ref_id(cell_of((int)ci, (int)cj, (int)ck, G), 0);
  const long long idb = ref_id(cell_of((int)bi, (int)bj, (int)bk, G), 1);
  if (dc < db) return idc;
  if (db < dc) return idb;
  return idc < idb ? idc : idb;
}

CBX_HD long floor_div(long a, long b) {  // store.cpp:80-84
  long q = a / b;
  if ((a % b != 0) && ((a < 0) != (b < 0))) --q;
  return q;
}

// store.cpp:91-105: periodic wrap of one atom; false if it does not converge
CBX_HD bool wrap_position(double& px, double& py, double& pz, const Geo& G) {
  for (int pass = 0; pass < 4; ++pass) {
    long qx, qy, qz;
    nearest_site_coord(px, py, pz, G.a0, qx, qy, qz);
    const long kx = floor_div(qx - 2 * G.g, 2 * G.bx);
    const long ky = floor_div(qy - G.g, G.by);
    const long kz = floor_div(qz - G.g, G.gbz);
    if (kx == 0 && ky == 0 && kz == 0) return true;
    px = xsub(px, xmul((double)kx, G.lx));
    py = xsub(py, xmul((double)ky, G.ly));
    pz = xsub(pz, xmul((double)kz, G.glz));
  }
  return false;
}

// local z cell of a (local) reference site id; floor semantics for ids
// outside the store (atoms hashed into another rank's slab)
CBX_HD long site_cz(long long id, const Geo& G) {
  const long long cell = id >= 0 ? (id >> 1) : -((-id + 1) >> 1);
  const long long plane = (long long)G.tx * G.ty;
  long long q = cell / plane;
  if (cell % plane != 0 && cell < 0) --q;
  return (long)q;
}
// 0: owned here; 1: owned by the rank above (z+); -1: by the rank below
CBX_HD int owner_dir(long long id, const Geo& G) {
  if (!G.slab) return 0;
  const long cz = site_cz(id, G);
  if (cz >= G.g && cz < G.g + G.bz) return 0;
  // global interior z index of the site, and of this slab's first plane
  const long gz = cz + G.zoff - G.g, lo = G.zoff, hi = G.zoff + G.bz;
  // the neighbour that is nearer in the periodic sense
  const long up = ((gz - hi) % G.gbz + G.gbz) % G.gbz, dn = ((lo - 1 - gz) % G.gbz + G.gbz) % G.gbz;
  return up <= dn ? 1 : -1;
}

// exact squared distance in the reference's operation order (vec3.h:14)
CBX_HD double exact_r2(double dx, double dy, double dz) {
  return xadd(xadd(xmul(dx, dx), xmul(dy, dy)), xmul(dz, dz));
}

}  // namespace cbx
