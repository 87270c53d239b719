// store_kernels.cu -- the per-step lattice-store machinery on the device.
//
// Reference (paths relative to /root/reference/proj/core/src):
//   Simulation::step kick + drift       sim.cpp:250-255  -> k_kick_drift (+clash)
//   canonicalize_positions              store.cpp:88-118 -> fused into k_kick_drift
//   update_hash pass 1 (evict)          store.cpp:46-54  -> fused into k_kick_drift
//   update_hash pass 2 (re-place)       store.cpp:56-75  -> k_rehash (one block)
//   fill_ghosts, slot images            store.cpp:120-158,184-188 -> k_ghost_fill
//   fill_ghosts, clash images           store.cpp:160-194 -> k_clash_images (one block)
//   second half-kick + measure          sim.cpp:262-270, 237-246 -> k_kick2 (+clash)
//   count_defects                       analysis.cpp:40-56 -> k_count_defects
//
// Positions, hashes and wraps use exact IEEE operations in the reference's
// order (cbx_internal.h), so slot ids, clash membership and bucket order are
// bit-identical to the reference.  Pass 2's sequential semantics (the first
// re-placed record claims a free slot) are reproduced by sorting all movers
// by (new site, old site, class, order) -- see k_rehash.
#include <algorithm>
#include <climits>
#include <cstdlib>

#include "cbx_device.cuh"
#include "p2p.cuh"
#include "finalize.cuh"

namespace cbx {

__device__ __forceinline__ int eam_blocks_dev(const KP& P) { return (int)((P.G.NI + 127) / 128); }

__device__ __forceinline__ double half_kick(const KP& P, double dt) {
  return xdiv(xmul(xmul(0.5, dt), P.accel), P.mass);  // sim.cpp:250
}

__device__ __forceinline__ bool site_is_ghost(long long id, const Geo& G) {
  int cx, cy, cz;
  cell_xyz(id >> 1, G, cx, cy, cz);
  return cell_is_ghost(cx, cy, cz, G);
}

// -------------------------------------------------- kick, drift, wrap, evict
__device__ void clash_kick_drift_body(const KP& P, int move, int blk, int nblk);

// zero_acc: also clear the site's rho / force accumulators once the half
// kick has read the force (the density and force passes of this step add
// into them; replaces two full-array memsets)
// images: also write the site's ghost images (the step path's k_ghost_fill)
__device__ void ghost_images(const KP& P, long long d, const double4& p);
__device__ void ghost_images_at(const KP& P, int par, int cx, int cy, int cz, const double4& p);
__device__ void clash_kick2_sums(const KP& P, int blk);
// a site's record as the sweep loads it (every load issued before the
// first use: one memory round trip per site)
struct KdSite {
  long long d;
  int par, cx, cy, cz;
  bool live;
  double4 p;
  double vx, vy, vz, fx, fy, fz;
};
__device__ __forceinline__ void kick_drift_load(const KP& P, int vb, KdSite& a) {
  a.live = map_site_xyz(P, vb, a.par, a.d, a.cx, a.cy, a.cz);
  if (!a.live) return;
  // 32-bit site index into per-component base pointers (a single store fits
  // 2^31 sites)
  const long long S = P.S;
  const int i = (int)a.d;
  a.p = P.pdf[i];
  a.vx = P.vel[i];
  a.vy = P.vel[S + i];
  a.vz = P.vel[2 * S + i];
  a.fx = P.frc[i];
  a.fy = P.frc[S + i];
  a.fz = P.frc[2 * S + i];
}
__device__ __forceinline__ void kick_drift_proc(const KP& P, int move, int zero_acc, int images,
                                                double dt, double hk, bool k2, double& v2s,
                                                double& v2m, const KdSite& a, double& ub2);
// one site per thread of virtual block vb (128 cells x 2 sublattices)
__device__ __forceinline__ void kick_drift_site(const KP& P, int move, int zero_acc, int images,
                                                int vb, double dt, double hk, bool k2,
                                                double& v2s, double& v2m, double& ub2) {
  KdSite a;
  kick_drift_load(P, vb, a);
  if (a.live) kick_drift_proc(P, move, zero_acc, images, dt, hk, k2, v2s, v2m, a, ub2);
}
// ub2: |u|^2 of the site's atom relative to its own lattice site (fast hash),
// kUbDirty when it took the wrap / nearest_site path, unchanged when vacant
__device__ __forceinline__ void kick_drift_proc(const KP& P, int move, int zero_acc, int images,
                                                double dt, double hk, bool k2, double& v2s,
                                                double& v2m, const KdSite& a, double& ub2) {
  const long long S = P.S;
  const long long d = a.d;
  const int i = (int)d;
  const int par = a.par, cx = a.cx, cy = a.cy, cz = a.cz;
  double* __restrict__ vxp = P.vel;
  double* __restrict__ vyp = P.vel + S;
  double* __restrict__ vzp = P.vel + 2 * S;
  double* __restrict__ fxp = P.frc;
  double* __restrict__ fyp = P.frc + S;
  double* __restrict__ fzp = P.frc + 2 * S;
  double4 p = a.p;
  double vx = a.vx, vy = a.vy, vz = a.vz;
  const double fx = a.fx, fy = a.fy, fz = a.fz;
  if (zero_acc) {
    P.rho[i] = 0.0;
    fxp[i] = 0.0;
    fyp[i] = 0.0;
    fzp[i] = 0.0;
  }
  if (p.x >= kVacantTest) {
    if (images) ghost_images_at(P, par, cx, cy, cz, p);
    return;
  }
  if (k2) {  // k_kick2 of the previous step (sim.cpp:262-270), same arithmetic
    vx = xadd(vx, xmul(fx, hk));
    vy = xadd(vy, xmul(fy, hk));
    vz = xadd(vz, xmul(fz, hk));
    const double v2 = exact_r2(vx, vy, vz);
    v2s += v2;
    v2m = fmax(v2m, v2);
  }
  if (move) {
    vx = xadd(vx, xmul(fx, hk));
    vy = xadd(vy, xmul(fy, hk));
    vz = xadd(vz, xmul(fz, hk));
    p.x = xadd(p.x, xmul(vx, dt));
    p.y = xadd(p.y, xmul(vy, dt));
    p.z = xadd(p.z, xmul(vz, dt));
    vxp[i] = vx;
    vyp[i] = vy;
    vzp[i] = vz;
  }
  const long long own = ref_of_dev(d, P.G.NC);
  // fast hash (canonicalize_positions + nearest_site, store.cpp:88-118 and
  // lattice.cpp:99-131, collapse to the identity for an atom inside the
  // Wigner-Seitz ball of its own interior site: the rounded corner / centre
  // candidates are that site and no wrap applies)
  bool near_own = false;
  ub2 = kUbDirty;
  if (P.hash_r2 > 0.0) {
    const double h = 0.5 * par;
    const double ux = p.x - ((double)cx + h) * P.G.a0, uy = p.y - ((double)cy + h) * P.G.a0,
                 uz = p.z - ((double)(cz + P.G.zoff) + h) * P.G.a0;
    const double u2 = fma(ux, ux, fma(uy, uy, uz * uz));
    near_own = u2 < P.hash_r2;
    if (near_own) ub2 = u2;
  }
  if (!near_own && !wrap_position(p.x, p.y, p.z, P.G)) {
    set_error(P.st, CBX_LOGIC);
    return;
  }
  const long long real = near_own ? own : nearest_site(p.x, p.y, p.z, P.G);
  if (real < 0) {
    if (atomicCAS(&P.st->err, 0, CBX_DOMAIN) == 0) {
      P.st->err_pos[0] = p.x;
      P.st->err_pos[1] = p.y;
      P.st->err_pos[2] = p.z;
    }
    return;
  }
  if (real != own) {  // pass 1: evict to the clash map under the new hash
    const int dir = owner_dir(real, P.G);
    const Movers& M = dir ? P.out : P.mv;
    const int m = atomicAdd(dir ? &P.st->n_out : &P.st->n_mov, 1);
    if (m >= P.cap_mov) {
      set_error(P.st, CBX_RUNTIME);
      return;
    }
    if (dir) M.dir[m] = dir;
    M.key[m] = real;
    M.walk[m] = real;
    M.cls[m] = 1;
    M.sub[m] = own;
    M.px[m] = p.x;
    M.py[m] = p.y;
    M.pz[m] = p.z;
    M.vx[m] = vx;
    M.vy[m] = vy;
    M.vz[m] = vz;
    M.tag[m] = P.tag[d];
    P.pdf[d] = make_double4(kVacant, kVacant, kVacant, 0.0);
    P.uf[d] = make_float4(kVacantF, kVacantF, kVacantF, __int_as_float(-1));
    if (images) ghost_images_at(P, par, cx, cy, cz, make_double4(kVacant, kVacant, kVacant, 0.0));
  } else {
    P.pdf[d] = p;
    P.uf[d] = make_float4((float)p.x, (float)p.y, (float)p.z, __int_as_float(-1));
    if (images) ghost_images_at(P, par, cx, cy, cz, p);
  }
}

// regional displacement bound of the warp's chunk (32 consecutive interior
// cells of one row when bx % 32 == 0): the largest |u| of its atoms, rounded
// up to kUbScale units; atomicMax because both sublattices' warps write it
__device__ __forceinline__ void ub_note_chunk(const KP& P, long long chunk, double v,
                                              unsigned long long stamp) {
  for (int o = 16; o > 0; o >>= 1) v = fmax(v, __shfl_xor_sync(0xffffffffu, v, o));
  if ((threadIdx.x & 31) == 0 && v >= 0.0) {
    const unsigned long long q =
        v >= kUbDirty ? kUbQMax
                      : min(kUbQMax, (unsigned long long)(sqrt(v) * kUbScale) + 2ull);
    atomicMax(P.ub + chunk, (stamp << kUbShift) | q);
  }
}
__device__ __forceinline__ void ub_note(const KP& P, int vb, double v, unsigned long long stamp) {
  ub_note_chunk(P, (long long)vb * 4 + ((threadIdx.x >> 5) & 3), v, stamp);
}

// a single wave of blocks (resident on every SM) walks the virtual blocks

// (two virtual blocks per thread with both sites' loads in flight measured
// slower at config 5: 1.89 vs 1.79 ms, 80 registers and spills)
__global__ void __launch_bounds__(256, 4)
    k_kick_drift(KP P, int move, int nsb, int zero_acc, int images, int nvb, int n_pairp,
                 int n_emb, int n_ke) {
  if (blockIdx.x == nsb) {  // an idle clash block: the previous step's StepState
    // sums (the step's dt is fixed when they are deferred)
    finalize_pending<256>(P);
  }
  // a failed step (device error or overlap, stable since the previous
  // step's passes) ends the replay: no further kick, drift or rehash
  if (P.st->err || P.st->n_ovl) return;
  // slab ranks with the merged kick: the neighbours' force partials of the
  // previous step (fused reverse halo) are in before any force is read
  if (P.rev_wait && !rev_wait(P, P.rev_wait)) return;
  if (blockIdx.x >= nsb) {  // the clash records (fused k_clash_kick_drift)
    if (P.st->k2_pending) clash_kick2_sums(P, blockIdx.x - nsb);
    clash_kick_drift_body(P, move, blockIdx.x - nsb, gridDim.x - nsb);
    return;
  }
  // the step's dt and half kick once per block (sim.cpp:250); a pending
  // second half kick of the previous step (same fixed dt) runs first
  __shared__ double s_kick[2];
  __shared__ int s_k2;
  __shared__ unsigned long long s_stamp;
  if (threadIdx.x == 0) {
    const double dt = P.st->dt_next;
    s_kick[0] = dt;
    s_kick[1] = half_kick(P, dt);
    s_k2 = P.st->k2_pending;
    if (P.ub) {
      s_stamp = P.ustamp[1];
      // the bounds of the previous step no longer describe the store; the
      // pass-2 kernel after this one publishes this step's stamp
      if (blockIdx.x == 0) P.ustamp[0] = 0;
    }
  }
  __syncthreads();
  const double dt = s_kick[0], hk = s_kick[1];
  const bool k2 = s_k2 != 0;
  const unsigned long long stamp = s_stamp;
  double v2s = 0.0, v2m = 0.0;
  for (int vb = blockIdx.x; vb < nvb; vb += nsb) {
    double ub2 = -1.0;
    kick_drift_site(P, move, zero_acc, images, vb, dt, hk, k2, v2s, v2m, ub2);
    if (P.ub) ub_note(P, vb, ub2, stamp);
  }
  if (k2) {  // the previous step's KE / v_max partials (k_kick2's, per block)
    __shared__ double sh[8];
    const double sv = block_sum<256>(v2s, sh);
    const double mv = block_max<256>(v2m, sh);
    if (threadIdx.x == 0) {
      P.part_ke[blockIdx.x] = sv;
      P.part_vmax[blockIdx.x] = mv;
    }
  }
}

// ---- kick/drift with TMA bulk staging (rows cut into runs of up to 128
// cells): one thread per CTA streams the inputs of the virtual blocks
// kKdStages ahead into shared memory (cp.async.bulk + mbarrier); the 256
// threads read their site from there, so no load occupies a register while
// it is in flight and each SM keeps ~165 KB of reads outstanding (the
// register-staged sweep above holds at most one site per thread).  A virtual
// block's 128 cells are consecutive in one row: per sublattice one 4 KB pdf
// run and, per velocity / force component, one run of 128 doubles copied
// from the 16-byte boundary below it (kKdChunk doubles).
constexpr int kKdChunk = 130;
struct KdStage {
  double4 pdf[2][128];
  double vel[3][2][kKdChunk];
  double frc[3][2][kKdChunk];
};
constexpr unsigned kKdStageBytes = sizeof(KdStage);
static_assert(kKdStageBytes % 16 == 0, "stage size");

// virtual block vb of the bulk sweep: segment seg (128 cells, the last one of
// a row shorter when bx % 128 != 0) of interior row `row` = vb / nsr
__host__ __device__ __forceinline__ int kd_segs(const Geo& G) { return (G.bx + 127) / 128; }
template <bool FR>  // FR: bx % 128 == 0, every run 128 cells
__device__ __forceinline__ long long kd_cell0(const KP& P, int vb, int& cx0, int& cy, int& cz,
                                              int& len, int& row) {
  const Geo& G = P.G;
  const int nsr = kd_segs(G);
  row = vb / nsr;
  cx0 = (vb - row * nsr) * 128;
  len = FR ? 128 : min(128, G.bx - cx0);
  cy = row % G.by;
  cz = row / G.by;
  return cell_of(cx0 + G.g, cy + G.g, cz + G.g, G);
}
template <bool FR>
__device__ __forceinline__ void kd_issue(const KP& P, KdStage* st, unsigned mbar, int vb) {
  int cx0, cy, cz, len, row;
  const long long c0 = kd_cell0<FR>(P, vb, cx0, cy, cz, len, row);
  const long long S = P.S, NC = P.G.NC;
  unsigned bytes = 0;
  for (int p = 0; p < 2; ++p)
    bytes += 32u * len + 48u * ((((p * NC + c0) & 1) + len + 1) & ~1);
  mbar_expect_tx(mbar, bytes);
  for (int p = 0; p < 2; ++p) {
    const long long d0 = p * NC + c0, a0 = d0 & ~1ll;
    // the 8-byte runs from the 16-byte boundary below, an even count
    const unsigned n8 = 8u * (unsigned)((((d0 & 1) + len + 1) & ~1));
    bulk_g2s(smem_addr(&st->pdf[p][0]), P.pdf + d0, 32u * len, mbar);
    for (int a = 0; a < 3; ++a) {
      bulk_g2s(smem_addr(&st->vel[a][p][0]), P.vel + a * S + a0, n8, mbar);
      bulk_g2s(smem_addr(&st->frc[a][p][0]), P.frc + a * S + a0, n8, mbar);
    }
  }
}

template <int NS, int MINB, bool FR>
__global__ void __launch_bounds__(256, MINB)
    k_kick_drift_bulk(KP P, int move, int nsb, int zero_acc, int images, int nvb) {
  if (blockIdx.x == nsb) finalize_pending<256>(P);
  if (P.st->err || P.st->n_ovl) return;
  if (P.rev_wait && !rev_wait(P, P.rev_wait)) return;
  if (blockIdx.x >= nsb) {
    if (P.st->k2_pending) clash_kick2_sums(P, blockIdx.x - nsb);
    clash_kick_drift_body(P, move, blockIdx.x - nsb, gridDim.x - nsb);
    return;
  }
  extern __shared__ __align__(128) unsigned char kd_smem[];
  KdStage* stg = reinterpret_cast<KdStage*>(kd_smem);
  __shared__ __align__(8) unsigned long long s_full[NS];
  __shared__ double s_kick[2];
  __shared__ int s_k2;
  __shared__ unsigned long long s_stamp;
  const int t = threadIdx.x;
  if (t == 0) {
    const double dt = P.st->dt_next;
    s_kick[0] = dt;
    s_kick[1] = half_kick(P, dt);
    s_k2 = P.st->k2_pending;
    if (P.ub) {
      s_stamp = P.ustamp[1];
      if (blockIdx.x == 0) P.ustamp[0] = 0;
    }
    for (int q = 0; q < NS; ++q) mbar_init(smem_addr(&s_full[q]));
    for (int q = 0; q < NS; ++q) {
      const int vb = blockIdx.x + q * nsb;
      if (vb < nvb) kd_issue<FR>(P, &stg[q], smem_addr(&s_full[q]), vb);
    }
  }
  __syncthreads();
  const double dt = s_kick[0], hk = s_kick[1];
  const bool k2 = s_k2 != 0;
  const unsigned long long stamp = s_stamp;
  const int par = t >> 7, i = t & 127;
  double v2s = 0.0, v2m = 0.0;
  int it = 0;
  for (int vb = blockIdx.x; vb < nvb; vb += nsb, ++it) {
    const int q = it % NS;
    mbar_wait(smem_addr(&s_full[q]), (unsigned)(it / NS) & 1u);
    const KdStage& st = stg[q];
    KdSite a;
    int cx0, len, row;
    const long long c0 = kd_cell0<FR>(P, vb, cx0, a.cy, a.cz, len, row);
    const long long d = par * P.G.NC + c0;
    const int o = (int)(d & 1) + i;
    double ub2 = -1.0;
    if (i < len) {
      a.d = d + i;
      a.par = par;
      a.cx = cx0 + i + P.G.g;
      a.cy += P.G.g;
      a.cz += P.G.g;
      a.live = true;
      a.p = st.pdf[par][i];
      a.vx = st.vel[0][par][o];
      a.vy = st.vel[1][par][o];
      a.vz = st.vel[2][par][o];
      a.fx = st.frc[0][par][o];
      a.fy = st.frc[1][par][o];
      a.fz = st.frc[2][par][o];
      kick_drift_proc(P, move, zero_acc, images, dt, hk, k2, v2s, v2m, a, ub2);
    }
    // chunk of 32 cells of the row (bx % 32 == 0 wherever P.ub is set)
    if (P.ub) ub_note_chunk(P, (long long)row * (P.G.bx >> 5) + (cx0 >> 5) + ((t >> 5) & 3),
                            ub2, stamp);
    __syncthreads();  // stage q is read by every thread: refill it
    if (t == 0) {
      const int vn = vb + NS * nsb;
      if (vn < nvb) kd_issue<FR>(P, &stg[q], smem_addr(&s_full[q]), vn);
    }
  }
  if (k2) {
    __shared__ double sh[8];
    const double sv = block_sum<256>(v2s, sh);
    const double mv = block_max<256>(v2m, sh);
    if (t == 0) {
      P.part_ke[blockIdx.x] = sv;
      P.part_vmax[blockIdx.x] = mv;
    }
  }
}

// merged kick: the clash records' part of the previous step's second half
// kick (clash_kick2_body) and of its StepState sums, before the rehash of
// this step reorders the records: one partial per clash block in the
// reserved slots n_part - kClashSlots + blk (finalize_body, clash_slots)
__device__ void clash_kick2_sums(const KP& P, int blk) {
  const int n = P.st->n_clash;
  double ee = 0.0, ep = 0.0, s2 = 0.0, m2 = 0.0;
  for (int i = blk * blockDim.x + threadIdx.x; i < n; i += kClashSlots * blockDim.x) {
    ee += P.cl.e_emb[i];
    ep += P.cl.e_pair[i];
    double v2 = 0.0;
    if (!P.cl.gf[i]) {
      const double hk = half_kick(P, P.st->dt_next);
      const double vx = xadd(P.cl.vx[i], xmul(P.cl.fx[i], hk));
      const double vy = xadd(P.cl.vy[i], xmul(P.cl.fy[i], hk));
      const double vz = xadd(P.cl.vz[i], xmul(P.cl.fz[i], hk));
      P.cl.vx[i] = vx;
      P.cl.vy[i] = vy;
      P.cl.vz[i] = vz;
      v2 = exact_r2(vx, vy, vz);
    }
    P.cl.v2[i] = v2;
    s2 += v2;
    m2 = fmax(m2, v2);
  }
  __shared__ double sh[8];
  const double a = block_sum<256>(ee, sh), b = block_sum<256>(ep, sh);
  const double c = block_sum<256>(s2, sh), d = block_max<256>(m2, sh);
  if (threadIdx.x == 0) {
    const int q = P.n_part - kClashSlots + blk;
    P.part_emb[q] = a;
    P.part_pair[q] = b;
    P.part_ke[q] = c;
    P.part_vmax[q] = d;
  }
}

__device__ void clash_kick_drift_body(const KP& P, int move, int blk, int nblk) {
  if (P.st->err || P.st->n_ovl) return;
  const int n = P.st->n_clash;
  for (int i = blk * blockDim.x + threadIdx.x; i < n; i += nblk * blockDim.x) {
    if (P.cl.gf[i]) continue;
    double px = P.cl.px[i], py = P.cl.py[i], pz = P.cl.pz[i];
    if (move) {
      const double dt = P.st->dt_next;
      const double hk = half_kick(P, dt);
      const double vx = xadd(P.cl.vx[i], xmul(P.cl.fx[i], hk));
      const double vy = xadd(P.cl.vy[i], xmul(P.cl.fy[i], hk));
      const double vz = xadd(P.cl.vz[i], xmul(P.cl.fz[i], hk));
      P.cl.vx[i] = vx;
      P.cl.vy[i] = vy;
      P.cl.vz[i] = vz;
      px = xadd(px, xmul(vx, dt));
      py = xadd(py, xmul(vy, dt));
      pz = xadd(pz, xmul(vz, dt));
    }
    if (!wrap_position(px, py, pz, P.G)) {
      set_error(P.st, CBX_LOGIC);
      return;
    }
    P.cl.px[i] = px;
    P.cl.py[i] = py;
    P.cl.pz[i] = pz;
    const long long real = nearest_site(px, py, pz, P.G);  // store.cpp:64
    if (real < 0 && atomicCAS(&P.st->err, 0, CBX_DOMAIN) == 0) {
      P.st->err_pos[0] = px;
      P.st->err_pos[1] = py;
      P.st->err_pos[2] = pz;
    }
    P.cl.hkey[i] = real;
    const int dir = real < 0 ? 0 : owner_dir(real, P.G);
    if (dir) {  // the record migrates with its walk position
      const int m = atomicAdd(&P.st->n_out, 1);
      if (m >= P.cap_mov) {
        set_error(P.st, CBX_RUNTIME);
        return;
      }
      const Movers& M = P.out;
      M.dir[m] = dir;
      M.key[m] = real;
      M.walk[m] = P.cl.key[i];
      M.cls[m] = 0;
      M.sub[m] = i;
      M.px[m] = px;
      M.py[m] = py;
      M.pz[m] = pz;
      M.vx[m] = P.cl.vx[i];
      M.vy[m] = P.cl.vy[i];
      M.vz[m] = P.cl.vz[i];
      M.tag[m] = P.cl.tag[i];
      P.cl.gf[i] = 3;  // gone
    }
  }
}
__global__ void k_clash_kick_drift(KP P, int move) {
  clash_kick_drift_body(P, move, blockIdx.x, gridDim.x);
}

// ---------------------------------------------------- single-block helpers
// bitonic sort of (k1, k2, k3, pl) ascending by (k1, k2, k3) over n_pad
// (power of two) entries in global scratch; one block, all threads call it
__device__ void block_sort(long long* k1, long long* k2, long long* k3, int* pl, int n_pad) {
  for (int k = 2; k <= n_pad; k <<= 1) {
    for (int j = k >> 1; j > 0; j >>= 1) {
      for (int i = threadIdx.x; i < n_pad; i += blockDim.x) {
        const int q = i ^ j;
        if (q <= i) continue;
        const bool up = (i & k) == 0;
        const long long a1 = k1[i], b1 = k1[q];
        bool gt;
        if (a1 != b1) gt = a1 > b1;
        else if (k2[i] != k2[q]) gt = k2[i] > k2[q];
        else gt = k3[i] > k3[q];
        if (gt == up) {
          k1[i] = b1;
          k1[q] = a1;
          long long t = k2[i];
          k2[i] = k2[q];
          k2[q] = t;
          t = k3[i];
          k3[i] = k3[q];
          k3[q] = t;
          const int u = pl[i];
          pl[i] = pl[q];
          pl[q] = u;
        }
      }
      __syncthreads();
    }
  }
}

// exclusive prefix over flags[0..n) -> pos[], returns the total (all threads)
__device__ int block_scan(const int* flag, int* pos, int n) {
  __shared__ int s_cnt[1024];
  const int chunk = (n + blockDim.x - 1) / blockDim.x;
  const int lo = threadIdx.x * chunk, hi = min(n, lo + chunk);
  int c = 0;
  for (int i = lo; i < hi; ++i) c += flag[i];
  s_cnt[threadIdx.x] = c;
  __syncthreads();
  if (threadIdx.x == 0) {
    int run = 0;
    for (int t = 0; t < (int)blockDim.x; ++t) {
      const int v = s_cnt[t];
      s_cnt[t] = run;
      run += v;
    }
    s_cnt[blockDim.x - 1 + 0] += 0;
  }
  __syncthreads();
  int run = s_cnt[threadIdx.x];
  for (int i = lo; i < hi; ++i) {
    pos[i] = run;
    run += flag[i];
  }
  __syncthreads();
  __shared__ int s_total;
  if (threadIdx.x == blockDim.x - 1) s_total = run;
  __syncthreads();
  const int tot = s_total;
  __syncthreads();
  return tot;
}

__device__ __forceinline__ int pad_pow2(int n) {
  int p = 1;
  while (p < n) p <<= 1;
  return p;
}

__device__ __forceinline__ void copy_record(const Clash& a, int i, const Clash& b, int j) {
  b.key[j] = a.key[i];
  b.hkey[j] = a.hkey[i];
  b.gf[j] = a.gf[i];
  b.src[j] = a.src[i];
  b.px[j] = a.px[i];
  b.py[j] = a.py[i];
  b.pz[j] = a.pz[i];
  b.vx[j] = a.vx[i];
  b.vy[j] = a.vy[i];
  b.vz[j] = a.vz[i];
  b.fx[j] = a.fx[i];
  b.fy[j] = a.fy[i];
  b.fz[j] = a.fz[i];
  b.rho[j] = a.rho[i];
  b.df[j] = a.df[i];
  b.e_emb[j] = a.e_emb[i];
  b.e_pair[j] = a.e_pair[i];
  b.v2[j] = a.v2[i];
  b.tag[j] = a.tag[i];
}

// ------------------------------------------------- update_hash pass 2
// The reference walks the clash map in key order (store.cpp:59-75); pass-1
// evictees sit at the end of bucket `new hash` in ascending old-site order
// (they were appended while scanning slots in id order).  Each record goes
// to its hashed slot if that slot is free and interior, else to keep[hash].
// A slot's state only changes through its own promotions, so records with
// the same hash form independent groups processed in walk order: sorting by
// (hash, walk key, class, order) makes the group's first record the one
// that claims a free slot and the rest the new bucket, in order.
__device__ void ghost_images(const KP& P, long long d, const double4& p);

// single-block store passes (after kick/drift, before the step's density
// pass): the status words are stable here, so a failure of an earlier step
// of the replay raises `halt` and the remaining passes of the call skip
__device__ bool halt_check(const KP& P) {
  __shared__ int s_halt;
  if (threadIdx.x == 0) {
    DevStatus* st = P.st;
    s_halt = (st->err | st->n_ovl) != 0;
    if (s_halt) st->halt = 1;
  }
  __syncthreads();
  return s_halt != 0;
}

// regional displacement bounds (cbx_device.cuh): a slot filled by pass 2
// makes its chunk unbounded for this step; once pass 2 is done the stamp of
// this step's k_kick_drift becomes the one the density pass accepts
__device__ __forceinline__ void ub_dirty(const KP& P, long long dr) {
  if (!P.ub) return;
  const Geo& G = P.G;
  int cx, cy, cz;
  cell_xyz(dr >= G.NC ? dr - G.NC : dr, G, cx, cy, cz);
  const long long e = ((long long)(cz - G.g) * G.by + (cy - G.g)) * G.bx + (cx - G.g);
  atomicMax(P.ub + (e >> 5), (P.ustamp[1] << kUbShift) | kUbQMax);
}
__device__ __forceinline__ void ub_publish(const KP& P) {
  if (!P.ub || P.st->err || P.st->n_ovl) return;
  const unsigned long long s = P.ustamp[1];
  P.ustamp[0] = s;
  P.ustamp[1] = s + 1;
}

__device__ void rehash_body(const KP& P) {
  if (P.st->err || P.st->n_ovl) return;
  const int n_old = P.st->n_clash;
  const int n_mov = min(P.st->n_mov, P.cap_mov);
  if (n_old == 0 && n_mov == 0) return;
  __shared__ int s_n;
  if (threadIdx.x == 0) s_n = 0;
  for (int i = threadIdx.x; i < n_old; i += blockDim.x)
    P.head[dev_of_ref(P.cl.key[i], P.G.NC)] = -1;
  __syncthreads();
  const Scratch& X = P.sc;
  for (int i = threadIdx.x; i < n_old; i += blockDim.x) {
    if (P.cl.gf[i]) continue;  // ghost images are rebuilt; gf 3 = migrated away
    const long long real = P.cl.hkey[i];
    if (real < 0) continue;
    const int k = atomicAdd(&s_n, 1);
    X.k1[k] = real;
    X.k2[k] = P.cl.key[i];
    X.k3[k] = (1ll << 60) + i;
    X.pl[k] = i;
  }
  __syncthreads();
  const int base = s_n;
  if (base + n_mov > P.cap_items) {
    if (threadIdx.x == 0) set_error(P.st, CBX_RUNTIME);
    return;
  }
  for (int m = threadIdx.x; m < n_mov; m += blockDim.x) {
    X.k1[base + m] = P.mv.key[m];
    X.k2[base + m] = P.mv.walk[m];
    X.k3[base + m] = (long long)P.mv.cls[m] * (1ll << 61) + (1ll << 60) + P.mv.sub[m];
    X.pl[base + m] = -(m + 1);
  }
  const int n = base + n_mov;
  const int n_pad = pad_pow2(n);
  for (int i = n + threadIdx.x; i < n_pad; i += blockDim.x) {
    X.k1[i] = LLONG_MAX;
    X.k2[i] = LLONG_MAX;
    X.k3[i] = LLONG_MAX;
    X.pl[i] = 0;
  }
  __syncthreads();
  block_sort(X.k1, X.k2, X.k3, X.pl, n_pad);
  const long long S = P.S;
  for (int p = threadIdx.x; p < n; p += blockDim.x) {
    int promote = 0;
    const long long real = X.k1[p];
    if (p == 0 || X.k1[p - 1] != real) {
      const long long dr = dev_of_ref(real, P.G.NC);
      if (P.pdf[dr].x >= kVacantTest && !site_is_ghost(real, P.G)) {
        promote = 1;
        const int q = X.pl[p];
        if (q >= 0) {
          P.uf[dr] = make_float4((float)P.cl.px[q], (float)P.cl.py[q], (float)P.cl.pz[q],
                                 __int_as_float(-1));
          P.pdf[dr] = make_double4(P.cl.px[q], P.cl.py[q], P.cl.pz[q], 0.0);
          P.vel[dr] = P.cl.vx[q];
          P.vel[S + dr] = P.cl.vy[q];
          P.vel[2 * S + dr] = P.cl.vz[q];
          P.tag[dr] = P.cl.tag[q];
        } else {
          const int m = -q - 1;
          P.uf[dr] = make_float4((float)P.mv.px[m], (float)P.mv.py[m], (float)P.mv.pz[m],
                                 __int_as_float(-1));
          P.pdf[dr] = make_double4(P.mv.px[m], P.mv.py[m], P.mv.pz[m], 0.0);
          P.vel[dr] = P.mv.vx[m];
          P.vel[S + dr] = P.mv.vy[m];
          P.vel[2 * S + dr] = P.mv.vz[m];
          P.tag[dr] = P.mv.tag[m];
        }
        P.frc[dr] = 0.0;
        P.frc[S + dr] = 0.0;
        P.frc[2 * S + dr] = 0.0;
        ghost_images(P, dr, P.pdf[dr]);  // the slot's periodic images follow it
        ub_dirty(P, dr);  // no displacement bound for the slot's chunk this step
      }
    }
    X.flag[p] = !promote;
  }
  __syncthreads();
  const int n_new = block_scan(X.flag, X.pos, n);
  for (int p = threadIdx.x; p < n; p += blockDim.x) {
    if (!X.flag[p]) continue;
    const int j = X.pos[p];
    const int q = X.pl[p];
    const Clash& B = P.cl2;
    B.key[j] = X.k1[p];
    B.gf[j] = 0;
    B.src[j] = j;
    if (q >= 0) {
      B.px[j] = P.cl.px[q];
      B.py[j] = P.cl.py[q];
      B.pz[j] = P.cl.pz[q];
      B.vx[j] = P.cl.vx[q];
      B.vy[j] = P.cl.vy[q];
      B.vz[j] = P.cl.vz[q];
      B.tag[j] = P.cl.tag[q];
      B.fx[j] = P.cl.fx[q];
      B.fy[j] = P.cl.fy[q];
      B.fz[j] = P.cl.fz[q];
    } else {
      const int m = -q - 1;
      B.px[j] = P.mv.px[m];
      B.py[j] = P.mv.py[m];
      B.pz[j] = P.mv.pz[m];
      B.vx[j] = P.mv.vx[m];
      B.vy[j] = P.mv.vy[m];
      B.vz[j] = P.mv.vz[m];
      B.tag[j] = P.mv.tag[m];
      B.fx[j] = 0.0;
      B.fy[j] = 0.0;
      B.fz[j] = 0.0;
    }
    B.rho[j] = 0.0;
    B.df[j] = 0.0;
    B.e_emb[j] = 0.0;
    B.e_pair[j] = 0.0;
    B.v2[j] = 0.0;
  }
  __syncthreads();
  for (int j = threadIdx.x; j < n_new; j += blockDim.x) copy_record(P.cl2, j, P.cl, j);
  if (threadIdx.x == 0) {
    P.st->n_clash = n_new;
    P.st->n_mov = 0;
  }
}
__global__ void __launch_bounds__(1024) k_rehash(KP P, int merge, int n_emb, int n_pairp,
                                                 int n_ke) {
  pdl_wait();
  pdl_trigger();
  if (halt_check(P)) return;
  if (merge && threadIdx.x == 0 && P.st->k2_pending) {
    // slab ranks (peer memory), merged kick: k_kick_drift ran the previous
    // step's second half kick; its StepState sums and the cross-rank
    // reduction become pending for the density pass's idle block
    DevStatus* st = P.st;
    st->fin_bad = 0;
    st->k2_pending = 0;
    st->fin_stepping = 1;
    st->fin_energies = 1;
    st->fin_nemb = n_emb;
    st->fin_npp = n_pairp;
    st->fin_nke = n_ke;
    st->fin_clash = kClashSlots;
    st->fin_reduce = 1;
    st->fin_pending = 1;
  }
  rehash_body(P);
  __syncthreads();
  if (threadIdx.x == 0) ub_publish(P);
}

// ------------------------------------------------------ ghost slot images
// the images of interior site d with content p, from the source side: what
// k_ghost_fill writes for every ghost whose source is d (same arithmetic)
__device__ void ghost_images(const KP& P, long long d, const double4& p) {
  const Geo& G = P.G;
  const int par = d >= G.NC;
  int cx, cy, cz;
  cell_xyz(d - par * G.NC, G, cx, cy, cz);
  ghost_images_at(P, par, cx, cy, cz, p);
}
__device__ void ghost_images_at(const KP& P, int par, int cx, int cy, int cz, const double4& p) {
  const Geo& G = P.G;
  // boxes at least 2g cells wide: at most one image shift per axis, the
  // images are the non-empty subsets of the shifted axes (the same position
  // arithmetic as the general enumeration below)
  if (G.kmx == 1 && G.kmy == 1 && G.kmz <= 1 && G.bx >= 2 * G.g && G.by >= 2 * G.g &&
      (G.kmz == 0 || G.bz >= 2 * G.g)) {
    const int sx = cx >= G.bx ? -1 : (cx < G.tx - G.bx ? 1 : 0);
    const int sy = cy >= G.by ? -1 : (cy < G.ty - G.by ? 1 : 0);
    const int sz = G.kmz == 0 ? 0 : (cz >= G.bz ? -1 : (cz < G.tz - G.bz ? 1 : 0));
    if (!(sx | sy | sz)) return;
    const bool vac = p.x >= kVacantTest;
    const float w = __int_as_float((int)(par * G.NC + cell_of(cx, cy, cz, G)));
    for (int m = 1; m < 8; ++m) {
      const int kx = (m & 1) ? sx : 0, ky = (m & 2) ? sy : 0, kz = (m & 4) ? sz : 0;
      if (((m & 1) && !sx) || ((m & 2) && !sy) || ((m & 4) && !sz)) continue;
      const long long di =
          par * G.NC + cell_of(cx + G.bx * kx, cy + G.by * ky, cz + G.bz * kz, G);
      if (vac) {
        P.pdf[di] = make_double4(kVacant, kVacant, kVacant, 0.0);
        P.uf[di] = make_float4(kVacantF, kVacantF, kVacantF, w);
        continue;
      }
      const double4 q = make_double4(xadd(p.x, xmul((double)kx, G.lx)),
                                     xadd(p.y, xmul((double)ky, G.ly)),
                                     xadd(p.z, xmul((double)kz, G.lz)), p.w);
      P.pdf[di] = q;
      P.uf[di] = make_float4((float)q.x, (float)q.y, (float)q.z, w);
    }
    return;
  }
  const long long d = par * G.NC + cell_of(cx, cy, cz, G);
  int xl = 0, xh = 0, yl = 0, yh = 0, zl = 0, zh = 0;  // valid image shifts per axis
  for (int k = 1; k <= G.kmx; ++k) {
    if (cx - k * G.bx >= 0) xl = -k;
    if (cx + k * G.bx < G.tx) xh = k;
  }
  for (int k = 1; k <= G.kmy; ++k) {
    if (cy - k * G.by >= 0) yl = -k;
    if (cy + k * G.by < G.ty) yh = k;
  }
  for (int k = 1; k <= G.kmz; ++k) {
    if (cz - k * G.bz >= 0) zl = -k;
    if (cz + k * G.bz < G.tz) zh = k;
  }
  if (xl == 0 && xh == 0 && yl == 0 && yh == 0 && zl == 0 && zh == 0) return;
  const bool vac = p.x >= kVacantTest;
  const float w = __int_as_float((int)d);
  for (int kz = zl; kz <= zh; ++kz)
    for (int ky = yl; ky <= yh; ++ky)
      for (int kx = xl; kx <= xh; ++kx) {
        if (kx == 0 && ky == 0 && kz == 0) continue;
        const long long di =
            par * G.NC + cell_of(cx + G.bx * kx, cy + G.by * ky, cz + G.bz * kz, G);
        if (vac) {
          P.pdf[di] = make_double4(kVacant, kVacant, kVacant, 0.0);
          P.uf[di] = make_float4(kVacantF, kVacantF, kVacantF, w);
          continue;
        }
        const double4 q = make_double4(xadd(p.x, xmul((double)kx, G.lx)),
                                       xadd(p.y, xmul((double)ky, G.ly)),
                                       xadd(p.z, xmul((double)kz, G.lz)), p.w);
        P.pdf[di] = q;
        P.uf[di] = make_float4((float)q.x, (float)q.y, (float)q.z, w);
      }
}

// each ghost site has one periodic source; its image position is the
// source's plus k*len, added per axis exactly like store.cpp:166-169
__global__ void k_ghost_fill(KP P) {
  pdl_wait();
  pdl_trigger();
  if (P.st->err) return;
  const long long g = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (g >= P.n_gh) return;
  const int dst = P.gh_dst[g], src = P.gh_src[g];
  const double4 p = P.pdf[src];
  if (p.x >= kVacantTest) {
    P.pdf[dst] = make_double4(kVacant, kVacant, kVacant, 0.0);
    P.uf[dst] = make_float4(kVacantF, kVacantF, kVacantF, __int_as_float(src));
    return;
  }
  const signed char* k = P.gh_k + 3 * g;
  const double4 q = make_double4(xadd(p.x, xmul((double)k[0], P.G.lx)),
                                 xadd(p.y, xmul((double)k[1], P.G.ly)),
                                 xadd(p.z, xmul((double)k[2], P.G.lz)), p.w);
  P.pdf[dst] = q;
  P.uf[dst] = make_float4((float)q.x, (float)q.y, (float)q.z, __int_as_float(src));
}

// --------------------------------------------------- ghost clash images
// store.cpp:160-194 for clash atoms: images of every interior record in
// (key, index) order, k loop z-y-x; a ghost bucket keeps its source
// bucket's order.  An image whose ghost slot is free would take the slot in
// the reference; update_hash never leaves an interior bucket over a vacant
// slot, so that state is rejected (CBX_INVALID_ARGUMENT) instead.
// z-slab ranks (G.kmz = 0) also receive the interior clash records of the
// neighbours' boundary planes (P.rem, position halo); each becomes a ghost
// record here with its x/y images, src = -(remote index + 2).
__device__ __forceinline__ int image_count(long long id, const Geo& G) {
  int cx, cy, cz;
  cell_xyz(id >> 1, G, cx, cy, cz);
  int c = 0;
  for (int kz = -G.kmz; kz <= G.kmz; ++kz)
    for (int ky = -G.kmy; ky <= G.kmy; ++ky)
      for (int kx = -G.kmx; kx <= G.kmx; ++kx) {
        if (kx == 0 && ky == 0 && kz == 0) continue;
        const int ix = cx + G.bx * kx, iy = cy + G.by * ky, iz = cz + G.bz * kz;
        if (ix < 0 || ix >= G.tx || iy < 0 || iy >= G.ty || iz < 0 || iz >= G.tz) continue;
        ++c;
      }
  return c;
}

__device__ void clash_images_body(const KP& P, int zero_rho) {
  if (zero_rho && threadIdx.x == 0) P.work[0] = 0;  // the density pass's brick queue
  if (P.st->err || P.st->n_ovl) return;
  const int n = P.st->n_clash;
  const int n_rem = P.st->n_remote;
  if (n == 0 && n_rem == 0) return;
  const Scratch& X = P.sc;
  const Geo& G = P.G;
  for (int i = threadIdx.x; i < n; i += blockDim.x) {
    P.head[dev_of_ref(P.cl.key[i], G.NC)] = -1;
    X.flag[i] = P.cl.gf[i] == 0;
  }
  __syncthreads();
  const int n_int = block_scan(X.flag, X.pos, n);
  // interior records, in order, to cl2[0..n_int)
  for (int i = threadIdx.x; i < n; i += blockDim.x)
    if (X.flag[i]) copy_record(P.cl, i, P.cl2, X.pos[i]);
  __syncthreads();
  // sources: interior records r < n_int emit images; remote records emit
  // themselves plus images
  const int n_src = n_int + n_rem;
  for (int r = threadIdx.x; r < n_src; r += blockDim.x) {
    const long long id = r < n_int ? P.cl2.key[r] : P.rem.key[r - n_int];
    X.flag[r] = image_count(id, G) + (r < n_int ? 0 : 1);
  }
  __syncthreads();
  const int n_img = block_scan(X.flag, X.pos, n_src);
  const int total = n_int + n_img;
  if (total > P.cap_clash || total > P.cap_items) {
    if (threadIdx.x == 0) set_error(P.st, CBX_RUNTIME);
    return;
  }
  // sort items: interior records (key, r, 0); ghost records (key, r, 1 + seq)
  for (int r = threadIdx.x; r < n_src; r += blockDim.x) {
    const bool local = r < n_int;
    const int rr = r - n_int;
    const long long id = local ? P.cl2.key[r] : P.rem.key[rr];
    if (local) {
      X.k1[r] = id;
      X.k2[r] = r;
      X.k3[r] = 0;
      X.pl[r] = r;
    }
    const double sx = local ? P.cl2.px[r] : P.rem.px[rr];
    const double sy = local ? P.cl2.py[r] : P.rem.py[rr];
    const double sz = local ? P.cl2.pz[r] : P.rem.pz[rr];
    const int par = (int)(id & 1);
    int cx, cy, cz;
    cell_xyz(id >> 1, G, cx, cy, cz);
    int w = n_int + X.pos[r], seq = 0;
    for (int kz = -G.kmz; kz <= G.kmz; ++kz)
      for (int ky = -G.kmy; ky <= G.kmy; ++ky)
        for (int kx = -G.kmx; kx <= G.kmx; ++kx) {
          if (kx == 0 && ky == 0 && kz == 0 && local) continue;
          const int ix = cx + G.bx * kx, iy = cy + G.by * ky, iz = cz + G.bz * kz;
          if (ix < 0 || ix >= G.tx || iy < 0 || iy >= G.ty || iz < 0 || iz >= G.tz) continue;
          const long long iid = ref_id(cell_of(ix, iy, iz, G), par);
          if (local && P.pdf[dev_of_ref(iid, G.NC)].x >= kVacantTest)
            set_error(P.st, CBX_INVALID_ARGUMENT);
          P.cl2.key[w] = iid;
          P.cl2.gf[w] = 1;
          P.cl2.src[w] = local ? r : -(rr + 2);
          P.cl2.px[w] = xadd(sx, xmul((double)kx, G.lx));
          P.cl2.py[w] = xadd(sy, xmul((double)ky, G.ly));
          P.cl2.pz[w] = xadd(sz, xmul((double)kz, G.lz));
          P.cl2.vx[w] = local ? P.cl2.vx[r] : P.rem.vx[rr];
          P.cl2.vy[w] = local ? P.cl2.vy[r] : P.rem.vy[rr];
          P.cl2.vz[w] = local ? P.cl2.vz[r] : P.rem.vz[rr];
          P.cl2.fx[w] = 0.0;
          P.cl2.fy[w] = 0.0;
          P.cl2.fz[w] = 0.0;
          P.cl2.rho[w] = local ? P.cl2.rho[r] : 0.0;
          P.cl2.df[w] = local ? P.cl2.df[r] : P.rem.df[rr];
          P.cl2.e_emb[w] = 0.0;
          P.cl2.e_pair[w] = 0.0;
          P.cl2.v2[w] = 0.0;
          P.cl2.tag[w] = local ? P.cl2.tag[r] : P.rem.tag[rr];
          // remote sources order after every local source of the same key
          X.k1[w] = iid;
          X.k2[w] = local ? r : (1ll << 40) + rr;
          X.k3[w] = 1 + seq;
          X.pl[w] = w;
          ++w;
          ++seq;
        }
  }
  const int n_pad = pad_pow2(total);
  for (int i = total + threadIdx.x; i < n_pad; i += blockDim.x) {
    X.k1[i] = LLONG_MAX;
    X.k2[i] = LLONG_MAX;
    X.k3[i] = LLONG_MAX;
    X.pl[i] = 0;
  }
  __syncthreads();
  block_sort(X.k1, X.k2, X.k3, X.pl, n_pad);
  // final position of every interior record (for the images' src links)
  for (int p = threadIdx.x; p < total; p += blockDim.x)
    if (X.k3[p] == 0) X.flag[X.pl[p]] = p;
  __syncthreads();
  for (int p = threadIdx.x; p < total; p += blockDim.x) {
    const int q = X.pl[p];
    copy_record(P.cl2, q, P.cl, p);
    if (zero_rho) P.cl.rho[p] = 0.0;  // the density pass follows (clash_zero fused)
    const int sq = P.cl2.src[q];
    P.cl.src[p] = P.cl2.gf[q] ? (sq >= 0 ? X.flag[sq] : sq) : p;
    if (p == 0 || X.k1[p - 1] != X.k1[p]) P.head[dev_of_ref(X.k1[p], G.NC)] = p;
  }
  if (threadIdx.x == 0) P.st->n_clash = total;
}
__global__ void __launch_bounds__(1024) k_clash_images(KP P, int zero_rho) {
  pdl_wait();
  pdl_trigger();
  clash_images_body(P, zero_rho);
}
// the store phase's two single-block passes in one launch (the step path,
// whose slot images k_kick_drift and rehash_body already wrote)
__global__ void __launch_bounds__(1024) k_rehash_images(KP P, int merge, int n_emb, int n_pairp,
                                                       int n_ke) {
  pdl_wait();
  pdl_trigger();
  if (halt_check(P)) return;
  if (merge && threadIdx.x == 0 && P.st->k2_pending) {
    // k_kick_drift ran the previous step's second half kick: its StepState
    // sums become pending (for the density pass's idle block)
    DevStatus* st = P.st;
    st->fin_bad = 0;  // that step completed (else this step would have halted)
    st->fin_reduce = 0;
    st->k2_pending = 0;
    st->fin_stepping = 1;
    st->fin_energies = 1;
    st->fin_nemb = n_emb;
    st->fin_npp = n_pairp;
    st->fin_nke = n_ke;
    st->fin_clash = kClashSlots;  // the records' sums are in the reserved slots
    st->fin_pending = 1;
  }
  rehash_body(P);
  __syncthreads();
  clash_images_body(P, 1);
  __syncthreads();
  if (threadIdx.x == 0) ub_publish(P);
}

// fp32 shadow of every site from pdf (after a host upload)
__global__ void k_uf_refresh(KP P) {
  const long long d = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (d >= P.S) return;
  const double4 p = P.pdf[d];
  const int t = P.tgt[d];
  const float w = __int_as_float(t == d ? -1 : t);
  P.uf[d] = p.x >= kVacantTest ? make_float4(kVacantF, kVacantF, kVacantF, w)
                               : make_float4((float)p.x, (float)p.y, (float)p.z, w);
}
void launch_uf_refresh(const KP& P, cudaStream_t s) {
  k_uf_refresh<<<(int)((P.S + 255) / 256), 256, 0, s>>>(P);
}

// zero the accumulators of the clash records: what 0 density, 1 force
__global__ void k_clash_zero(KP P, int what) {
  const int n = P.st->n_clash;
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    if (what == 0) {
      P.cl.rho[i] = 0.0;
    } else {
      P.cl.fx[i] = 0.0;
      P.cl.fy[i] = 0.0;
      P.cl.fz[i] = 0.0;
      P.cl.e_pair[i] = 0.0;
    }
  }
}

// ---------------------------------------------- second half kick + measure
// Blocks [0, nsb) sweep the interior sites (grid-stride, one KE / v_max
// partial per block), blocks [nsb, grid) the clash records; the last block
// to arrive sums every partial into StepState (finalize_body), so one
// kernel ends the step.
__device__ void clash_kick2_body(const KP& P, int kick, int blk, int nblk) {
  if (P.st->err || P.st->n_ovl) return;
  const int n = P.st->n_clash;
  for (int i = blk * blockDim.x + threadIdx.x; i < n; i += nblk * blockDim.x) {
    if (P.cl.gf[i]) {
      P.cl.v2[i] = 0.0;
      continue;
    }
    double vx = P.cl.vx[i], vy = P.cl.vy[i], vz = P.cl.vz[i];
    if (kick) {
      const double hk = half_kick(P, P.st->dt_next);
      vx = xadd(vx, xmul(P.cl.fx[i], hk));
      vy = xadd(vy, xmul(P.cl.fy[i], hk));
      vz = xadd(vz, xmul(P.cl.fz[i], hk));
      P.cl.vx[i] = vx;
      P.cl.vy[i] = vy;
      P.cl.vz[i] = vz;
    }
    P.cl.v2[i] = exact_r2(vx, vy, vz);
  }
}


// fin: the last block to finish runs finalize_body (the StepState sums) --
// one launch less per step than a separate k_finalize
__global__ void __launch_bounds__(256, 6) k_kick2(KP P, int kick, int nsb, int fin, int stepping,
                                                  int energies, int n_pairp, int n_emb, int nvb) {
  pdl_wait();
  pdl_trigger();
  if (P.rev_wait && !rev_wait(P, P.rev_wait)) return;  // the neighbours' force partials
  // a standalone second half kick completes a merged-kick step (host flush)
  if (blockIdx.x == 0 && threadIdx.x == 0) P.st->k2_pending = 0;
  __shared__ double sh[8];
  if (blockIdx.x >= nsb) {  // the clash records (fused k_clash_kick2)
    clash_kick2_body(P, kick, blockIdx.x - nsb, gridDim.x - nsb);
  } else {
    double v2s = 0.0, v2m = 0.0;
    for (int vb = blockIdx.x; vb < nvb; vb += nsb) {
    double v2 = 0.0;
    int par;
    long long d;
    if (!P.st->err && !P.st->n_ovl && map_site(P, par, d, vb)) {
      // every load of the site issued before the first use (one memory round
      // trip per thread; a vacant slot's velocity/force reads are discarded)
      const long long S = P.S;
      const double px = P.pdf[d].x;
      double vx = P.vel[d], vy = P.vel[S + d], vz = P.vel[2 * S + d];
      const double fx = P.frc[d], fy = P.frc[S + d], fz = P.frc[2 * S + d];
      const double dt = P.st->dt_next;
      if (px < kVacantTest) {
        if (kick) {
          const double hk = half_kick(P, dt);
          vx = xadd(vx, xmul(fx, hk));
          vy = xadd(vy, xmul(fy, hk));
          vz = xadd(vz, xmul(fz, hk));
          P.vel[d] = vx;
          P.vel[S + d] = vy;
          P.vel[2 * S + d] = vz;
        }
        v2 = exact_r2(vx, vy, vz);
      }
    }
    v2s += v2;
    v2m = fmax(v2m, v2);
    }
    const double s = block_sum<256>(v2s, sh);
    const double m = block_max<256>(v2m, sh);
    if (threadIdx.x == 0) {
      P.part_ke[blockIdx.x] = s;
      P.part_vmax[blockIdx.x] = m;
    }
  }
  if (fin == 2) {  // deferred: the next step's k_kick_drift (or the host) sums
    if (blockIdx.x == 0 && threadIdx.x == 0) {
      P.st->fin_stepping = stepping;
      P.st->fin_energies = energies;
      P.st->fin_nemb = n_emb;
      P.st->fin_npp = n_pairp;
      P.st->fin_nke = nsb;
      P.st->fin_clash = 0;
      P.st->fin_bad = P.st->err | P.st->n_ovl;  // this step's outcome, stable here
      P.st->fin_reduce = 0;
      P.st->fin_pending = 1;
    }
    return;
  }
  if (!fin) return;
  __shared__ int s_last;
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence();  // this block's partials before its count
    s_last = atomicAdd(&P.st->fin_count, 1u) == gridDim.x - 1;
  }
  __syncthreads();
  if (!s_last) return;
  __threadfence();
  if (threadIdx.x == 0) P.st->fin_count = 0;
  // through the device copy of P: a noinline callee taking the parameter
  // struct by reference would copy it to the stack of every thread
  finalize_body<256>(*P.dself, stepping, energies, P.part_emb, n_emb, P.part_pair, n_pairp, nsb);
}

__global__ void k_clash_kick2(KP P, int kick) {
  clash_kick2_body(P, kick, blockIdx.x, gridDim.x);
}

// ------------------------------------------------------------- finalize
// (finalize_body / finalize_pending: finalize.cuh)
// L (device copy, slab ranks on the P2P transport): the cross-rank
// StepState reduction follows in the same kernel -- also after a device
// error, so the ranks stay in step
__global__ void __launch_bounds__(1024) k_finalize(KP P, int stepping, int energies,
                                                   int n_pairp, int n_emb, int n_ke,
                                                   const P2PLinks* L) {
  pdl_wait();
  pdl_trigger();
  finalize_body<1024>(P, stepping, energies, P.part_emb, n_emb, P.part_pair, n_pairp, n_ke);
  if (L) {
    __syncthreads();
    __threadfence();
    if (threadIdx.x == 0) p2p_reduce_thread(P, *L, energies, stepping >= 0);
  }
}

// ---------------------------------------------------------- count_defects
__global__ void __launch_bounds__(256) k_count_defects(KP P, unsigned long long* out) {
  int par;
  long long d;
  unsigned vac = 0;
  if (map_site(P, par, d) && P.pdf[d].x >= kVacantTest) vac = 1;
  for (int o = 16; o > 0; o >>= 1) vac += __shfl_xor_sync(0xffffffffu, vac, o);
  if ((threadIdx.x & 31) == 0 && vac) atomicAdd(&out[0], (unsigned long long)vac);
  if (blockIdx.x == 0) {  // clash buckets
    const int n = P.st->n_clash;
    for (int i = threadIdx.x; i < n; i += blockDim.x) {
      if (P.cl.gf[i]) continue;
      if (i > 0 && P.cl.key[i - 1] == P.cl.key[i]) continue;
      int sz = 0;
      for (int j = i; j < n && P.cl.key[j] == P.cl.key[i]; ++j) ++sz;
      const bool valid = P.pdf[dev_of_ref(P.cl.key[i], P.G.NC)].x < kVacantTest;
      atomicAdd(&out[1], (unsigned long long)((valid ? 1 : 0) + sz - 1));
      if (!valid) atomicAdd(&out[2], 1ull);  // vacancies to subtract
    }
  }
}

// -------------------------------------------------------------- launchers
constexpr int kClashBlocks = kClashSlots;  // blocks of 256 threads for clash-record sweeps
// per-site sweeps: one resident wave (blocks per SM x SMs) over eam_blocks
// virtual blocks
static int site_wave(const KP& P, int per_sm) {
  static int sms = [] {
    int n = 148, dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
    return n;
  }();
  static const int wave = ab_flag("CBX_SITE_WAVE", 1);  // 0: one block per virtual block
  return wave ? std::max(1, std::min(eam_blocks(P), per_sm * sms)) : eam_blocks(P);
}
// the bulk-staged sweep (a virtual block is a run of up to 128 cells of one
// row); CBX_KD_BULK=0 (A/B build) keeps the register sweep
bool kd_bulk(const KP& P) {
  static const int on = ab_flag("CBX_KD_BULK", 1);
  // rows of at least 96 cells: segments of 128 (the last of a row shorter)
  // keep >= 75 % of the lanes busy; narrower boxes take the register sweep
  return on && (P.G.bx % 128 == 0 || P.G.bx >= 96);
}
static int kd_nvb(const KP& P) { return kd_segs(P.G) * P.G.by * P.G.bz; }
// stages x CTAs per SM of the bulk sweep (CBX_KD_CFG, A/B build: 42 = 4 x 2)
static int kd_cfg() {
  static const int c = ab_flag("CBX_KD_CFG", 42);
  return c;
}
int kick_drift_grid(const KP& P) {
  return kd_bulk(P) ? site_wave(P, kd_cfg() % 10) : site_wave(P, 4);
}
template <int NS, int MINB>
static void launch_kd_bulk(const KP& P, int move, cudaStream_t s, int zero_acc, int images,
                           int nsb) {
  static bool attr = false;
  const int bytes = NS * (int)kKdStageBytes;
  if (!attr) {
    cudaFuncSetAttribute(k_kick_drift_bulk<NS, MINB, true>,
                         cudaFuncAttributeMaxDynamicSharedMemorySize, bytes);
    cudaFuncSetAttribute(k_kick_drift_bulk<NS, MINB, false>,
                         cudaFuncAttributeMaxDynamicSharedMemorySize, bytes);
    attr = true;
  }
  if (P.G.bx % 128 == 0)
    k_kick_drift_bulk<NS, MINB, true><<<nsb + kClashBlocks, 256, bytes, s>>>(
        P, move, nsb, zero_acc, images, kd_nvb(P));
  else
    k_kick_drift_bulk<NS, MINB, false><<<nsb + kClashBlocks, 256, bytes, s>>>(
        P, move, nsb, zero_acc, images, kd_nvb(P));
}
void launch_kick_drift(const KP& P, int move, cudaStream_t s, int zero_acc, int images,
                       int n_pairp) {
  const int nsb = kick_drift_grid(P);
  if (kd_bulk(P)) {
    switch (kd_cfg()) {
      case 33: launch_kd_bulk<3, 3>(P, move, s, zero_acc, images, nsb); break;
      case 23: launch_kd_bulk<2, 3>(P, move, s, zero_acc, images, nsb); break;
      case 52: launch_kd_bulk<5, 2>(P, move, s, zero_acc, images, nsb); break;
      case 81: launch_kd_bulk<8, 1>(P, move, s, zero_acc, images, nsb); break;
      default: launch_kd_bulk<4, 2>(P, move, s, zero_acc, images, nsb);
    }
    return;
  }
  k_kick_drift<<<nsb + kClashBlocks, 256, 0, s>>>(P, move, nsb, zero_acc, images, eam_blocks(P),
                                                   n_pairp > 0 ? n_pairp : P.n_pair_part,
                                                   embed_grid(P), kick_grid(P));
}
void launch_rehash_images(const KP& P, cudaStream_t s, int merge, int n_emb, int n_pairp,
                          int n_ke) {
  launch_pdl(k_rehash_images, 1, 1024, 0, s, P, merge, n_emb, n_pairp, n_ke);
}
void launch_rehash(const KP& P, cudaStream_t s, int merge, int n_emb, int n_pairp, int n_ke) {
  launch_pdl(k_rehash, 1, 1024, 0, s, P, merge, n_emb, n_pairp, n_ke);
}
void launch_ghost_fill(const KP& P, cudaStream_t s) {
  if (P.n_gh) launch_pdl(k_ghost_fill, (int)((P.n_gh + 255) / 256), 256, 0, s, P);
}
void launch_clash_images(const KP& P, cudaStream_t s, int zero_rho) {
  launch_pdl(k_clash_images, 1, 1024, 0, s, P, zero_rho);
}
void launch_clash_zero(const KP& P, int what, cudaStream_t s) {
  k_clash_zero<<<8, 256, 0, s>>>(P, what);
}
int kick_grid(const KP& P) { return site_wave(P, 6); }
// stepping > -2: the StepState finalize runs in the last k_kick2 block
void launch_kick2(const KP& P, int kick, int stepping, int energies, cudaStream_t s, int fin,
                  int n_pairp) {
  const int nsb = kick_grid(P);
  launch_pdl(k_kick2, nsb + kClashBlocks, 256, 0, s, P, kick, nsb, stepping > -2 ? fin : 0,
             stepping, energies, n_pairp > 0 ? n_pairp : P.n_pair_part, embed_grid(P),
             eam_blocks(P));
}
__global__ void __launch_bounds__(1024) k_finalize_pending(KP P) { finalize_pending<1024>(P); }
void launch_finalize_pending(const KP& P, cudaStream_t s) {
  k_finalize_pending<<<1, 1024, 0, s>>>(P);
}
void launch_finalize(const KP& P, int stepping, int energies, cudaStream_t s,
                     const P2PLinks* links) {
  launch_pdl(k_finalize, 1, 1024, 0, s, P, stepping, energies, P.n_pair_part, embed_grid(P),
             kick_grid(P), links);
}
void launch_count_defects(const KP& P, unsigned long long* out, cudaStream_t s) {
  k_count_defects<<<eam_blocks(P), 256, 0, s>>>(P, out);
}

}  // namespace cbx

namespace cbx {
bool pdl_enabled() {
  static const bool on = ab_flag("CBX_PDL", 1) != 0;
  return on;
}
}  // namespace cbx
