// eam_kernels.cu -- the three EAM passes on sm_100a.
//
// Reference: core/src/forces.cpp (paths relative to /root/reference/proj).
//   density_slots  109-137   -> k_density<NEWTON3|FULL>
//   pair_slots     139-174   -> k_force<NEWTON3|FULL>
//   embed_slots    256-275   -> k_embed (+ refresh_ghosts 296-303 fused)
//   visit_clash_pairs + density_clash / pair_clash 185-254 -> k_clash<...>
//   embed_clash    277-288   -> k_clash_embed
//   fold_rho / fold_force 290-309 -> folded at scatter time: every partner
//       contribution is added to the partner's owner (tgt[]), which is the
//       ghost image's periodic source.
//
// The paper's red/blue colouring (forces.cpp:343-366) is replaced by one of
//   NEWTON3: the reference's half lists (56 candidates / 29 pairs per atom);
//            partner contributions are reduced into owners with RED.ADD.F64.
//   FULL:    full lists, each owner accumulates only itself (plain stores,
//            bitwise deterministic); 2x the pair work.
// Both visit exactly the reference's candidate set and compute every r^2 in
// the reference's orientation and operation order (no FMA), so in-cutoff
// decisions are bit-identical; the pair arithmetic after the cutoff test is
// ordinary fp64 (within 1e-10 of the reference, tests/test_gpu_parity.py).
#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <vector>

#include "cbx_device.cuh"
#include "p2p.cuh"
#include "finalize.cuh"

namespace cbx {

__constant__ int c_half_n[2];
__constant__ int c_full_n[2];
__constant__ int c_half_nin[2];  // leading offsets with lattice distance <= cutoff
__constant__ int c_full_nin[2];
__constant__ int c_half[2][kMaxOffsets];
__constant__ int c_full[2][kMaxOffsets];
__constant__ long long c_full_flat[2][kMaxOffsets];

void upload_offsets(const int* half_dev[2], const int half_n[2], const int* full_dev[2],
                    const int full_n[2], const long long* full_flat[2], const int half_nin[2],
                    const int full_nin[2], cudaStream_t s) {
  cudaMemcpyToSymbolAsync(c_half_nin, half_nin, 2 * sizeof(int), 0, cudaMemcpyHostToDevice, s);
  cudaMemcpyToSymbolAsync(c_full_nin, full_nin, 2 * sizeof(int), 0, cudaMemcpyHostToDevice, s);
  cudaMemcpyToSymbolAsync(c_half_n, half_n, 2 * sizeof(int), 0, cudaMemcpyHostToDevice, s);
  cudaMemcpyToSymbolAsync(c_full_n, full_n, 2 * sizeof(int), 0, cudaMemcpyHostToDevice, s);
  for (int p = 0; p < 2; ++p) {
    cudaMemcpyToSymbolAsync(c_half, half_dev[p], half_n[p] * sizeof(int),
                            p * kMaxOffsets * sizeof(int), cudaMemcpyHostToDevice, s);
    cudaMemcpyToSymbolAsync(c_full, full_dev[p], full_n[p] * sizeof(int),
                            p * kMaxOffsets * sizeof(int), cudaMemcpyHostToDevice, s);
    cudaMemcpyToSymbolAsync(c_full_flat, full_flat[p], full_n[p] * sizeof(long long),
                            p * kMaxOffsets * sizeof(long long), cudaMemcpyHostToDevice, s);
  }
}

// ---------------------------------------------------------------- splines
// spline.cpp:79-93 with the reference's clamps; value only / value+deriv
__device__ __forceinline__ double seg_value(const Tab& T, double x) {
  if (x < T.x0) x = T.x0;
  if (x > T.xl) x = T.xl;
  int i = (int)((x - T.x0) / T.h);
  i = max(0, min(i, T.nseg - 1));
  const double t = x - (T.x0 + T.h * (double)i);
  const double* g = T.seg + 7 * (size_t)i;
  return ((__ldg(g) * t + __ldg(g + 1)) * t + __ldg(g + 2)) * t + __ldg(g + 3);
}
__device__ __forceinline__ void seg_eval(const Tab& T, double x, double& v, double& dv) {
  if (x < T.x0) x = T.x0;
  if (x > T.xl) x = T.xl;
  int i = (int)((x - T.x0) / T.h);
  i = max(0, min(i, T.nseg - 1));
  const double t = x - (T.x0 + T.h * (double)i);
  const double* g = T.seg + 7 * (size_t)i;
  v = ((__ldg(g) * t + __ldg(g + 1)) * t + __ldg(g + 2)) * t + __ldg(g + 3);
  dv = (__ldg(g + 4) * t + __ldg(g + 5)) * t + __ldg(g + 6);
}
// F(rho) and F'(rho) from the normalised records (clamped like spline_eval,
// spline.cpp:79-93): u = (x - x0)/h by one FMA, segment by a round-down add
__device__ __forceinline__ void emb_eval_fast(const KP& P, double x, double& v, double& dv) {
  x = fmin(fmax(x, P.emb.x0), P.emb.xl);
  const double u = fma(x, P.fe.ih, P.fe.c0);
  const double t = __dadd_rd(u, 4503599627370496.0);
  const double s = u - (t - 4503599627370496.0);
  const int i = min(__double2loint(t), P.fe.nseg);
  const double* r = P.fe.rec + 4 * (size_t)i;
  const double2 ab = __ldg(reinterpret_cast<const double2*>(r));
  const double2 cd = __ldg(reinterpret_cast<const double2*>(r) + 1);
  v = fma(fma(fma(ab.x, s, ab.y), s, cd.x), s, cd.y);
  dv = fma(fma(ab.x, 1.5 * s, ab.y), s + s, cd.x) * P.fe.ih;
}

__device__ __forceinline__ double seg_deriv(const Tab& T, double x) {
  if (x < T.x0) x = T.x0;
  if (x > T.xl) x = T.xl;
  int i = (int)((x - T.x0) / T.h);
  i = max(0, min(i, T.nseg - 1));
  const double t = x - (T.x0 + T.h * (double)i);
  const double* g = T.seg + 7 * (size_t)i;
  return (__ldg(g + 4) * t + __ldg(g + 5)) * t + __ldg(g + 6);
}

// EamPotential::density(r).value, potential.cpp:11-17 (guard counted)
__device__ __forceinline__ double pair_rho(const KP& P, double r2) {
  double r = sqrt(r2);
  if (r < P.dens.x0) {
    atomicAdd(&P.st->r_underflow, 1ull);
    r = P.dens.x0;
  }
  return seg_value(P.dens, r);
}

// the force of one pair: fp of forces.cpp:164 and phi of 168
__device__ __forceinline__ void pair_force(const KP& P, double r2, double dfsum, double& fp,
                                           double& phi) {
  const double r = sqrt(r2);
  // EamPotential::pair (potential.cpp:19-31)
  double rp = r;
  if (rp < P.zr.x0) {
    atomicAdd(&P.st->r_underflow, 1ull);
    rp = P.zr.x0;
  } else if (rp > P.cutoff) {
    rp = P.cutoff;
  }
  double z, dz;
  seg_eval(P.zr, rp, z, dz);
  phi = z / rp;
  const double dphi = (dz * rp - z) / (rp * rp);
  // EamPotential::density(r).deriv
  double rd = r;
  if (rd < P.dens.x0) {
    atomicAdd(&P.st->r_underflow, 1ull);
    rd = P.dens.x0;
  }
  const double drho = seg_deriv(P.dens, rd);
  fp = -(dfsum * drho + dphi) / r;
}

__device__ __forceinline__ void report_overlap(const KP& P, unsigned long long key,
                                               unsigned long long ta, unsigned long long tb,
                                               double r2) {
  const int k = atomicAdd(&P.st->n_ovl, 1);
  if (k < kMaxOverlapRecords) {
    P.st->ovl_key[k] = key;
    P.st->ovl_a[k] = ta;
    P.st->ovl_b[k] = tb;
    P.st->ovl_r2[k] = r2;
  }
}

int eam_blocks(const KP& P) { return (int)((P.G.NI + 127) / 128); }

// the reference orientation of a full-list pair (a, j) with j at a negative
// offset: the reference visits it from the partner's side, with the partner
// as driver and an image of `a` when j is a ghost.  Returns d = a - partner
// whose components are the exact negation of the reference's d.
__device__ __forceinline__ void full_orient(const KP& P, const double4& a, long long j,
                                            const double4& p, double& dx, double& dy,
                                            double& dz) {
  const int t = __ldg(&P.tgt[j]);
  if (t == j) {
    dx = xsub(a.x, p.x);
    dy = xsub(a.y, p.y);
    dz = xsub(a.z, p.z);
    return;
  }
  // ghost j = image of source t under shift k: the reference pair is
  // (t, image of a under -k), d_ref = s - (a + (-k) L)
  const long long cell = j >= P.G.NC ? j - P.G.NC : j;
  int cx, cy, cz;
  cell_xyz(cell, P.G, cx, cy, cz);
  const long kx = floor_div(cx - P.G.g, P.G.bx), ky = floor_div(cy - P.G.g, P.G.by),
             kz = floor_div(cz - P.G.g, P.G.bz);
  const double4 s = P.pdf[t];
  const double ix = xadd(a.x, xmul((double)(-kx), P.G.lx));
  const double iy = xadd(a.y, xmul((double)(-ky), P.G.ly));
  const double iz = xadd(a.z, xmul((double)(-kz), P.G.lz));
  dx = -xsub(s.x, ix);
  dy = -xsub(s.y, iy);
  dz = -xsub(s.z, iz);
}

// ------------------------------------------------------------ density pass
template <bool FULL>
__global__ void __launch_bounds__(256) k_density(KP P) {
  if (P.st->err || P.st->halt) return;
  int par;
  long long d;
  if (!map_site(P, par, d)) return;
  const double4 a = P.pdf[d];
  if (a.x >= kVacantTest) {
    if (FULL) P.rho[d] = 0.0;
    return;
  }
  const int n = FULL ? c_full_n[par] : c_half_n[par];
  double acc = 0.0;
  unsigned cand = 0, pairs = 0;
  for (int k = 0; k < n; ++k) {
    const long long j = d + (FULL ? c_full[par][k] : c_half[par][k]);
    const double4 p = ldg4(&P.pdf[j]);
    double dx, dy, dz;
    if (FULL && c_full_flat[par][k] < 0) {
      if (p.x >= kVacantTest) continue;
      full_orient(P, a, j, p, dx, dy, dz);
    } else {
      dx = xsub(a.x, p.x);
      dy = xsub(a.y, p.y);
      dz = xsub(a.z, p.z);
    }
    const double r2 = exact_r2(dx, dy, dz);
    ++cand;
    if (r2 > P.cut2) continue;
    if (r2 < kOverlapR2) {
      const long long rd = ref_of_dev(d, P.G.NC), rj = ref_of_dev(j, P.G.NC);
      report_overlap(P, ((unsigned long long)min(rd, rj) << 12) | (unsigned)k, P.tag[d],
                     P.tag[__ldg(&P.tgt[j])], r2);
      continue;
    }
    ++pairs;
    const double rho = pair_rho(P, r2);
    acc += rho;
    if (!FULL) atomicAdd(&P.rho[__ldg(&P.tgt[j])], rho);
  }
  if (FULL) P.rho[d] = acc;
  else atomicAdd(&P.rho[d], acc);
  if (P.count_pairs) {
    atomicAdd(&P.st->cnt_cand, (unsigned long long)cand);
    atomicAdd(&P.st->cnt_pair, (unsigned long long)pairs);
  }
}

// -------------------------------------------------------------- force pass
template <bool FULL>
__global__ void __launch_bounds__(256) k_force(KP P) {
  zero_pair_tail(P, gridDim.x);
  __shared__ double sh[8];
  double e = 0.0;
  int par;
  long long d;
  const bool live = !P.st->err && !P.st->n_ovl && map_site(P, par, d);
  if (live) {
    const double4 a = P.pdf[d];
    if (a.x < kVacantTest) {
      const int n = FULL ? c_full_n[par] : c_half_n[par];
      double fx = 0.0, fy = 0.0, fz = 0.0;
      const long long S = P.S;
      for (int k = 0; k < n; ++k) {
        const long long j = d + (FULL ? c_full[par][k] : c_half[par][k]);
        const double4 p = ldg4(&P.pdf[j]);
        double dx, dy, dz;
        if (FULL && c_full_flat[par][k] < 0) {
          if (p.x >= kVacantTest) continue;
          full_orient(P, a, j, p, dx, dy, dz);
        } else {
          dx = xsub(a.x, p.x);
          dy = xsub(a.y, p.y);
          dz = xsub(a.z, p.z);
        }
        const double r2 = exact_r2(dx, dy, dz);
        if (r2 > P.cut2) continue;
        if (r2 < kOverlapR2) {
          const long long rd = ref_of_dev(d, P.G.NC), rj = ref_of_dev(j, P.G.NC);
          report_overlap(P, (1ull << 61) | ((unsigned long long)min(rd, rj) << 12) | (unsigned)k,
                         P.tag[d], P.tag[__ldg(&P.tgt[j])], r2);
          continue;
        }
        double fp, phi;
        pair_force(P, r2, a.w + p.w, fp, phi);
        const double gx = dx * fp, gy = dy * fp, gz = dz * fp;
        fx += gx;
        fy += gy;
        fz += gz;
        if (FULL) {
          e += 0.5 * phi;
        } else {
          e += phi;
          const int t = __ldg(&P.tgt[j]);
          atomicAdd(&P.frc[t], -gx);
          atomicAdd(&P.frc[S + t], -gy);
          atomicAdd(&P.frc[2 * S + t], -gz);
        }
      }
      if (FULL) {
        P.frc[d] = fx;
        P.frc[S + d] = fy;
        P.frc[2 * S + d] = fz;
      } else {
        atomicAdd(&P.frc[d], fx);
        atomicAdd(&P.frc[S + d], fy);
        atomicAdd(&P.frc[2 * S + d], fz);
      }
    } else if (FULL) {
      P.frc[d] = 0.0;
      P.frc[P.S + d] = 0.0;
      P.frc[2 * P.S + d] = 0.0;
    }
  }
  const double s = block_sum<256>(e, sh);
  if (threadIdx.x == 0) P.part_pair[blockIdx.x] = s;
}

// ---------------------------------------------------------- embedding pass
// interior sites: dF = F'(rho), E += F(rho) (embed_slots); ghost sites take
// F'(rho of their source) -- the refresh_ghosts copy, computed in place
__device__ void clash_embed_body(const KP& P, int blk, int nblk) {
  if (P.st->err || P.st->n_ovl) return;
  const int n = P.st->n_clash;
  for (int i = blk * blockDim.x + threadIdx.x; i < n; i += nblk * blockDim.x) {
    const int s = P.cl.gf[i] ? P.cl.src[i] : i;
    if (s < 0) continue;  // remote source: dF arrives with the dF halo
    const double r = P.cl.rho[s];
    double v, dv;
    seg_eval(P.emb, r, v, dv);
    if (!P.cl.gf[i]) {
      if (r < P.emb.x0 || r > P.emb.xl) atomicAdd(&P.st->rho_clamp, 1ull);
      P.cl.e_emb[i] = v;
    } else {
      P.cl.e_emb[i] = 0.0;
    }
    P.cl.df[i] = dv;
  }
}

// blocks [0, nsb): all slots, grid-stride, one energy partial per block;
// blocks [nsb, grid): the clash records (fused k_clash_embed)
__global__ void __launch_bounds__(256, 6) k_embed(KP P, int nsb, int literal) {
  pdl_wait();
  pdl_trigger();
  if (P.rev_wait && !rev_wait(P, P.rev_wait)) return;  // the neighbours' density partials
  if (blockIdx.x >= nsb) {
    clash_embed_body(P, blockIdx.x - nsb, gridDim.x - nsb);
    // the records' force accumulators for the force pass (clash_zero fused)
    const int n = P.st->n_clash;
    for (int i = (blockIdx.x - nsb) * blockDim.x + threadIdx.x; i < n;
         i += (gridDim.x - nsb) * blockDim.x) {
      P.cl.fx[i] = 0.0;
      P.cl.fy[i] = 0.0;
      P.cl.fz[i] = 0.0;
      P.cl.e_pair[i] = 0.0;
    }
    return;
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) P.work[1] = 0;  // the force pass's brick queue
  __shared__ double sh[8];
  double e = 0.0;
  const bool ok = !P.st->err && !P.st->n_ovl;
  for (long long d = (long long)blockIdx.x * blockDim.x + threadIdx.x; ok && d < P.S;
       d += (long long)nsb * blockDim.x) {
    // the site's position and owner in one round trip, then the owner's rho
    const double px = P.pdf[d].x;
    const int t = P.tgt[d];
    if (px >= kVacantTest) continue;
    const double r = P.rho[t];
    double v, dv;
    if (literal) seg_eval(P.emb, r, v, dv);
    else emb_eval_fast(P, r, v, dv);
    // owned here: interior site (a z-halo site of a slab rank also has
    // t == d, but its rho is a partial and its dF comes from the owner)
    bool owned = t == d;
    if (owned && P.G.slab) {
      const long cz = site_cz(ref_of_dev(d, P.G.NC), P.G);
      owned = cz >= P.G.g && cz < P.G.g + P.G.bz;
    }
    if (owned) {
      if (r < P.emb.x0 || r > P.emb.xl) atomicAdd(&P.st->rho_clamp, 1ull);
      e += v;
    }
    P.pdf[d].w = dv;
  }
  const double s = block_sum<256>(e, sh);
  if (threadIdx.x == 0) P.part_emb[blockIdx.x] = s;
}
int embed_blocks(const KP& P) { return (int)((P.S + 255) / 256); }
int embed_grid(const KP& P) {
  int sms = 148, dev = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  return std::max(1, std::min(embed_blocks(P), 6 * sms));  // one resident wave (256, 6)
}

__global__ void k_clash_embed(KP P) { clash_embed_body(P, blockIdx.x, gridDim.x); }

// ------------------------------------------------------------ clash pairs
// forces.cpp:185-225, one warp per interior clash record; partner classes:
// own slot, later bucket mates, slot atoms at id + full offsets (incl.
// ghosts -> owner), interior buckets with nid > id (symmetric), ghost
// buckets (one-sided, half energy).  All partner updates are RED adds.
// blk / nblk: this block's index among the blocks sweeping the records
// (the standalone kernel, or the extra blocks of a fused pass)
template <int MODE>  // 0 density, 1 force
__device__ void clash_body(const KP& P, int blk, int nblk) {
  if (P.st->err || P.st->halt) return;
  if (MODE == 1 && P.st->n_ovl) return;
  const int n = P.st->n_clash;
  if (n == 0) return;
  const int lane = threadIdx.x & 31;
  const int gw = (blk * blockDim.x + threadIdx.x) >> 5;
  const int nw = (nblk * blockDim.x) >> 5;
  const long long S = P.S;
  for (int i = gw; i < n; i += nw) {
    if (P.cl.gf[i]) continue;
    const long long id = P.cl.key[i];
    const int par = (int)(id & 1);
    const long long dow = dev_of_ref(id, P.G.NC);
    const double ax = P.cl.px[i], ay = P.cl.py[i], az = P.cl.pz[i];
    const double adf = MODE ? P.cl.df[i] : 0.0;
    double acc = 0.0, fx = 0.0, fy = 0.0, fz = 0.0, e = 0.0;
    // partner: (px,py,pz,pdf), symmetric target: kind 0 slot idx, 1 clash idx, -1 none
    auto visit = [&](double px, double py, double pz, double pdf, int kind, long long tidx,
                     unsigned long long ptag, unsigned long long seq) {
      const double dx = xsub(ax, px), dy = xsub(ay, py), dz = xsub(az, pz);
      const double r2 = exact_r2(dx, dy, dz);
      if (r2 > P.cut2) return;
      if (r2 < kOverlapR2) {
        report_overlap(P, (1ull << 62) | (MODE ? (1ull << 61) : 0ull) |
                              ((unsigned long long)i << 24) | seq,
                       P.cl.tag[i], ptag, r2);
        return;
      }
      if (MODE == 0) {
        const double rho = pair_rho(P, r2);
        acc += rho;
        if (kind == 0) atomicAdd(acc_ptr<-1>(P, tidx), rho);
        else if (kind == 1) atomicAdd(&P.cl.rho[tidx], rho);
      } else {
        double fp, phi;
        pair_force(P, r2, adf + pdf, fp, phi);
        const double gx = dx * fp, gy = dy * fp, gz = dz * fp;
        fx += gx;
        fy += gy;
        fz += gz;
        if (kind == 0) {
          atomicAdd(acc_ptr<0>(P, tidx), -gx);
          atomicAdd(acc_ptr<1>(P, tidx), -gy);
          atomicAdd(acc_ptr<2>(P, tidx), -gz);
          e += phi;
        } else if (kind == 1) {
          atomicAdd(&P.cl.fx[tidx], -gx);
          atomicAdd(&P.cl.fy[tidx], -gy);
          atomicAdd(&P.cl.fz[tidx], -gz);
          e += phi;
        } else {
          e += 0.5 * phi;
        }
      }
    };
    if (lane == 0) {  // own slot
      const double4 o = P.pdf[dow];
      if (o.x < kVacantTest) visit(o.x, o.y, o.z, o.w, 0, dow, P.tag[dow], 0);
    }
    for (int j = i + 1 + lane; j < n && P.cl.key[j] == id; j += 32)  // later mates
      visit(P.cl.px[j], P.cl.py[j], P.cl.pz[j], MODE ? P.cl.df[j] : 0.0, 1, j, P.cl.tag[j],
            1 + (j - i));
    const int nf = c_full_n[par];
    for (int k = lane; k < nf; k += 32) {
      const long long nd = dow + c_full[par][k];
      const double4 s = P.pdf[nd];
      if (s.x < kVacantTest)
        visit(s.x, s.y, s.z, s.w, 0, P.tgt[nd], P.tag[P.tgt[nd]], 4096 + 64 * k);
      const int h = P.head[nd];
      if (h < 0) continue;
      const long long nid = id + c_full_flat[par][k];
      const bool ghost = P.cl.gf[h] != 0;
      if (!ghost && nid <= id) continue;
      for (int j = h; j < n && P.cl.key[j] == nid; ++j)
        visit(P.cl.px[j], P.cl.py[j], P.cl.pz[j], MODE ? P.cl.df[j] : 0.0, ghost ? -1 : 1, j,
              P.cl.tag[j], 4096 + 64 * k + 1 + (j - h));
    }
    // warp reduction of the driver's own sums
    for (int o = 16; o > 0; o >>= 1) {
      acc += __shfl_xor_sync(0xffffffffu, acc, o);
      fx += __shfl_xor_sync(0xffffffffu, fx, o);
      fy += __shfl_xor_sync(0xffffffffu, fy, o);
      fz += __shfl_xor_sync(0xffffffffu, fz, o);
      e += __shfl_xor_sync(0xffffffffu, e, o);
    }
    if (lane == 0) {
      if (MODE == 0) {
        atomicAdd(&P.cl.rho[i], acc);
      } else {
        atomicAdd(&P.cl.fx[i], fx);
        atomicAdd(&P.cl.fy[i], fy);
        atomicAdd(&P.cl.fz[i], fz);
        P.cl.e_pair[i] = e;
      }
    }
  }
}
template <int MODE>
__global__ void __launch_bounds__(256) k_clash(KP P) {
  clash_body<MODE>(P, blockIdx.x, gridDim.x);
}
template __device__ void clash_body<0>(const KP&, int, int);
template __device__ void clash_body<1>(const KP&, int, int);

#include "stencil_fast.cuh"

// ------------------------------------------------------------- launchers
// mode: 0 fast half list (Newton-3), 1 fast full list, 2 reference-literal half list
// return true when the clash-record pass ran inside the same kernel
bool launch_density(const KP& P, int mode, cudaStream_t s) {
  if (mode == 2) k_density<false><<<eam_blocks(P), 256, 0, s>>>(P);
  else return launch_density_fast(P, mode, fast_grid(P, false, mode), s);
  return false;
}
bool launch_force(const KP& P, int mode, cudaStream_t s) {
  if (mode == 2) k_force<false><<<eam_blocks(P), 256, 0, s>>>(P);
  else return launch_force_fast(P, mode, fast_grid(P, true, mode), s);
  return false;
}
// partials any force kernel may write (per warp / per block); the finalize
// sums this many (the rest of part_pair is zeroed before every force pass)
int pair_partials(const KP& P, int mode) {
  (void)mode;
  int sms = 148, dev = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  // one partial per CTA: the literal pass (eam_blocks), the 1024-thread
  // mask-replay pass (one CTA per SM + clash blocks), the 128-thread pass
  int n = std::max(eam_blocks(P), sms + 8);
  for (int m = 0; m < 2; ++m) n = std::max(n, fast_grid(P, true, m));
  return std::min(n, P.n_part);
}
int force_partials(const KP& P, int mode) {
  if (mode == 2) return eam_blocks(P);
  if (!P.use_mask) return fast_grid(P, true, mode);
  int sms = 148, dev = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  return std::max(1, std::min(sms, unit_count(P.G)));  // launch_force_lean
}
void launch_embed(const KP& P, cudaStream_t s, bool literal) {
  const int nsb = embed_grid(P);
  launch_pdl(k_embed, nsb + 16, 256, 0, s, P, nsb, literal ? 1 : 0);
}
void launch_clash_density(const KP& P, cudaStream_t s) { k_clash<0><<<16, 256, 0, s>>>(P); }
void launch_clash_force(const KP& P, cudaStream_t s) { k_clash<1><<<16, 256, 0, s>>>(P); }

}  // namespace cbx
