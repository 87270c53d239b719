// slab.cu -- z-slab domain decomposition: the pack /
// unpack kernels of the per-step exchanges between neighbouring ranks.
//
// A rank owns global interior z planes [zoff, zoff + bz) and keeps g halo
// planes below and above.  Positions, hashes and keys stay in the global
// frame; halo planes are contiguous id ranges of every per-site array
// (ids are z-major, lattice.cpp:10-15), so slot data moves without
// packing.  Exchanges per step (the analogue of fill_ghosts for z and of
// fold_rho / refresh_ghosts / fold_force, store.cpp:120-195,
// forces.cpp:290-309, across ranks):
//   MIGRANTS  atoms whose new hash lies in a neighbour's slab (pass 1 / 2 of
//             update_hash with their walk position preserved)
//   POS       boundary planes -> neighbour's halo (+ boundary clash records)
//   RHO       halo density partials -> owner (reverse, added via tgt[])
//   DF        boundary planes' dF -> neighbour's halo
//   FRC       halo force partials -> owner (reverse)
#include "cbx_device.cuh"

namespace cbx {

struct MigRec {  // 88 bytes
  double px, py, pz, vx, vy, vz;
  unsigned long long tag;
  long long key, walk, sub, cls;
};
struct RemRec {  // 72 bytes
  long long key;
  double px, py, pz, vx, vy, vz, df;
  unsigned long long tag;
};

__device__ __forceinline__ long long plane_ids(const Geo& G) { return 2ll * G.tx * G.ty; }

// ------------------------------------------------------------- migrants
__global__ void k_pack_migrants(KP P, int dir, unsigned char* buf, long long cap) {
  const int n = min(P.st->n_out, P.cap_mov);
  long long* cnt = reinterpret_cast<long long*>(buf);
  MigRec* rec = reinterpret_cast<MigRec*>(buf + 16);
  __shared__ int s_n;
  if (threadIdx.x == 0) s_n = 0;
  __syncthreads();
  const long long pid = plane_ids(P.G);
  for (int i = threadIdx.x; i < n; i += blockDim.x) {
    if (P.out.dir[i] != dir) continue;
    const int k = atomicAdd(&s_n, 1);
    if (16 + (long long)(k + 1) * sizeof(MigRec) > cap) {
      set_error(P.st, CBX_RUNTIME);
      continue;
    }
    MigRec r;
    r.px = P.out.px[i];
    r.py = P.out.py[i];
    r.pz = P.out.pz[i];
    r.vx = P.out.vx[i];
    r.vy = P.out.vy[i];
    r.vz = P.out.vz[i];
    r.tag = P.out.tag[i];
    r.key = P.out.key[i] + P.G.zoff * pid;  // global ids
    r.walk = P.out.walk[i] + P.G.zoff * pid;
    r.cls = P.out.cls[i];
    r.sub = r.cls == 1 ? P.out.sub[i] + P.G.zoff * pid : P.out.sub[i];
    rec[k] = r;
  }
  __syncthreads();
  if (threadIdx.x == 0)
    cnt[0] = min((long long)s_n, (cap - 16) / (long long)sizeof(MigRec));  // records written
}

__global__ void k_unpack_migrants(KP P, const unsigned char* buf, long long gshift) {
  const long long n = reinterpret_cast<const long long*>(buf)[0];
  const MigRec* rec = reinterpret_cast<const MigRec*>(buf + 16);
  const long long pid = plane_ids(P.G);
  const long long off = -P.G.zoff * pid;  // global -> local ids (no periodic shift:
  (void)gshift;                           // the sender wrapped the position)
  for (long long i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    const int m = atomicAdd(&P.st->n_mov, 1);
    if (m >= P.cap_mov) {
      set_error(P.st, CBX_RUNTIME);
      return;
    }
    const MigRec r = rec[i];
    P.mv.key[m] = r.key + off;
    P.mv.walk[m] = r.walk + off;
    P.mv.cls[m] = (int)r.cls;
    P.mv.sub[m] = r.cls == 1 ? r.sub + off : r.sub;
    P.mv.px[m] = r.px;
    P.mv.py[m] = r.py;
    P.mv.pz[m] = r.pz;  // already wrapped into the global box by the sender
    P.mv.vx[m] = r.vx;
    P.mv.vy[m] = r.vy;
    P.mv.vz[m] = r.vz;
    P.mv.tag[m] = r.tag;
  }
}

// ------------------------------------------------------------ slot planes
// kind: 1 POS (pdf + tag, boundary planes -> halo), 3 DF (pdf.w),
//       2 RHO, 4 FRC (halo -> owner's boundary planes)
__device__ __forceinline__ int plane_lo(const Geo& G, int kind, int dir) {
  const bool forward = kind == 1 || kind == 3;
  if (forward) return dir < 0 ? G.g : G.bz;          // my boundary interior planes
  return dir < 0 ? 0 : G.bz + G.g;                    // my halo planes
}
__device__ __forceinline__ int plane_lo_recv(const Geo& G, int kind, int from) {
  const bool forward = kind == 1 || kind == 3;
  if (forward) return from < 0 ? 0 : G.bz + G.g;     // into my halo
  return from < 0 ? G.g : G.bz;                       // into my boundary planes
}

__global__ void k_pack_planes(KP P, int kind, int dir, unsigned char* buf) {
  const Geo& G = P.G;
  const long long n = (long long)G.g * G.txy;  // sites per sublattice
  const long long base = (long long)plane_lo(G, kind, dir) * G.txy;
  for (long long q = blockIdx.x * blockDim.x + threadIdx.x; q < 2 * n;
       q += gridDim.x * blockDim.x) {
    const int par = q >= n;
    const long long d = par * G.NC + base + (q - par * n);
    if (kind == 1) {
      reinterpret_cast<double4*>(buf)[q] = P.pdf[d];
      reinterpret_cast<unsigned long long*>(buf + 2 * n * sizeof(double4))[q] = P.tag[d];
    } else if (kind == 3) {
      reinterpret_cast<double*>(buf)[q] = P.pdf[d].w;
    } else if (kind == 2) {
      reinterpret_cast<double*>(buf)[q] = P.rho[d];
    } else {
      for (int a = 0; a < 3; ++a) reinterpret_cast<double*>(buf)[a * 2 * n + q] = P.frc[a * P.S + d];
    }
  }
}

__global__ void k_unpack_planes(KP P, int kind, int from, const unsigned char* buf,
                                long long gshift) {
  const Geo& G = P.G;
  const long long n = (long long)G.g * G.txy;
  const long long base = (long long)plane_lo_recv(G, kind, from) * G.txy;
  const double dz = xmul((double)gshift, G.glz);
  for (long long q = blockIdx.x * blockDim.x + threadIdx.x; q < 2 * n;
       q += gridDim.x * blockDim.x) {
    const int par = q >= n;
    const long long d = par * G.NC + base + (q - par * n);
    if (kind == 1) {
      double4 p = reinterpret_cast<const double4*>(buf)[q];
      if (p.x < kVacantTest) {
        p.z = xadd(p.z, dz);  // periodic image across the global z boundary
        P.uf[d] = make_float4((float)p.x, (float)p.y, (float)p.z, __int_as_float(-1));
      } else {
        P.uf[d] = make_float4(kVacantF, kVacantF, kVacantF, __int_as_float(-1));
      }
      P.pdf[d] = p;
      P.tag[d] = reinterpret_cast<const unsigned long long*>(buf + 2 * n * sizeof(double4))[q];
    } else if (kind == 3) {
      P.pdf[d].w = reinterpret_cast<const double*>(buf)[q];
    } else if (kind == 2) {
      atomicAdd(&P.rho[P.tgt[d]], reinterpret_cast<const double*>(buf)[q]);
    } else {
      const int t = P.tgt[d];
      for (int a = 0; a < 3; ++a)
        atomicAdd(&P.frc[a * P.S + t], reinterpret_cast<const double*>(buf)[a * 2 * n + q]);
    }
  }
}

// boundary clash records (interior, gf 0) of the planes sent with POS / DF,
// in list order (so DF matches POS record by record)
__global__ void k_pack_clash(KP P, int kind, int dir, unsigned char* buf, long long cap) {
  const Geo& G = P.G;
  const int lo = plane_lo(G, kind, dir), hi = lo + G.g;
  const int n = P.st->n_clash;
  long long* cnt = reinterpret_cast<long long*>(buf);
  RemRec* rec = reinterpret_cast<RemRec*>(buf + 16);
  const long long pid = plane_ids(G);
  if (threadIdx.x == 0) {  // one thread: list order
    long long k = 0;
    for (int i = 0; i < n; ++i) {
      if (P.cl.gf[i]) continue;
      const long cz = site_cz(P.cl.key[i], G);
      if (cz < lo || cz >= hi) continue;
      if (16 + (k + 1) * (long long)sizeof(RemRec) > cap) {
        set_error(P.st, CBX_RUNTIME);
        break;
      }
      RemRec r;
      r.key = P.cl.key[i] + G.zoff * pid;
      r.px = P.cl.px[i];
      r.py = P.cl.py[i];
      r.pz = P.cl.pz[i];
      r.vx = P.cl.vx[i];
      r.vy = P.cl.vy[i];
      r.vz = P.cl.vz[i];
      r.df = P.cl.df[i];
      r.tag = P.cl.tag[i];
      rec[k++] = r;
    }
    cnt[0] = k;
  }
}

__global__ void k_unpack_clash(KP P, int kind, const unsigned char* buf, long long gshift,
                               int* base_out) {
  const long long n = reinterpret_cast<const long long*>(buf)[0];
  const RemRec* rec = reinterpret_cast<const RemRec*>(buf + 16);
  if (threadIdx.x != 0) return;
  const long long pid = plane_ids(P.G);
  if (kind == 1) {  // POS: append as remote sources
    const int base = P.st->n_remote;
    *base_out = base;
    for (long long i = 0; i < n; ++i) {
      const int m = base + (int)i;
      if (m >= P.cap_rem) {
        set_error(P.st, CBX_RUNTIME);
        return;
      }
      const RemRec r = rec[i];
      P.rem.key[m] = r.key + gshift * (long long)P.G.gbz * pid - P.G.zoff * pid;
      P.rem.px[m] = r.px;
      P.rem.py[m] = r.py;
      P.rem.pz[m] = xadd(r.pz, xmul((double)gshift, P.G.glz));
      P.rem.vx[m] = r.vx;
      P.rem.vy[m] = r.vy;
      P.rem.vz[m] = r.vz;
      P.rem.df[m] = r.df;
      P.rem.tag[m] = r.tag;
    }
    P.st->n_remote = base + (int)n;
  } else {  // DF: refresh the remote sources' dF, same order as POS
    const int base = *base_out;
    for (long long i = 0; i < n; ++i) P.rem.df[base + i] = rec[i].df;
  }
}

// dF of ghost clash records derived from remote sources
__global__ void k_remote_df(KP P) {
  const int n = P.st->n_clash;
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x)
    if (P.cl.gf[i] && P.cl.src[i] <= -2) P.cl.df[i] = P.rem.df[-P.cl.src[i] - 2];
}

// ---------------------------------------------------------------- launchers
long long slab_plane_bytes(const KP& P, int kind) {
  const long long n = 2ll * P.G.g * P.G.txy;
  switch (kind) {
    case 1: return n * (sizeof(double4) + 8);
    case 2: case 3: return n * 8;
    default: return n * 24;
  }
}
// fixed message size of the in-graph NCCL exchange (sizes cannot depend on
// device-side counts inside a captured step): the planes plus room for
// kMsgRecords records; more sets CBX_RUNTIME on the sender
long long slab_msg_bytes(const KP& P, int kind) {
  const long long R = std::min<long long>(P.cap_rem, kMsgRecords);
  const long long M = std::min<long long>(P.cap_mov, kMsgRecords);
  long long b;
  if (kind == 0) {
    b = 16 + M * (long long)sizeof(MigRec);
  } else {
    b = slab_plane_bytes(P, kind);
    if (kind == 1 || kind == 3) b += 16 + R * (long long)sizeof(RemRec);
  }
  return (b + 255) / 256 * 256;
}

long long slab_buffer_bytes(const KP& P, int kind) {
  if (kind == 0) return 16 + (long long)P.cap_mov * sizeof(MigRec);
  long long b = slab_plane_bytes(P, kind);
  if (kind == 1 || kind == 3) b += 16 + (long long)P.cap_rem * sizeof(RemRec);
  return (b + 255) / 256 * 256;
}

void launch_pack(const KP& P, int kind, int dir, unsigned char* buf, long long cap,
                 cudaStream_t s) {
  if (kind == 0) {
    k_pack_migrants<<<1, 1024, 0, s>>>(P, dir, buf, cap);
    return;
  }
  const long long pb = slab_plane_bytes(P, kind);
  const long long n = 2ll * P.G.g * P.G.txy;
  k_pack_planes<<<(int)std::min<long long>((n + 255) / 256, 4096), 256, 0, s>>>(P, kind, dir, buf);
  if (kind == 1 || kind == 3) k_pack_clash<<<1, 32, 0, s>>>(P, kind, dir, buf + pb, cap - pb);
}

void launch_unpack(const KP& P, int kind, int from, const unsigned char* buf, long long gshift,
                   int* rem_base, cudaStream_t s) {
  if (kind == 0) {
    k_unpack_migrants<<<8, 256, 0, s>>>(P, buf, gshift);
    return;
  }
  const long long pb = slab_plane_bytes(P, kind);
  const long long n = 2ll * P.G.g * P.G.txy;
  k_unpack_planes<<<(int)std::min<long long>((n + 255) / 256, 4096), 256, 0, s>>>(P, kind, from,
                                                                                buf, gshift);
  if (kind == 1 || kind == 3) k_unpack_clash<<<1, 32, 0, s>>>(P, kind, buf + pb, gshift, rem_base);
}

void launch_remote_df(const KP& P, cudaStream_t s) { k_remote_df<<<8, 256, 0, s>>>(P); }

// ------------------------------------------------- step-state all-reduce
// red = {pair, embedding, kinetic, max_speed}: the local sums go in, the
// all-reduced values (sum, sum, sum, max) come back into the StepState
__global__ void k_slab_red_in(KP P, double* red) {
  if (threadIdx.x != 0) return;
  const DevStatus* st = P.st;
  red[0] = st->pair;
  red[1] = st->embedding;
  red[2] = st->kinetic;
  red[3] = st->max_speed;
}
__global__ void k_slab_red_out(KP P, const double* red, int energies, int kinetic) {
  if (threadIdx.x != 0) return;
  DevStatus* st = P.st;
  if (energies) {
    st->pair = red[0];
    st->embedding = red[1];
  }
  if (kinetic) {
    st->kinetic = red[2];
    st->max_speed = red[3];
    if (st->adaptive) {  // adaptive_dt on the global max speed, sim.cpp:94-98
      double dt = st->dt_max;
      if (st->max_speed > 0.0) dt = fmin(dt, xdiv(st->max_disp, st->max_speed));
      st->dt_next = fmax(dt, 1e-7);
    }
  }
}
void launch_slab_red_in(const KP& P, double* red, cudaStream_t s) {
  k_slab_red_in<<<1, 32, 0, s>>>(P, red);
}
void launch_slab_red_out(const KP& P, const double* red, int energies, int kinetic,
                         cudaStream_t s) {
  k_slab_red_out<<<1, 32, 0, s>>>(P, red, energies, kinetic);
}

}  // namespace cbx
