// slab.cu -- z-slab domain decomposition: the pack /
// unpack work of the per-step exchanges between neighbouring ranks, as
// staging kernels (host-driven and NCCL transports) and as fused peer-memory
// kernels (P2P transport: the sender stores straight into the receiver's
// buffer over NVLink and raises a flag; the receiver waits on the flag).
//
// A rank owns global interior z planes [zoff, zoff + bz) and keeps g halo
// planes below and above.  Positions, hashes and keys stay in the global
// frame; halo planes are contiguous id ranges of every per-site array
// (ids are z-major, lattice.cpp:10-15), so slot data moves without
// gathering.  Exchanges per step (the analogue of fill_ghosts for z and of
// fold_rho / refresh_ghosts / fold_force, store.cpp:120-195,
// forces.cpp:290-309, across ranks):
//   MIGRANTS  atoms whose new hash lies in a neighbour's slab (pass 1 / 2 of
//             update_hash with their walk position preserved)
//   POS       boundary planes -> neighbour's halo (+ boundary clash records)
//   RHO       halo density partials -> owner (reverse, added via tgt[])
//   DF        boundary planes' dF -> neighbour's halo
//   FRC       halo force partials -> owner (reverse)
#include <algorithm>
#include <cstdlib>

#include "cbx_device.cuh"
#include "p2p.cuh"

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

// message buffers are read once, through L2 (the P2P sender writes them
// from another GPU)
__device__ __forceinline__ double ldcg(const double* p) { return __ldcg(p); }
__device__ __forceinline__ long long ldcg(const long long* p) { return __ldcg(p); }
__device__ __forceinline__ unsigned long long ldcg(const unsigned long long* p) {
  return (unsigned long long)__ldcg(reinterpret_cast<const long long*>(p));
}
__device__ __forceinline__ double4 ldcg(const double4* p) {
  const double2 a = __ldcg(reinterpret_cast<const double2*>(p));
  const double2 b = __ldcg(reinterpret_cast<const double2*>(p) + 1);
  return make_double4(a.x, a.y, b.x, b.y);
}
__device__ __forceinline__ MigRec ldcg_mig(const MigRec* r) {
  MigRec m;
  const double* s = reinterpret_cast<const double*>(r);
  double* d = reinterpret_cast<double*>(&m);
#pragma unroll
  for (int i = 0; i < 11; ++i) d[i] = __ldcg(s + i);
  return m;
}
__device__ __forceinline__ RemRec ldcg_rem(const RemRec* r) {
  RemRec m;
  const double* s = reinterpret_cast<const double*>(r);
  double* d = reinterpret_cast<double*>(&m);
#pragma unroll
  for (int i = 0; i < 9; ++i) d[i] = __ldcg(s + i);
  return m;
}

// ------------------------------------------------------------- migrants
// one block: the outbound records of direction `dir` (list order is free:
// rehash sorts movers by their keys)
__device__ void pack_migrants_block(const KP& P, int dir, unsigned char* buf, long long cap) {
  const int n = min(P.st->n_out, P.cap_mov);
  long long* cnt = reinterpret_cast<long long*>(buf);
  MigRec* rec = reinterpret_cast<MigRec*>(buf + 16);
  __shared__ int s_n;
  if (threadIdx.x == 0) s_n = 0;
  __syncthreads();
  const long long pid = plane_ids(P.G);
  const long long room = (cap - 16) / (long long)sizeof(MigRec);
  for (int i = threadIdx.x; i < n; i += blockDim.x) {
    if (P.out.dir[i] != dir) continue;
    const int k = atomicAdd(&s_n, 1);
    if (k >= room) {
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
  if (threadIdx.x == 0) cnt[0] = min((long long)s_n, room);
}

__device__ void unpack_migrants(const KP& P, const unsigned char* buf, long long i0,
                                long long stride) {
  const long long n = ldcg(reinterpret_cast<const long long*>(buf));
  const MigRec* rec = reinterpret_cast<const MigRec*>(buf + 16);
  const long long off = -P.G.zoff * plane_ids(P.G);  // global -> local ids
  for (long long i = i0; i < n; i += stride) {
    const int m = atomicAdd(&P.st->n_mov, 1);
    if (m >= P.cap_mov) {
      set_error(P.st, CBX_RUNTIME);
      return;
    }
    const MigRec r = ldcg_mig(rec + i);
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

__global__ void k_pack_migrants(KP P, int dir, unsigned char* buf, long long cap) {
  pack_migrants_block(P, dir, buf, cap);
}
__global__ void k_unpack_migrants(KP P, const unsigned char* buf) {
  unpack_migrants(P, buf, blockIdx.x * blockDim.x + threadIdx.x, gridDim.x * blockDim.x);
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

__device__ __forceinline__ void pack_plane_site(const KP& P, int kind, int dir,
                                                unsigned char* buf, long long q) {
  const Geo& G = P.G;
  const long long n = (long long)G.g * G.txy;  // sites per sublattice
  const int par = q >= n;
  const long long d = par * G.NC + (long long)plane_lo(G, kind, dir) * G.txy + (q - par * n);
  if (kind == 1) {
    reinterpret_cast<double4*>(buf)[q] = P.pdf[d];
    reinterpret_cast<unsigned long long*>(buf + 2 * n * sizeof(double4))[q] = P.tag[d];
  } else if (kind == 3) {
    reinterpret_cast<double*>(buf)[q] = P.pdf[d].w;
  } else if (kind == 2) {
    reinterpret_cast<double*>(buf)[q] = P.rho[d];
  } else {
    for (int a = 0; a < 3; ++a)
      reinterpret_cast<double*>(buf)[a * 2 * n + q] = P.frc[a * P.S + d];
  }
}

__device__ __forceinline__ void unpack_plane_site(const KP& P, int kind, int from,
                                                  const unsigned char* buf, double dz,
                                                  long long q) {
  const Geo& G = P.G;
  const long long n = (long long)G.g * G.txy;
  const int par = q >= n;
  const long long d =
      par * G.NC + (long long)plane_lo_recv(G, kind, from) * G.txy + (q - par * n);
  if (kind == 1) {
    // a fresh halo site: its rho / force partials of this step start at 0
    P.rho[d] = 0.0;
    P.frc[d] = 0.0;
    P.frc[P.S + d] = 0.0;
    P.frc[2 * P.S + d] = 0.0;
    double4 p = ldcg(reinterpret_cast<const double4*>(buf) + q);
    const int t = P.tgt[d];
    const float w = __int_as_float(t == d ? -1 : t);  // owner column (x/y image) or self
    if (p.x < kVacantTest) {
      p.z = xadd(p.z, dz);  // periodic image across the global z boundary
      P.uf[d] = make_float4((float)p.x, (float)p.y, (float)p.z, w);
    } else {
      P.uf[d] = make_float4(kVacantF, kVacantF, kVacantF, w);
    }
    P.pdf[d] = p;
    P.tag[d] = ldcg(reinterpret_cast<const unsigned long long*>(buf + 2 * n * sizeof(double4)) + q);
  } else if (kind == 3) {
    P.pdf[d].w = ldcg(reinterpret_cast<const double*>(buf) + q);
  } else if (kind == 2) {
    atomicAdd(&P.rho[P.tgt[d]], ldcg(reinterpret_cast<const double*>(buf) + q));
  } else {
    const int t = P.tgt[d];
    for (int a = 0; a < 3; ++a)
      atomicAdd(&P.frc[a * P.S + t], ldcg(reinterpret_cast<const double*>(buf) + a * 2 * n + q));
  }
}

__global__ void k_pack_planes(KP P, int kind, int dir, unsigned char* buf) {
  const long long n2 = 2ll * P.G.g * P.G.txy;
  for (long long q = blockIdx.x * blockDim.x + threadIdx.x; q < n2; q += gridDim.x * blockDim.x)
    pack_plane_site(P, kind, dir, buf, q);
}

__global__ void k_unpack_planes(KP P, int kind, int from, const unsigned char* buf,
                                long long gshift) {
  const long long n2 = 2ll * P.G.g * P.G.txy;
  const double dz = xmul((double)gshift, P.G.glz);
  for (long long q = blockIdx.x * blockDim.x + threadIdx.x; q < n2; q += gridDim.x * blockDim.x)
    unpack_plane_site(P, kind, from, buf, dz, q);
}

// boundary clash records (interior, gf 0) of the planes sent with POS / DF,
// in list order (so DF matches POS record by record); one thread
__device__ void pack_clash_thread(const KP& P, int kind, int dir, unsigned char* buf,
                                  long long cap) {
  const Geo& G = P.G;
  const int lo = plane_lo(G, kind, dir), hi = lo + G.g;
  const int n = P.st->n_clash;
  long long* cnt = reinterpret_cast<long long*>(buf);
  RemRec* rec = reinterpret_cast<RemRec*>(buf + 16);
  const long long pid = plane_ids(G);
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

__device__ void unpack_clash_thread(const KP& P, int kind, const unsigned char* buf,
                                    long long gshift, int* base_out) {
  const long long n = ldcg(reinterpret_cast<const long long*>(buf));
  const RemRec* rec = reinterpret_cast<const RemRec*>(buf + 16);
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
      const RemRec r = ldcg_rem(rec + i);
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
    for (long long i = 0; i < n; ++i) P.rem.df[base + i] = ldcg(&rec[i].df);
  }
}

__global__ void k_pack_clash(KP P, int kind, int dir, unsigned char* buf, long long cap) {
  if (threadIdx.x == 0) pack_clash_thread(P, kind, dir, buf, cap);
}
__global__ void k_unpack_clash(KP P, int kind, const unsigned char* buf, long long gshift,
                               int* base_out) {
  if (threadIdx.x == 0) unpack_clash_thread(P, kind, buf, gshift, base_out);
}

// dF of ghost clash records derived from remote sources
__global__ void k_remote_df(KP P) {
  const int n = P.st->n_clash;
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x)
    if (P.cl.gf[i] && P.cl.src[i] <= -2) P.cl.df[i] = P.rem.df[-P.cl.src[i] - 2];
}

// ------------------------------------------------------ P2P (peer memory)
// both directions of one exchange, stored into the neighbours' buffers
__global__ void __launch_bounds__(256) k_p2p_send(KP P, P2PLinks L, int kind) {
  unsigned char* dn = L.dst[kind][0];  // my "down" packet: the rank below's from-above buffer
  unsigned char* up = L.dst[kind][1];
  if (kind == 0) {
    if (blockIdx.x == 0) pack_migrants_block(P, -1, dn, L.msg[0]);
    else if (blockIdx.x == 1) pack_migrants_block(P, +1, up, L.msg[0]);
  } else {
    const long long n2 = 2ll * P.G.g * P.G.txy;
    for (long long q = blockIdx.x * blockDim.x + threadIdx.x; q < 2 * n2;
         q += gridDim.x * blockDim.x) {
      const bool hi = q >= n2;
      pack_plane_site(P, kind, hi ? 1 : -1, hi ? up : dn, hi ? q - n2 : q);
    }
    if ((kind == 1 || kind == 3) && threadIdx.x == 0 && blockIdx.x < 2) {
      const long long pb = L.plane_bytes[kind];
      unsigned char* b = blockIdx.x == 0 ? dn : up;
      pack_clash_thread(P, kind, blockIdx.x == 0 ? -1 : 1, b + pb, L.msg[kind] - pb);
    }
  }
  signal_peers(L, kind);
}

// one exchange in one kernel: pack into the neighbours' memory, raise the
// flags (last block), wait for the neighbours' packets, unpack.  The grid is
// capped at the co-resident block count (the waiting blocks must not keep
// blocks of the same launch from running their pack).
__global__ void __launch_bounds__(256) k_p2p_xchg(KP P, P2PLinks L, int kind, long long gs_lo,
                                                  long long gs_hi, int* rem_base) {
  unsigned char* dn = L.dst[kind][0];
  unsigned char* up = L.dst[kind][1];
  if (kind == 0) {
    if (blockIdx.x == 0) pack_migrants_block(P, -1, dn, L.msg[0]);
    else if (blockIdx.x == 1) pack_migrants_block(P, +1, up, L.msg[0]);
  } else {
    const long long n2 = 2ll * P.G.g * P.G.txy;
    for (long long q = blockIdx.x * blockDim.x + threadIdx.x; q < 2 * n2;
         q += gridDim.x * blockDim.x) {
      const bool hi = q >= n2;
      pack_plane_site(P, kind, hi ? 1 : -1, hi ? up : dn, hi ? q - n2 : q);
    }
    if ((kind == 1 || kind == 3) && threadIdx.x == 0 && blockIdx.x < 2) {
      const long long pb = L.plane_bytes[kind];
      unsigned char* b = blockIdx.x == 0 ? dn : up;
      pack_clash_thread(P, kind, blockIdx.x == 0 ? -1 : 1, b + pb, L.msg[kind] - pb);
    }
  }
  // arrival + flags (signal_peers without the early return)
  __shared__ unsigned long long s_epoch;
  __syncthreads();
  if (threadIdx.x == 0) {
    // read the epoch before arriving: the last block bumps it only after
    // every block's arrival, so all blocks see the same value
    const unsigned long long e0 = *(volatile unsigned long long*)&L.epoch[kind];
    __threadfence();
    const unsigned t = atomicAdd(&L.done[kind], 1u);
    if (t == gridDim.x - 1) {
      __threadfence();
      L.done[kind] = 0;
      L.epoch[kind] = e0 + 1;
      __threadfence_system();
      st_relaxed_sys(L.flag_dst[kind][0], e0 + 1);
      st_relaxed_sys(L.flag_dst[kind][1], e0 + 1);
    }
    s_epoch = e0 + 1;
  }
  __syncthreads();
  const unsigned long long* fl[2] = {L.flag_src[kind][0], L.flag_src[kind][1]};
  if (!wait_flags(P, fl, 2, s_epoch)) return;
  const unsigned char* lo = L.src[kind][0];
  const unsigned char* hi = L.src[kind][1];
  if (kind == 0) {
    const long long i0 = blockIdx.x * blockDim.x + threadIdx.x, st = gridDim.x * blockDim.x;
    unpack_migrants(P, lo, i0, st);
    unpack_migrants(P, hi, i0, st);
    return;
  }
  const long long n2 = 2ll * P.G.g * P.G.txy;
  const double dz_lo = xmul((double)gs_lo, P.G.glz), dz_hi = xmul((double)gs_hi, P.G.glz);
  for (long long q = blockIdx.x * blockDim.x + threadIdx.x; q < 2 * n2;
       q += gridDim.x * blockDim.x) {
    const bool h = q >= n2;
    unpack_plane_site(P, kind, h ? 1 : -1, h ? hi : lo, h ? dz_hi : dz_lo, h ? q - n2 : q);
  }
  if ((kind == 1 || kind == 3) && blockIdx.x == 0 && threadIdx.x == 0) {
    const long long pb = L.plane_bytes[kind];
    unpack_clash_thread(P, kind, lo + pb, gs_lo, rem_base + 0);
    unpack_clash_thread(P, kind, hi + pb, gs_hi, rem_base + 1);
  }
}

// wait for both neighbours' packets of this exchange, then unpack them
__global__ void __launch_bounds__(256) k_p2p_recv(KP P, P2PLinks L, int kind, long long gs_lo,
                                                  long long gs_hi, int* rem_base) {
  const unsigned long long* fl[2] = {L.flag_src[kind][0], L.flag_src[kind][1]};
  if (!wait_flags(P, fl, 2, L.epoch[kind])) return;
  const unsigned char* lo = L.src[kind][0];  // from the rank below
  const unsigned char* hi = L.src[kind][1];
  if (kind == 0) {
    const long long i0 = blockIdx.x * blockDim.x + threadIdx.x, st = gridDim.x * blockDim.x;
    unpack_migrants(P, lo, i0, st);
    unpack_migrants(P, hi, i0, st);
    return;
  }
  const long long n2 = 2ll * P.G.g * P.G.txy;
  const double dz_lo = xmul((double)gs_lo, P.G.glz), dz_hi = xmul((double)gs_hi, P.G.glz);
  for (long long q = blockIdx.x * blockDim.x + threadIdx.x; q < 2 * n2;
       q += gridDim.x * blockDim.x) {
    const bool h = q >= n2;
    unpack_plane_site(P, kind, h ? 1 : -1, h ? hi : lo, h ? dz_hi : dz_lo, h ? q - n2 : q);
  }
  if ((kind == 1 || kind == 3) && blockIdx.x == 0 && threadIdx.x == 0) {
    const long long pb = L.plane_bytes[kind];
    unpack_clash_thread(P, kind, lo + pb, gs_lo, rem_base + 0);  // below first, as the
    unpack_clash_thread(P, kind, hi + pb, gs_hi, rem_base + 1);  // staged path does
  }
}

// end of a pass with the fused reverse halo: its partials are in the
// neighbours' memory (the pass grid has completed), publish them
__global__ void k_rev_signal(KP P, int kind) {
  pdl_wait();
  pdl_trigger();
  if (threadIdx.x != 0) return;
  const P2PLinks& L = *P.lk;
  __threadfence_system();
  const unsigned long long e = L.epoch[kind] + 1;
  L.epoch[kind] = e;
  __threadfence_system();
  st_relaxed_sys(L.flag_dst[kind][0], e);
  st_relaxed_sys(L.flag_dst[kind][1], e);
}
void launch_rev_signal(const KP& P, int kind, cudaStream_t s) {
  launch_pdl(k_rev_signal, 1, 32, 0, s, P, kind);
}
__global__ void k_rev_wait(KP P, int kind) {
  pdl_wait();
  pdl_trigger();
  rev_wait(P, kind);
}
void launch_rev_wait(const KP& P, int kind, cudaStream_t s) {
  launch_pdl(k_rev_wait, 1, 32, 0, s, P, kind);
}

__global__ void k_p2p_reduce(KP P, P2PLinks L, int energies, int kinetic) {
  if (threadIdx.x == 0) p2p_reduce_thread(P, L, energies, kinetic);
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
// fixed message size of an in-graph exchange (sizes cannot depend on
// device-side counts inside a captured step; all ranks share txy and g, so
// they agree on it): the planes plus room for kMsgRecords records; more
// sets CBX_RUNTIME on the sender
long long slab_msg_bytes(const KP& P, int kind) {
  long long b;
  if (kind == 0) {
    b = 16 + kMsgRecords * (long long)sizeof(MigRec);
  } else {
    b = slab_plane_bytes(P, kind);
    if (kind == 1 || kind == 3) b += 16 + kMsgRecords * (long long)sizeof(RemRec);
  }
  return (b + 255) / 256 * 256;
}

long long slab_buffer_bytes(const KP& P, int kind) {
  if (kind == 0) return 16 + (long long)P.cap_mov * sizeof(MigRec);
  long long b = slab_plane_bytes(P, kind);
  if (kind == 1 || kind == 3) b += 16 + (long long)P.cap_rem * sizeof(RemRec);
  return (b + 255) / 256 * 256;
}

static int plane_grid(const KP& P, int dirs) {
  const long long n = dirs * 2ll * P.G.g * P.G.txy;
  return (int)std::max<long long>(2, std::min<long long>((n + 255) / 256, 4 * 148));
}

void launch_pack(const KP& P, int kind, int dir, unsigned char* buf, long long cap,
                 cudaStream_t s) {
  if (kind == 0) {
    k_pack_migrants<<<1, 1024, 0, s>>>(P, dir, buf, cap);
    return;
  }
  const long long pb = slab_plane_bytes(P, kind);
  k_pack_planes<<<plane_grid(P, 1), 256, 0, s>>>(P, kind, dir, buf);
  if (kind == 1 || kind == 3) k_pack_clash<<<1, 32, 0, s>>>(P, kind, dir, buf + pb, cap - pb);
}

void launch_unpack(const KP& P, int kind, int from, const unsigned char* buf, long long gshift,
                   int* rem_base, cudaStream_t s) {
  if (kind == 0) {
    k_unpack_migrants<<<8, 256, 0, s>>>(P, buf);
    return;
  }
  const long long pb = slab_plane_bytes(P, kind);
  k_unpack_planes<<<plane_grid(P, 1), 256, 0, s>>>(P, kind, from, buf, gshift);
  if (kind == 1 || kind == 3) k_unpack_clash<<<1, 32, 0, s>>>(P, kind, buf + pb, gshift, rem_base);
}

void launch_remote_df(const KP& P, cudaStream_t s) { k_remote_df<<<8, 256, 0, s>>>(P); }

int launch_p2p_exchange(const KP& P, const P2PLinks& L, int kind, long long gs_lo,
                        long long gs_hi, int* rem_base, cudaStream_t s) {
  static const int fused = !ab_flag("CBX_P2P_SPLIT", 0);
  if (fused) {
    static int cap = 0;
    if (!cap) {  // co-resident blocks of the fused kernel
      int per_sm = 0, sms = 148, dev = 0;
      cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_p2p_xchg, 256, 0);
      cudaGetDevice(&dev);
      cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
      cap = std::max(2, std::min(per_sm, 2) * sms);
    }
    const int grid = kind == 0 ? 2 : std::min(plane_grid(P, 2), cap);
    k_p2p_xchg<<<grid, 256, 0, s>>>(P, L, kind, gs_lo, gs_hi, rem_base);
    return 1;
  }
  const int grid = kind == 0 ? 2 : plane_grid(P, 2);
  k_p2p_send<<<grid, 256, 0, s>>>(P, L, kind);
  k_p2p_recv<<<kind == 0 ? 8 : plane_grid(P, 2), 256, 0, s>>>(P, L, kind, gs_lo, gs_hi,
                                                                rem_base);
  return 2;
}
// the two halves of one exchange as separate launches (lockstep driving:
// the receiver is launched only after every sender's kernel completed)
void launch_p2p_send(const KP& P, const P2PLinks& L, int kind, cudaStream_t s) {
  k_p2p_send<<<kind == 0 ? 2 : plane_grid(P, 2), 256, 0, s>>>(P, L, kind);
}
void launch_p2p_recv(const KP& P, const P2PLinks& L, int kind, long long gs_lo, long long gs_hi,
                     int* rem_base, cudaStream_t s) {
  k_p2p_recv<<<kind == 0 ? 8 : plane_grid(P, 2), 256, 0, s>>>(P, L, kind, gs_lo, gs_hi,
                                                                rem_base);
}
void launch_p2p_reduce(const KP& P, const P2PLinks& L, int energies, int kinetic,
                       cudaStream_t s) {
  k_p2p_reduce<<<1, 32, 0, s>>>(P, L, energies, kinetic);
}

// ------------------------------------------------- step-state all-reduce
// (NCCL transport) red = {pair, embedding, kinetic, max_speed}: the local
// sums go in, the all-reduced values (sum, sum, sum, max) come back
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
