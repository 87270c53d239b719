// stencil_tile.cuh -- shared-memory tiled variant of the fast stencils
// (included by eam_kernels.cu after stencil_fast.cuh).
//
// A CTA stages one 8x8x4-cell brick plus a 2-cell halo of (x, y, z, dF)
// records and owner indices into shared memory, so every partner read is a
// shared-memory load; L1 is left to the spline tables.  Decisions, the
// pair mask, the RED scatter and the guard paths are those of
// stencil_fast.cuh.  Requires every offset to stay within 2 cells (true at
// the engine's index cutoff 5.6 + 0.3 a0); the host falls back otherwise.
#pragma once
// (no namespace: included inside namespace cbx)

constexpr int kTBX = 8, kTBY = 8, kTBZ = 4, kTH = 2;
constexpr int kTX = kTBX + 2 * kTH, kTY = kTBY + 2 * kTH, kTZ = kTBZ + 2 * kTH;
constexpr int kTC = kTX * kTY * kTZ;  // cells per tile (per sublattice)
constexpr size_t kTileSmem = 2 * (size_t)kTC * (sizeof(double4) + sizeof(int));

__constant__ int c_half_tile[2][kMaxOffsets];
__constant__ int c_full_tile[2][kMaxOffsets];

__host__ __device__ __forceinline__ int tile_brick_count(const Geo& G) {
  return ((G.bx + kTBX - 1) / kTBX) * ((G.by + kTBY - 1) / kTBY) * ((G.bz + kTBZ - 1) / kTBZ);
}

struct TileRef {
  double4* T;
  int* O;
};

// stage brick b: records of cells [origin - H, origin + B + H) of both sublattices
__device__ __forceinline__ void tile_fill(const KP& P, int brick, TileRef t, int& bx0, int& by0,
                                          int& bz0) {
  const Geo& G = P.G;
  const int nbx = (G.bx + kTBX - 1) / kTBX, nby = (G.by + kTBY - 1) / kTBY;
  bx0 = (brick % nbx) * kTBX;
  by0 = ((brick / nbx) % nby) * kTBY;
  bz0 = (brick / (nbx * nby)) * kTBZ;
  const int gx = bx0 + G.g - kTH, gy = by0 + G.g - kTH, gz = bz0 + G.g - kTH;
  for (int i = threadIdx.x; i < 2 * kTC; i += blockDim.x) {
    const int par = i >= kTC;
    const int l = i - par * kTC;
    const int lx = l % kTX, ly = (l / kTX) % kTY, lz = l / (kTX * kTY);
    const int cx = gx + lx, cy = gy + ly, cz = gz + lz;
    double4 r = make_double4(kVacant, kVacant, kVacant, 0.0);
    int o = 0;
    if (cx < G.tx && cy < G.ty && cz < G.tz) {
      const int d = (int)(par * G.NC + cell_of(cx, cy, cz, G));
      double a, b, c, w;
      ld256(P.pdf + d, a, b, c, w);
      r = make_double4(a, b, c, w);
      o = __ldg(P.tgt + d);
    }
    t.T[i] = r;
    t.O[i] = o;
  }
}

__device__ __forceinline__ double4 lds4(const double4* p) {
  const double2 a = reinterpret_cast<const double2*>(p)[0];
  const double2 b = reinterpret_cast<const double2*>(p)[1];
  return make_double4(a.x, a.y, b.x, b.y);
}

// ------------------------------------------------------------ density (N3)
template <bool FULL, int B>
__device__ __forceinline__ void density_site_tile(const KP& P, KP* Pp, TileRef tl, int par, int ts,
                                                  int d) {
  const double4 a = lds4(tl.T + ts);
  const double ax = a.x, ay = a.y, az = a.z;
  if (ax >= kVacantTest) {
    if (FULL) P.rho[d] = 0.0;
    return;
  }
  const int n = FULL ? c_full_n[par] : c_half_n[par];
  const int nin = FULL ? c_full_nin[par] : c_half_nin[par];
  const int* offs = FULL ? c_full[par] : c_half[par];
  const int* toffs = FULL ? c_full_tile[par] : c_half_tile[par];
  const double lo = P.cut2_lo, g2 = P.guard_r2, hi2 = P.cut2_hi;
  double acc = 0.0;
  unsigned long long m0 = 0, m1 = 0;
  for (int k0 = 0; k0 < n; k0 += B) {
    int seg[B], t[B];
    bool in[B];
    double s[B], r2[B], dx[B], dy[B], dz[B];
    bool rare = false;
#pragma unroll
    for (int b = 0; b < B; ++b) {
      const int k = min(k0 + b, n - 1);
      const int tj = ts + toffs[k];
      const double4 p = lds4(tl.T + tj);
      t[b] = tl.O[tj];
      dx[b] = xsub(ax, p.x);
      dy[b] = xsub(ay, p.y);
      dz[b] = xsub(az, p.z);
      r2[b] = fma(dz[b], dz[b], fma(dy[b], dy[b], dx[b] * dx[b]));
      const bool live_k = k0 + b < n;
      in[b] = live_k && r2[b] <= lo && r2[b] >= g2;
      rare |= live_k && !in[b] && r2[b] <= hi2;
    }
    if (rare) {
#pragma unroll
      for (int b = 0; b < B; ++b) {
        if (in[b] || k0 + b >= n || r2[b] > hi2) continue;
        const int k = k0 + b, j = d + offs[k];
        const double4 p = lds4(tl.T + ts + toffs[k]);
        const int st = decide<FULL>(P, par, k, j, ax, ay, az, p.x, p.y, p.z, dx[b], dy[b], dz[b],
                                    r2[b]);
        if (st == 1) {
          in[b] = true;
        } else if (st == 2) {
          m1 |= kGuardBit;
          acc += guard_rho(Pp, d, j, t[b], dx[b], dy[b], dz[b], FULL);
        }
      }
    }
#pragma unroll
    for (int b = 0; b < B; ++b) seg[b] = seg_index(P.fd, r2[b] * rsqrt(r2[b]), s[b]);
    double tA[B], tB[B], tC[B], tD[B];
#pragma unroll
    for (int b = 0; b < B; ++b)
      if (in[b]) ld256(P.fd.rec + 4 * (size_t)seg[b], tA[b], tB[b], tC[b], tD[b]);
#pragma unroll
    for (int b = 0; b < B; ++b) {
      if (in[b]) {
        const double rho = fma(fma(fma(tA[b], s[b], tB[b]), s[b], tC[b]), s[b], tD[b]);
        acc += rho;
        if (!FULL) red_add(&P.rho[t[b]], rho);
        set_bit(m0, m1, k0 + b);
      }
    }
  }
  (void)nin;
  if (FULL) P.rho[d] = acc;
  else red_add(&P.rho[d], acc);
  P.pmask[2 * (size_t)d] = m0;
  P.pmask[2 * (size_t)d + 1] = m1;
}

// ------------------------------------------------------------ force (mask)
template <bool FULL>
__device__ __forceinline__ double force_site_tile(const KP& P, KP* Pp, TileRef tl, int par,
                                                  int ts, int d) {
  const long long S = P.S;
  const double4 a = lds4(tl.T + ts);
  const double ax = a.x, ay = a.y, az = a.z, adf = a.w;
  if (ax >= kVacantTest) {
    if (FULL) {
      P.frc[d] = 0.0;
      P.frc[S + d] = 0.0;
      P.frc[2 * S + d] = 0.0;
    }
    return 0.0;
  }
  unsigned long long m0 = P.pmask[2 * (size_t)d], m1 = P.pmask[2 * (size_t)d + 1];
  const bool guard = (m1 & kGuardBit) != 0;
  m1 &= ~kGuardBit;
  const int* offs = FULL ? c_full[par] : c_half[par];
  const int* toffs = FULL ? c_full_tile[par] : c_half_tile[par];
  const double ih = P.ff.ih;
  double fx = 0.0, fy = 0.0, fz = 0.0, e = 0.0;
  while (m0 | m1) {
    int k[2];
    bool v[2];
#pragma unroll
    for (int b = 0; b < 2; ++b) {
      v[b] = (m0 | m1) != 0;
      if (m0) {
        k[b] = __ffsll(m0) - 1;
        m0 &= m0 - 1;
      } else if (m1) {
        k[b] = 63 + __ffsll(m1);
        m1 &= m1 - 1;
      } else {
        k[b] = k[0];  // padding lane: a real in-cutoff partner, result discarded
      }
    }
    int t[2], seg[2];
    double pw[2], dx[2], dy[2], dz[2], s[2], ri[2];
#pragma unroll
    for (int b = 0; b < 2; ++b) {
      const int tj = ts + toffs[k[b]];
      const double4 p = lds4(tl.T + tj);
      t[b] = tl.O[tj];
      pw[b] = p.w;
      dx[b] = xsub(ax, p.x);
      dy[b] = xsub(ay, p.y);
      dz[b] = xsub(az, p.z);
      const double r2 = fma(dz[b], dz[b], fma(dy[b], dy[b], dx[b] * dx[b]));
      ri[b] = rsqrt(r2);
      seg[b] = seg_index(P.ff, r2 * ri[b], s[b]);
    }
#pragma unroll
    for (int b = 0; b < 2; ++b) {
      if (!v[b]) continue;
      const PairOut o = pair_eval(P.ff.rec + 8 * (size_t)seg[b], s[b], ri[b], ih, adf + pw[b],
                                  dx[b], dy[b], dz[b]);
      fx -= o.qx;
      fy -= o.qy;
      fz -= o.qz;
      if (FULL) {
        e = fma(0.5, o.phi, e);
      } else {
        e += o.phi;
        red_add(&P.frc[t[b]], o.qx);
        red_add(&P.frc[S + t[b]], o.qy);
        red_add(&P.frc[2 * S + t[b]], o.qz);
      }
    }
  }
  if (guard) {
    const int n = FULL ? c_full_n[par] : c_half_n[par];
    for (int kk = 0; kk < n; ++kk) {
      const int jj = d + offs[kk];
      const double4 p = lds4(tl.T + ts + toffs[kk]);
      const double ddx = xsub(ax, p.x), ddy = xsub(ay, p.y), ddz = xsub(az, p.z);
      const double r2 = fma(ddz, ddz, fma(ddy, ddy, ddx * ddx));
      if (decide<FULL>(P, par, kk, jj, ax, ay, az, p.x, p.y, p.z, ddx, ddy, ddz, r2) != 2) continue;
      double q[4];
      if (guard_force(Pp, d, jj, tl.O[ts + toffs[kk]], ddx, ddy, ddz, adf + p.w, FULL, q)) {
        fx -= q[0];
        fy -= q[1];
        fz -= q[2];
        e = FULL ? fma(0.5, q[3], e) : e + q[3];
      }
    }
  }
  if (FULL) {
    P.frc[d] = fx;
    P.frc[S + d] = fy;
    P.frc[2 * S + d] = fz;
  } else {
    red_add(&P.frc[d], fx);
    red_add(&P.frc[S + d], fy);
    red_add(&P.frc[2 * S + d], fz);
  }
  return e;
}

// 8 warps; warp w: z-plane w >> 1, rows 4 (w & 1) .. +3; both sublattices
__device__ __forceinline__ bool tile_site(const Geo& G, int bx0, int by0, int bz0, int par,
                                          int& ts, int& d) {
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int lx = lane & 7, ly = (lane >> 3) + 4 * (w & 1), lz = w >> 1;
  const int cx = bx0 + lx, cy = by0 + ly, cz = bz0 + lz;
  ts = par * kTC + ((lz + kTH) * kTY + (ly + kTH)) * kTX + (lx + kTH);
  const bool live = cx < G.bx && cy < G.by && cz < G.bz;
  d = live ? (int)(par * G.NC + cell_of(cx + G.g, cy + G.g, cz + G.g, G)) : 0;
  return live;
}

template <bool FULL>
__global__ void __launch_bounds__(256, 2) k_density_tile(KP P) {
  if (P.st->err) return;
  extern __shared__ __align__(16) unsigned char smem[];
  TileRef tl{reinterpret_cast<double4*>(smem),
             reinterpret_cast<int*>(smem + 2 * (size_t)kTC * sizeof(double4))};
  const int nb = tile_brick_count(P.G);
  for (;;) {
    const int b = next_brick(&P.work[0]);
    if (b >= nb) break;
    int bx0, by0, bz0;
    tile_fill(P, b, tl, bx0, by0, bz0);
    __syncthreads();
    for (int par = 0; par < 2; ++par) {
      int ts, d;
      if (tile_site(P.G, bx0, by0, bz0, par, ts, d))
        density_site_tile<FULL, 4>(P, P.dself, tl, par, ts, d);
    }
  }
}

template <bool FULL>
__global__ void __launch_bounds__(256, 2) k_force_tile(KP P) {
  zero_pair_tail(P, gridDim.x * blockDim.x / 32);
  if (P.st->err || P.st->n_ovl) return;
  extern __shared__ __align__(16) unsigned char smem[];
  TileRef tl{reinterpret_cast<double4*>(smem),
             reinterpret_cast<int*>(smem + 2 * (size_t)kTC * sizeof(double4))};
  const int nb = tile_brick_count(P.G);
  double e = 0.0;
  for (;;) {
    const int b = next_brick(&P.work[1]);
    if (b >= nb) break;
    int bx0, by0, bz0;
    tile_fill(P, b, tl, bx0, by0, bz0);
    __syncthreads();
    for (int par = 0; par < 2; ++par) {
      int ts, d;
      if (tile_site(P.G, bx0, by0, bz0, par, ts, d))
        e += force_site_tile<FULL>(P, P.dself, tl, par, ts, d);
    }
  }
  for (int o = 16; o > 0; o >>= 1) e += __shfl_xor_sync(0xffffffffu, e, o);
  if ((threadIdx.x & 31) == 0) P.part_pair[(blockIdx.x * blockDim.x + threadIdx.x) >> 5] = e;
}

int tile_grid(const KP& P, bool force, int mode) {
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(k_density_tile<false>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         (int)kTileSmem);
    cudaFuncSetAttribute(k_density_tile<true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         (int)kTileSmem);
    cudaFuncSetAttribute(k_force_tile<false>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         (int)kTileSmem);
    cudaFuncSetAttribute(k_force_tile<true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         (int)kTileSmem);
    attr = true;
  }
  int per_sm = 0;
  const void* f = force ? (mode ? (const void*)k_force_tile<true> : (const void*)k_force_tile<false>)
                        : (mode ? (const void*)k_density_tile<true>
                                : (const void*)k_density_tile<false>);
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, f, 256, kTileSmem);
  int sms = 148, dev = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  return max(1, min(sms * max(per_sm, 1), tile_brick_count(P.G)));
}

void launch_density_tile(const KP& P, int mode, cudaStream_t s) {
  const int g = tile_grid(P, false, mode);
  if (mode) k_density_tile<true><<<g, 256, kTileSmem, s>>>(P);
  else k_density_tile<false><<<g, 256, kTileSmem, s>>>(P);
}
void launch_force_tile(const KP& P, int mode, int grid, cudaStream_t s) {
  if (mode) k_force_tile<true><<<grid, 256, kTileSmem, s>>>(P);
  else k_force_tile<false><<<grid, 256, kTileSmem, s>>>(P);
}
