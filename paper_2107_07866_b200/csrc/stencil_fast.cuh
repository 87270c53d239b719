// stencil_fast.cuh -- the density and force passes, B200 fast path
// (included by eam_kernels.cu: one translation unit with the offset tables
// in constant memory).
//
// Same candidate set, orientation and exact in-cutoff decisions as
// eam_kernels.cu (which mirrors the reference's arithmetic literally and
// serves as CBX_STENCIL_REFERENCE); this variant is organised for sm_100a:
//
// * candidate filter in fp32 on a 16-byte shadow record uf[] = (x, y, z,
//   owner) -- one LDG.128 per candidate instead of a 32-byte fp64 gather, and
//   the fp32 pipe instead of the fp64 pipe.  The float distance is only a
//   filter: candidates within `band` of the cutoff (a bound on the float
//   error derived from the box extent, host side) get the exact fp64 r^2 of
//   the reference (operation order of forces.cpp:123-125), so every
//   in-cutoff decision is bit-identical to the reference.
// * fp64 work only for in-cutoff pairs: one 256-bit load of the partner's
//   (x, y, z, dF) and one or two 256-bit loads of a 32-byte-aligned spline
//   record in the normalised variable s in [0, 1) (coefficients A=a h^3,
//   B=b h^2, C=c h, D=d of the reference segment, spline.h:19-22).
// * 1/r from the fp64 reciprocal square root, the segment index from a
//   round-down add of 2^52 (no fp64<->int conversions).
// * persistent CTAs pull 8x4x4-cell bricks from an atomic work counter; the
//   4 warps of a CTA take one z-plane each and sweep both sublattices, so
//   the brick's neighbourhood (~55 KB) stays in L1 across all its
//   candidates, and the launch tail is one brick.
// * candidates are processed in batches (4 for density, 2 for force): the
//   batch's filter loads, then its partner loads, then its table loads are
//   issued back to back, so each warp keeps several L1/L2 requests in flight.
// * fold_rho / fold_force (forces.cpp:290-309): partner contributions are
//   RED-added to the partner's owner (interior site or periodic source).
#pragma once
// (no namespace: included inside namespace cbx)

__device__ __forceinline__ void ld256(const void* p, double& a, double& b, double& c,
                                      double& d) {
  asm volatile("ld.global.nc.v4.f64 {%0,%1,%2,%3}, [%4];"
               : "=d"(a), "=d"(b), "=d"(c), "=d"(d)
               : "l"(p));
}
__device__ __forceinline__ float4 ld128f(const float4* p) { return __ldg(p); }

constexpr double kTwo52 = 4503599627370496.0;

// segment index and normalised offset: u = (r - x0)/h, i = floor(u), s = u - i
__device__ __forceinline__ int seg_index(const FastTab& T, double r, double& s) {
  const double u = fma(r, T.ih, T.c0);
  const double t = __dadd_rd(u, kTwo52);  // 2^52 + floor(u) for 0 <= u < 2^52
  s = u - (t - kTwo52);
  return min(__double2loint(t), T.nseg);  // segment nseg is the padded one
}

// 1/r and r from r^2 (rsqrt + Newton steps, ~1 ulp)
__device__ __forceinline__ double rinv_of(double r2) { return rsqrt(r2); }


constexpr int kBrickX = 8, kBrickY = 4, kBrickZ = 4;

// guard pass (r below the first knot, overlaps): revisit the site's list
// and treat only the pairs the hot loop skipped (fp64 r^2 < guard_r2) with
// the reference-literal evaluation of eam_kernels.cu.  Never taken in
// thermal runs; kept out of the hot loop's register budget.
__device__ __forceinline__ bool guard_pair(const KP& P, int par, int d, int k, bool full,
                                           double ax, double ay, double az, const float4& af,
                                           int& j, int& tgt, double& dx, double& dy, double& dz,
                                           double& pw) {
  j = d + (full ? c_full[par][k] : c_half[par][k]);
  const float4 pf = P.uf[j];
  const float fx = af.x - pf.x, fy = af.y - pf.y, fz = af.z - pf.z;
  if (fmaf(fz, fz, fmaf(fy, fy, fx * fx)) > P.band_hi) return false;
  const double4 p = P.pdf[j];
  dx = xsub(ax, p.x);
  dy = xsub(ay, p.y);
  dz = xsub(az, p.z);
  pw = p.w;
  if (fma(dz, dz, fma(dy, dy, dx * dx)) >= P.guard_r2) return false;
  const int tw = __float_as_int(pf.w);
  tgt = tw < 0 ? j : tw;
  return true;
}

template <bool FULL, bool UNUSED>
__device__ __noinline__ double guard_pass(const KP& P, int par, int d, double ax, double ay,
                                          double az, double aw, float4 af) {
  const int n = FULL ? c_full_n[par] : c_half_n[par];
  double acc = 0.0;
  for (int k = 0; k < n; ++k) {
    int j, tgt;
    double dx, dy, dz, pw;
    if (!guard_pair(P, par, d, k, FULL, ax, ay, az, af, j, tgt, dx, dy, dz, pw)) continue;
    const double r2x = exact_r2(dx, dy, dz);
    if (r2x < kOverlapR2) {
      const long long rd = ref_of_dev(d, P.G.NC), rj = ref_of_dev(j, P.G.NC);
      report_overlap(P, ((unsigned long long)min(rd, rj) << 12) | (unsigned)k, P.tag[d],
                     P.tag[tgt], r2x);
      continue;
    }
    const double rho = pair_rho(P, r2x);
    acc += rho;
    if (!FULL) atomicAdd(&P.rho[tgt], rho);
  }
  return acc;
}

template <bool FULL>
__device__ __noinline__ void guard_force(const KP& P, int par, int d, double ax, double ay,
                                         double az, double adf, float4 af, double* out) {
  const int n = FULL ? c_full_n[par] : c_half_n[par];
  const long long S = P.S;
  double fx = 0.0, fy = 0.0, fz = 0.0, e = 0.0;
  for (int k = 0; k < n; ++k) {
    int j, tgt;
    double dx, dy, dz, pw;
    if (!guard_pair(P, par, d, k, FULL, ax, ay, az, af, j, tgt, dx, dy, dz, pw)) continue;
    const double r2x = exact_r2(dx, dy, dz);
    if (r2x < kOverlapR2) {
      const long long rd = ref_of_dev(d, P.G.NC), rj = ref_of_dev(j, P.G.NC);
      report_overlap(P, (1ull << 61) | ((unsigned long long)min(rd, rj) << 12) | (unsigned)k,
                     P.tag[d], P.tag[tgt], r2x);
      continue;
    }
    double fp, phi;
    pair_force(P, r2x, adf + pw, fp, phi);
    const double qx = -fp * dx, qy = -fp * dy, qz = -fp * dz;
    fx -= qx;
    fy -= qy;
    fz -= qz;
    if (FULL) {
      e = fma(0.5, phi, e);
    } else {
      e += phi;
      atomicAdd(&P.frc[tgt], qx);
      atomicAdd(&P.frc[S + tgt], qy);
      atomicAdd(&P.frc[2 * S + tgt], qz);
    }
  }
  out[0] = fx;
  out[1] = fy;
  out[2] = fz;
  out[3] = e;
}

// ------------------------------------------------------------------ density
template <bool FULL, int B>
__device__ __forceinline__ void density_site(const KP& P, int par, int d, bool live) {
  const double4* __restrict__ pdf = P.pdf;
  const float4* __restrict__ uf = P.uf;
  float4 af = make_float4(kVacantF, kVacantF, kVacantF, 0.f);
  if (live) af = uf[d];
  if (af.x >= kVacantF) {
    if (FULL && live) P.rho[d] = 0.0;
    return;
  }
  double ax, ay, az, aw;
  ld256(pdf + d, ax, ay, az, aw);
  const int n = FULL ? c_full_n[par] : c_half_n[par];
  const int* offs = FULL ? c_full[par] : c_half[par];
  const float hi = P.band_hi, lo = P.band_lo;
  double acc = 0.0;
  bool slow = false;
  for (int k0 = 0; k0 < n; k0 += B) {
    int j[B];
    float4 pf[B];
#pragma unroll
    for (int b = 0; b < B; ++b) {
      j[b] = d + offs[min(k0 + b, n - 1)];
      pf[b] = ld128f(uf + j[b]);
    }
    bool go[B], band[B];
#pragma unroll
    for (int b = 0; b < B; ++b) {
      const float fx = af.x - pf[b].x, fy = af.y - pf[b].y, fz = af.z - pf[b].z;
      const float r2f = fmaf(fz, fz, fmaf(fy, fy, fx * fx));
      go[b] = (k0 + b < n) && r2f <= hi;
      band[b] = r2f >= lo;
    }
    double px[B], py[B], pz[B];
#pragma unroll
    for (int b = 0; b < B; ++b) {
      if (go[b]) {
        double w;
        ld256(pdf + j[b], px[b], py[b], pz[b], w);
      }
    }
    double s[B];
    int seg[B];
#pragma unroll
    for (int b = 0; b < B; ++b) {
      if (!go[b]) continue;
      const double dx = xsub(ax, px[b]), dy = xsub(ay, py[b]), dz = xsub(az, pz[b]);
      if (band[b]) {  // near the cutoff: the reference's exact r^2 decides
        double ex = dx, ey = dy, ez = dz;
        if (FULL && c_full_flat[par][k0 + b] < 0)
          full_orient(P, make_double4(ax, ay, az, aw), j[b], make_double4(px[b], py[b], pz[b], 0.0),
                      ex, ey, ez);
        if (exact_r2(ex, ey, ez) > P.cut2) {
          go[b] = false;
          continue;
        }
      }
      const double r2 = fma(dz, dz, fma(dy, dy, dx * dx));
      if (r2 < P.guard_r2) {  // overlap / sub-table separation: second pass below
        go[b] = false;
        slow = true;
        continue;
      }
      const double r = r2 * rsqrt(r2);
      seg[b] = seg_index(P.fd, r, s[b]);
    }
    double tA[B], tB[B], tC[B], tD[B];
#pragma unroll
    for (int b = 0; b < B; ++b)
      if (go[b]) ld256(P.fd.rec + 4 * (size_t)seg[b], tA[b], tB[b], tC[b], tD[b]);
#pragma unroll
    for (int b = 0; b < B; ++b) {
      if (!go[b]) continue;
      const double rho = fma(fma(fma(tA[b], s[b], tB[b]), s[b], tC[b]), s[b], tD[b]);
      acc += rho;
      if (!FULL) {
        const int tw = __float_as_int(pf[b].w);
        atomicAdd(&P.rho[tw < 0 ? j[b] : tw], rho);
      }
    }
  }
  if (slow) acc += guard_pass<FULL, false>(P, par, d, ax, ay, az, aw, af);
  if (FULL) P.rho[d] = acc;
  else atomicAdd(&P.rho[d], acc);
}

// -------------------------------------------------------------------- force
template <bool FULL, int B>
__device__ __forceinline__ double force_site(const KP& P, int par, int d, bool live) {
  const double4* __restrict__ pdf = P.pdf;
  const float4* __restrict__ uf = P.uf;
  const long long S = P.S;
  float4 af = make_float4(kVacantF, kVacantF, kVacantF, 0.f);
  if (live) af = uf[d];
  if (af.x >= kVacantF) {
    if (FULL && live) {
      P.frc[d] = 0.0;
      P.frc[S + d] = 0.0;
      P.frc[2 * S + d] = 0.0;
    }
    return 0.0;
  }
  double ax, ay, az, adf;
  ld256(pdf + d, ax, ay, az, adf);
  const int n = FULL ? c_full_n[par] : c_half_n[par];
  const int* offs = FULL ? c_full[par] : c_half[par];
  const float hi = P.band_hi, lo = P.band_lo;
  const double ih = P.ff.ih;
  double fx = 0.0, fy = 0.0, fz = 0.0, e = 0.0;
  bool slow = false;
  for (int k0 = 0; k0 < n; k0 += B) {
    int j[B];
    float4 pf[B];
#pragma unroll
    for (int b = 0; b < B; ++b) {
      j[b] = d + offs[min(k0 + b, n - 1)];
      pf[b] = ld128f(uf + j[b]);
    }
    bool go[B], band[B];
#pragma unroll
    for (int b = 0; b < B; ++b) {
      const float gx = af.x - pf[b].x, gy = af.y - pf[b].y, gz = af.z - pf[b].z;
      const float r2f = fmaf(gz, gz, fmaf(gy, gy, gx * gx));
      go[b] = (k0 + b < n) && r2f <= hi;
      band[b] = r2f >= lo;
    }
    double px[B], py[B], pz[B], pw[B];
#pragma unroll
    for (int b = 0; b < B; ++b)
      if (go[b]) ld256(pdf + j[b], px[b], py[b], pz[b], pw[b]);
    double dxs[B], dys[B], dzs[B], s[B], ri[B];
    int seg[B];
#pragma unroll
    for (int b = 0; b < B; ++b) {
      if (!go[b]) continue;
      const double dx = xsub(ax, px[b]), dy = xsub(ay, py[b]), dz = xsub(az, pz[b]);
      dxs[b] = dx;
      dys[b] = dy;
      dzs[b] = dz;
      if (band[b]) {
        double ex = dx, ey = dy, ez = dz;
        if (FULL && c_full_flat[par][k0 + b] < 0)
          full_orient(P, make_double4(ax, ay, az, adf), j[b],
                      make_double4(px[b], py[b], pz[b], pw[b]), ex, ey, ez);
        if (exact_r2(ex, ey, ez) > P.cut2) {
          go[b] = false;
          continue;
        }
      }
      const double r2 = fma(dz, dz, fma(dy, dy, dx * dx));
      if (r2 < P.guard_r2) {
        go[b] = false;
        slow = true;
        continue;
      }
      ri[b] = rsqrt(r2);
      seg[b] = seg_index(P.ff, r2 * ri[b], s[b]);
    }
    double zA[B], zB[B], zC[B], zD[B], qA[B], qB[B], qC[B], qD[B];
#pragma unroll
    for (int b = 0; b < B; ++b) {
      if (!go[b]) continue;
      const double* rec = P.ff.rec + 8 * (size_t)seg[b];
      ld256(rec, zA[b], zB[b], zC[b], zD[b]);
      ld256(rec + 4, qA[b], qB[b], qC[b], qD[b]);
    }
#pragma unroll
    for (int b = 0; b < B; ++b) {
      if (!go[b]) continue;
      const double sb = s[b], s15 = 1.5 * sb, s2 = sb + sb;
      const double z = fma(fma(fma(zA[b], sb, zB[b]), sb, zC[b]), sb, zD[b]);
      const double zs = fma(fma(zA[b], s15, zB[b]), s2, zC[b]);  // dz/ds
      const double ps = fma(fma(qA[b], s15, qB[b]), s2, qC[b]);  // drho/ds
      const double phi = z * ri[b];
      // phi' = (z' - phi)/r;  -fp = ((dFa + dFp) rho' + phi')/r;  d/dr = ih d/ds
      const double dphi = fma(zs, ih, -phi) * ri[b];
      const double mfp = fma((adf + pw[b]) * ps, ih, dphi) * ri[b];
      const double qx = mfp * dxs[b], qy = mfp * dys[b], qz = mfp * dzs[b];
      fx -= qx;
      fy -= qy;
      fz -= qz;
      if (FULL) {
        e = fma(0.5, phi, e);
      } else {
        e += phi;
        const int tw = __float_as_int(pf[b].w);
        const int tgt = tw < 0 ? j[b] : tw;
        atomicAdd(&P.frc[tgt], qx);
        atomicAdd(&P.frc[S + tgt], qy);
        atomicAdd(&P.frc[2 * S + tgt], qz);
      }
    }
  }
  if (slow) {
    double g[4];
    guard_force<FULL>(P, par, d, ax, ay, az, adf, af, g);
    fx += g[0];
    fy += g[1];
    fz += g[2];
    e += g[3];
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
  return e;
}

// persistent CTAs over bricks: warp w owns z-plane w of the brick and sweeps
// both sublattices (even then odd: balanced half-list lengths 46 + 66)
__device__ __forceinline__ int next_brick(int* ctr) {
  __shared__ int s_brick;
  __syncthreads();
  if (threadIdx.x == 0) s_brick = atomicAdd(ctr, 1);
  __syncthreads();
  return s_brick;
}

__device__ __forceinline__ bool brick_site(const Geo& G, int brick, int par, long long& d) {
  const int nbx = (G.bx + kBrickX - 1) / kBrickX, nby = (G.by + kBrickY - 1) / kBrickY;
  const int bxi = brick % nbx, r = brick / nbx;
  const int byi = r % nby, bzi = r / nby;
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int cx = bxi * kBrickX + (lane & 7), cy = byi * kBrickY + (lane >> 3),
            cz = bzi * kBrickZ + w;
  const bool live = cx < G.bx && cy < G.by && cz < G.bz;
  d = live ? par * G.NC + cell_of(cx + G.g, cy + G.g, cz + G.g, G) : 0;
  return live;
}

__host__ __device__ __forceinline__ int brick_count(const Geo& G) {
  return ((G.bx + kBrickX - 1) / kBrickX) * ((G.by + kBrickY - 1) / kBrickY) *
         ((G.bz + kBrickZ - 1) / kBrickZ);
}

template <bool FULL>
__global__ void __launch_bounds__(128, 4) k_density_fast(KP P) {
  if (P.st->err) return;
  const int nb = brick_count(P.G);
  for (;;) {
    const int b = next_brick(&P.work[0]);
    if (b >= nb) break;
    for (int par = 0; par < 2; ++par) {
      long long d;
      const bool live = brick_site(P.G, b, par, d);
      density_site<FULL, 4>(P, par, (int)d, live);
    }
  }
}

template <bool FULL, int B>
__global__ void __launch_bounds__(128, 4) k_force_fast(KP P) {
  if (P.st->err || P.st->n_ovl) return;
  const int nb = brick_count(P.G);
  double e = 0.0;
  for (;;) {
    const int b = next_brick(&P.work[1]);
    if (b >= nb) break;
    for (int par = 0; par < 2; ++par) {
      long long d;
      const bool live = brick_site(P.G, b, par, d);
      e += force_site<FULL, B>(P, par, (int)d, live);
    }
  }
  for (int o = 16; o > 0; o >>= 1) e += __shfl_xor_sync(0xffffffffu, e, o);
  if ((threadIdx.x & 31) == 0) P.part_pair[(blockIdx.x * blockDim.x + threadIdx.x) >> 5] = e;
}

int fast_grid(const KP& P, bool force, int mode) {
  int per_sm = 0;
  if (force)
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(
        &per_sm, mode ? (const void*)k_force_fast<true, 2> : (const void*)k_force_fast<false, 2>,
        128, 0);
  else
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(
        &per_sm, mode ? (const void*)k_density_fast<true> : (const void*)k_density_fast<false>,
        128, 0);
  int sms = 148;
  int dev = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const int blocks = sms * (per_sm > 0 ? per_sm : 1);
  return max(1, min(blocks, brick_count(P.G)));
}

void launch_density_fast(const KP& P, int mode, int grid, cudaStream_t s) {
  if (mode) k_density_fast<true><<<grid, 128, 0, s>>>(P);
  else k_density_fast<false><<<grid, 128, 0, s>>>(P);
}
void launch_force_fast(const KP& P, int mode, int grid, cudaStream_t s) {
  static const int batch = [] {
    const char* e = getenv("CBX_FORCE_BATCH");
    return e ? atoi(e) : 2;
  }();
  if (batch == 1) {
    if (mode) k_force_fast<true, 1><<<grid, 128, 0, s>>>(P);
    else k_force_fast<false, 1><<<grid, 128, 0, s>>>(P);
  } else {
    if (mode) k_force_fast<true, 2><<<grid, 128, 0, s>>>(P);
    else k_force_fast<false, 2><<<grid, 128, 0, s>>>(P);
  }
}
