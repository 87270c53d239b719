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
// * persistent warps pull 32-cell chunks of one sublattice from an atomic
//   work counter, so the tail of a launch is one chunk, not a wave.
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

// ------------------------------------------------------------------ density
template <bool FULL>
__device__ __forceinline__ void density_site(const KP& P, int par, long long d) {
  const double4* __restrict__ pdf = P.pdf;
  const float4* __restrict__ uf = P.uf;
  const float4 af = uf[d];
  if (af.x >= kVacantF) {
    if (FULL) P.rho[d] = 0.0;
    return;
  }
  double ax, ay, az, aw;
  ld256(pdf + d, ax, ay, az, aw);
  const int n = FULL ? c_full_n[par] : c_half_n[par];
  const float hi = P.band_hi, lo = P.band_lo;
  double acc = 0.0;
#pragma unroll 2
  for (int k = 0; k < n; ++k) {
    const long long j = d + (FULL ? c_full[par][k] : c_half[par][k]);
    const float4 pf = ld128f(uf + j);
    const float fx = af.x - pf.x, fy = af.y - pf.y, fz = af.z - pf.z;
    const float r2f = fmaf(fz, fz, fmaf(fy, fy, fx * fx));
    if (r2f > hi) continue;
    double px, py, pz, pw;
    ld256(pdf + j, px, py, pz, pw);
    const double dx = xsub(ax, px), dy = xsub(ay, py), dz = xsub(az, pz);
    if (r2f >= lo) {  // near the cutoff: the reference's exact r^2 decides
      double ex = dx, ey = dy, ez = dz;
      if (FULL && c_full_flat[par][k] < 0) {
        const double4 a4 = make_double4(ax, ay, az, aw), p4 = make_double4(px, py, pz, pw);
        full_orient(P, a4, j, p4, ex, ey, ez);
      }
      if (exact_r2(ex, ey, ez) > P.cut2) continue;
    }
    const double r2 = fma(dz, dz, fma(dy, dy, dx * dx));
    const int tw = __float_as_int(pf.w);
    const long long tgt = tw < 0 ? j : (long long)tw;
    double rho;
    if (r2 < P.guard_r2) {  // overlap / sub-table separations: the reference path
      const double r2x = exact_r2(dx, dy, dz);
      if (r2x < kOverlapR2) {
        const long long rd = ref_of_dev(d, P.G.NC), rj = ref_of_dev(j, P.G.NC);
        report_overlap(P, ((unsigned long long)min(rd, rj) << 12) | (unsigned)k, P.tag[d],
                       P.tag[tgt], r2x);
        continue;
      }
      rho = pair_rho(P, r2x);
    } else {
      const double r = r2 * rinv_of(r2);
      double s;
      const int i = seg_index(P.fd, r, s);
      double A, B, C, D;
      ld256(P.fd.rec + 4 * (size_t)i, A, B, C, D);
      rho = fma(fma(fma(A, s, B), s, C), s, D);
    }
    acc += rho;
    if (!FULL) atomicAdd(&P.rho[tgt], rho);
  }
  if (FULL) P.rho[d] = acc;
  else atomicAdd(&P.rho[d], acc);
}

// -------------------------------------------------------------------- force
template <bool FULL>
__device__ __forceinline__ double force_site(const KP& P, int par, long long d) {
  const double4* __restrict__ pdf = P.pdf;
  const float4* __restrict__ uf = P.uf;
  const long long S = P.S;
  const float4 af = uf[d];
  if (af.x >= kVacantF) {
    if (FULL) {
      P.frc[d] = 0.0;
      P.frc[S + d] = 0.0;
      P.frc[2 * S + d] = 0.0;
    }
    return 0.0;
  }
  double ax, ay, az, adf;
  ld256(pdf + d, ax, ay, az, adf);
  const int n = FULL ? c_full_n[par] : c_half_n[par];
  const float hi = P.band_hi, lo = P.band_lo;
  const double ih = P.ff.ih;
  double fx = 0.0, fy = 0.0, fz = 0.0, e = 0.0;
#pragma unroll 2
  for (int k = 0; k < n; ++k) {
    const long long j = d + (FULL ? c_full[par][k] : c_half[par][k]);
    const float4 pf = ld128f(uf + j);
    const float gx = af.x - pf.x, gy = af.y - pf.y, gz = af.z - pf.z;
    const float r2f = fmaf(gz, gz, fmaf(gy, gy, gx * gx));
    if (r2f > hi) continue;
    double px, py, pz, pdf_j;
    ld256(pdf + j, px, py, pz, pdf_j);
    const double dx = xsub(ax, px), dy = xsub(ay, py), dz = xsub(az, pz);
    if (r2f >= lo) {
      double ex = dx, ey = dy, ez = dz;
      if (FULL && c_full_flat[par][k] < 0) {
        const double4 a4 = make_double4(ax, ay, az, adf), p4 = make_double4(px, py, pz, pdf_j);
        full_orient(P, a4, j, p4, ex, ey, ez);
      }
      if (exact_r2(ex, ey, ez) > P.cut2) continue;
    }
    const double r2 = fma(dz, dz, fma(dy, dy, dx * dx));
    const int tw = __float_as_int(pf.w);
    const long long tgt = tw < 0 ? j : (long long)tw;
    double mfp, phi;  // mfp = -fp of forces.cpp:164
    if (r2 < P.guard_r2) {
      const double r2x = exact_r2(dx, dy, dz);
      if (r2x < kOverlapR2) {
        const long long rd = ref_of_dev(d, P.G.NC), rj = ref_of_dev(j, P.G.NC);
        report_overlap(P, (1ull << 61) | ((unsigned long long)min(rd, rj) << 12) | (unsigned)k,
                       P.tag[d], P.tag[tgt], r2x);
        continue;
      }
      double fp;
      pair_force(P, r2x, adf + pdf_j, fp, phi);
      mfp = -fp;
    } else {
      const double ri = rinv_of(r2);
      const double r = r2 * ri;
      double s;
      const int i = seg_index(P.ff, r, s);
      const double* rec = P.ff.rec + 8 * (size_t)i;
      double zA, zB, zC, zD, pA, pB, pC, pD;
      ld256(rec, zA, zB, zC, zD);
      ld256(rec + 4, pA, pB, pC, pD);
      const double s15 = 1.5 * s, s2 = s + s;
      const double z = fma(fma(fma(zA, s, zB), s, zC), s, zD);
      const double zs = fma(fma(zA, s15, zB), s2, zC);  // dz/ds
      const double ps = fma(fma(pA, s15, pB), s2, pC);  // drho/ds
      phi = z * ri;
      // phi' = (z' - phi)/r,  -fp = ((dFa + dFp) rho' + phi')/r, d/dr = ih d/ds
      const double dphi = fma(zs, ih, -phi) * ri;
      mfp = fma((adf + pdf_j) * ps, ih, dphi) * ri;
    }
    const double qx = mfp * dx, qy = mfp * dy, qz = mfp * dz;
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

// persistent warps: chunk c covers 32 interior cells of sublattice c & 1
__device__ __forceinline__ int next_chunk(int* ctr) {
  int c = 0;
  if ((threadIdx.x & 31) == 0) c = atomicAdd(ctr, 1);
  return __shfl_sync(0xffffffffu, c, 0);
}

template <bool FULL>
__global__ void __launch_bounds__(128, 6) k_density_fast(KP P) {
  if (P.st->err) return;
  const int lane = threadIdx.x & 31;
  const int nchunk = (int)(2 * ((P.G.NI + 31) / 32));
  for (;;) {
    const int c = next_chunk(&P.work[0]);
    if (c >= nchunk) break;
    const int par = c & 1;
    const long long e = (long long)(c >> 1) * 32 + lane;
    if (e < P.G.NI) density_site<FULL>(P, par, par * P.G.NC + interior_cell(e, P.G));
  }
}

template <bool FULL>
__global__ void __launch_bounds__(128, 6) k_force_fast(KP P) {
  if (P.st->err || P.st->n_ovl) return;
  const int lane = threadIdx.x & 31;
  const int nchunk = (int)(2 * ((P.G.NI + 31) / 32));
  double e = 0.0;
  for (;;) {
    const int c = next_chunk(&P.work[1]);
    if (c >= nchunk) break;
    const int par = c & 1;
    const long long el = (long long)(c >> 1) * 32 + lane;
    if (el < P.G.NI) e += force_site<FULL>(P, par, par * P.G.NC + interior_cell(el, P.G));
  }
  // per-warp partial energies (deterministic only per schedule; summed in
  // k_finalize in slot order)
  for (int o = 16; o > 0; o >>= 1) e += __shfl_xor_sync(0xffffffffu, e, o);
  if (lane == 0) P.part_pair[(blockIdx.x * blockDim.x + threadIdx.x) >> 5] = e;
}

int fast_grid(const KP& P, bool force, int mode) {
  int per_sm = 0;
  if (force)
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(
        &per_sm, mode ? (const void*)k_force_fast<true> : (const void*)k_force_fast<false>, 128, 0);
  else
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(
        &per_sm, mode ? (const void*)k_density_fast<true> : (const void*)k_density_fast<false>,
        128, 0);
  int sms = 148;
  int dev = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const int chunks = (int)(2 * ((P.G.NI + 31) / 32));
  const int blocks = sms * (per_sm > 0 ? per_sm : 1);
  return max(1, min(blocks, (chunks + 3) / 4));
}

void launch_density_fast(const KP& P, int mode, int grid, cudaStream_t s) {
  if (mode) k_density_fast<true><<<grid, 128, 0, s>>>(P);
  else k_density_fast<false><<<grid, 128, 0, s>>>(P);
}
void launch_force_fast(const KP& P, int mode, int grid, cudaStream_t s) {
  if (mode) k_force_fast<true><<<grid, 128, 0, s>>>(P);
  else k_force_fast<false><<<grid, 128, 0, s>>>(P);
}


