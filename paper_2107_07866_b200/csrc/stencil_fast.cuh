// stencil_fast.cuh -- the density and force passes, B200 fast path
// (included by eam_kernels.cu: one translation unit with the offset tables
// in constant memory).
//
// Same candidate set, orientation and exact in-cutoff decisions as
// eam_kernels.cu (which mirrors the reference's arithmetic literally and
// serves as CBX_STENCIL_REFERENCE).  Organised for sm_100a:
//
// * offset lists are ordered by lattice distance and split (host side) into
//   "inner" sites (lattice distance <= cutoff: shells 1-5, 29 of the 56
//   half-list candidates) and "skin" sites (shells 6-8, index skin of
//   sim.cpp:73).  Inner candidates go straight to a 256-bit load of the
//   partner's (x, y, z, dF) and the fp64 r^2; skin candidates are first
//   filtered in fp32 on the 16-byte shadow uf[] = (x, y, z, owner).
// * every in-cutoff decision is exact: an fp64/fp32 distance only decides
//   when it is farther from the cutoff than its rounding bound (host side);
//   otherwise the reference's r^2 (operation order of forces.cpp:123-125,
//   no FMA) decides, so the pair set is bit-identical to the reference.
// * spline records are 32-byte aligned in the normalised variable
//   s = (r - x0)/h - i (A = a h^3, B = b h^2, C = c h, D = d of the
//   reference segment, spline.h:19-22); 1/r from the fp64 rsqrt; the segment
//   index from a round-down add of 2^52 (no fp64<->int conversions).
// * candidates are processed in batches whose loads are issued back to back
//   (memory-level parallelism), partner contributions are RED.ADD.F64 to the
//   partner's owner -- fold_rho / fold_force of forces.cpp:290-309 at
//   scatter time.
// * persistent CTAs pull 8x4x4-cell bricks from an atomic work counter; the
//   4 warps of a CTA take one z-plane each and sweep both sublattices, so the
//   brick's neighbourhood stays in L1 and the launch tail is one brick.
#pragma once
// (no namespace: included inside namespace cbx)

__device__ __forceinline__ void ld256(const void* p, double& a, double& b, double& c,
                                      double& d) {
  // not volatile: a pure read of data that is constant during the kernel,
  // free to be scheduled early by the compiler
  asm("ld.global.nc.v4.f64 {%0,%1,%2,%3}, [%4];" : "=d"(a), "=d"(b), "=d"(c), "=d"(d) : "l"(p));
}
__device__ __forceinline__ void red_add(double* p, double v) {
  // no "memory" clobber: reductions need no ordering within the pass
  asm volatile("red.global.add.f64 [%0], %1;" ::"l"(p), "d"(v));
}

constexpr double kTwo52 = 4503599627370496.0;
// per-site pair mask written by the density pass (bit k: offset k in cutoff
// on the fast path; top bit: the site has guard pairs) and replayed by the
// force pass, so the force pass never re-filters candidates
constexpr unsigned long long kGuardBit = 1ull << 63;
constexpr int kMaskBits = 127;
__device__ __forceinline__ void set_bit(unsigned long long& m0, unsigned long long& m1, int k) {
  if (k < 64) m0 |= 1ull << k;
  else m1 |= 1ull << (k - 64);
}
constexpr int kBrickX = 8, kBrickY = 4, kBrickZ = 4;

// segment index and normalised offset: u = (r - x0)/h, i = floor(u), s = u - i
__device__ __forceinline__ int seg_index(const FastTab& T, double r, double& s) {
  const double u = fma(r, T.ih, T.c0);
  const double t = __dadd_rd(u, kTwo52);  // 2^52 + floor(u) for 0 <= u < 2^52
  s = u - (t - kTwo52);
  return min(__double2loint(t), T.nseg);  // segment nseg is the padded one
}

__device__ __forceinline__ unsigned long long pair_key(const KP& P, long long d, long long j,
                                                       unsigned long long phase) {
  const long long a = ref_of_dev(d, P.G.NC), b = ref_of_dev(j, P.G.NC);
  const long long lo = min(a, b), hi = max(a, b);
  return phase | ((unsigned long long)lo << 24) | (unsigned long long)((hi - lo) & 0xffffff);
}

// the decision for one candidate once its fp64 displacement is known:
// 0 out, 1 in (fast path), 2 guard (r below the first knot or overlap)
template <bool FULL>
__device__ __forceinline__ int decide(const KP& P, int par, int k, int j, double ax, double ay,
                                      double az, double px, double py, double pz, double dx,
                                      double dy, double dz, double r2) {
  if (r2 > P.cut2_lo) {  // within rounding of the cutoff: exact reference r^2
    if (r2 > P.cut2_hi) return 0;
    double ex = dx, ey = dy, ez = dz;
    if (FULL && c_full_flat[par][k] < 0)
      full_orient(P, make_double4(ax, ay, az, 0.0), j, make_double4(px, py, pz, 0.0), ex, ey, ez);
    if (exact_r2(ex, ey, ez) > P.cut2) return 0;
  }
  return r2 < P.guard_r2 ? 2 : 1;
}

// guard pairs (r below the first knot, overlaps): the reference-literal
// evaluation of eam_kernels.cu, out of the hot loop
__device__ __noinline__ double guard_rho(KP* P, long long d, int j, int tgt, double dx, double dy,
                                         double dz, int full) {
  const double r2x = exact_r2(dx, dy, dz);
  if (r2x < kOverlapR2) {
    report_overlap(*P, pair_key(*P, d, j, 0), P->tag[d], P->tag[tgt], r2x);
    return 0.0;
  }
  const double rho = pair_rho(*P, r2x);
  if (!full) red_add(&P->rho[tgt], rho);
  return rho;
}
__device__ __noinline__ bool guard_force(KP* P, long long d, int j, int tgt, double dx,
                                         double dy, double dz, double dfsum, int full,
                                         double* q) {
  const double r2x = exact_r2(dx, dy, dz);
  if (r2x < kOverlapR2) {
    report_overlap(*P, pair_key(*P, d, j, 1ull << 61), P->tag[d], P->tag[tgt], r2x);
    return false;
  }
  double fp, phi;
  pair_force(*P, r2x, dfsum, fp, phi);
  q[0] = -fp * dx;
  q[1] = -fp * dy;
  q[2] = -fp * dz;
  q[3] = phi;
  if (!full) {
    red_add(&P->frc[tgt], q[0]);
    red_add(&P->frc[P->S + tgt], q[1]);
    red_add(&P->frc[2 * P->S + tgt], q[2]);
  }
  return true;
}

// ------------------------------------------------------------------ density
// one skin candidate that passed the fp32 filter (rare): full decision
template <bool FULL>
__device__ __forceinline__ double skin_density(const KP& P, KP* Pp, int par, int k, int d, int jj,
                                               int tw, double ax, double ay, double az,
                                               unsigned long long& m0, unsigned long long& m1) {
  double px, py, pz, w;
  ld256(P.pdf + jj, px, py, pz, w);
  const double dx = xsub(ax, px), dy = xsub(ay, py), dz = xsub(az, pz);
  const double r2 = fma(dz, dz, fma(dy, dy, dx * dx));
  const int stt = decide<FULL>(P, par, k, jj, ax, ay, az, px, py, pz, dx, dy, dz, r2);
  if (!stt) return 0.0;
  const int to = tw < 0 ? jj : tw;
  if (stt == 2) {
    m1 |= kGuardBit;
    return guard_rho(Pp, d, jj, to, dx, dy, dz, FULL);
  }
  set_bit(m0, m1, k);
  double s;
  const int sg = seg_index(P.fd, r2 * rsqrt(r2), s);
  double A, Bc, Cc, D;
  ld256(P.fd.rec + 4 * (size_t)sg, A, Bc, Cc, D);
  const double rho = fma(fma(fma(A, s, Bc), s, Cc), s, D);
  if (!FULL) red_add(&P.rho[to], rho);
  return rho;
}

// 32-byte density records staged in shared memory: chunk c of record i at
// 16-byte slot 2 i + (c ^ ((i >> 2) & 1)) (8 distinct bank quads for random i)
__device__ __forceinline__ int smem_slot32(int i, int c) { return 2 * i + (c ^ ((i >> 2) & 1)); }

template <bool FULL, int B, bool SMEM = false>
__device__ __forceinline__ void density_site(const KP& P, KP* Pp, int par, int d, bool live,
                                             const double2* T = nullptr, int seg_lo = 0) {
  const double4* __restrict__ pdf = P.pdf;
  const int* __restrict__ tgt = P.tgt;
  double ax = kVacant, ay = 0, az = 0, aw = 0;
  if (live) ld256(pdf + d, ax, ay, az, aw);
  if (ax >= kVacantTest) {
    if (FULL && live) P.rho[d] = 0.0;
    return;
  }
  const int n = FULL ? c_full_n[par] : c_half_n[par];
  const int nin = FULL ? c_full_nin[par] : c_half_nin[par];
  const int* offs = FULL ? c_full[par] : c_half[par];
  const double lo = P.cut2_lo, g2 = P.guard_r2;
  double acc = 0.0;
  unsigned long long m0 = 0, m1 = 0;
  // inner shells: direct fp64 gather, batched; the common case is decided
  // by one compare, the near-cutoff / guard cases drop to decide()
  for (int k0 = 0; k0 < nin; k0 += B) {
    int j[B], t[B], seg[B];
    bool in[B];
    double px[B], py[B], pz[B], s[B], r2[B];
#pragma unroll
    for (int b = 0; b < B; ++b) {
      j[b] = d + offs[min(k0 + b, nin - 1)];
      double w;
      ld256(pdf + j[b], px[b], py[b], pz[b], w);
      t[b] = __ldg(tgt + j[b]);
    }
    bool rare = false;
#pragma unroll
    for (int b = 0; b < B; ++b) {
      const double dx = xsub(ax, px[b]), dy = xsub(ay, py[b]), dz = xsub(az, pz[b]);
      r2[b] = fma(dz, dz, fma(dy, dy, dx * dx));
      const bool live_k = k0 + b < nin;
      in[b] = live_k && r2[b] <= lo && r2[b] >= g2;
      rare |= live_k && !in[b] && (r2[b] <= P.cut2_hi);
    }
    if (rare) {
#pragma unroll
      for (int b = 0; b < B; ++b) {
        if (in[b] || k0 + b >= nin || r2[b] > P.cut2_hi) continue;
        const double dx = xsub(ax, px[b]), dy = xsub(ay, py[b]), dz = xsub(az, pz[b]);
        const int st = decide<FULL>(P, par, k0 + b, j[b], ax, ay, az, px[b], py[b], pz[b], dx, dy,
                                    dz, r2[b]);
        if (st == 1) {
          in[b] = true;
        } else if (st == 2) {
          m1 |= kGuardBit;
          acc += guard_rho(Pp, d, j[b], t[b], dx, dy, dz, FULL);
        }
      }
    }
#pragma unroll
    for (int b = 0; b < B; ++b) seg[b] = seg_index(P.fd, r2[b] * rsqrt(r2[b]), s[b]);
    double tA[B], tB[B], tC[B], tD[B];
#pragma unroll
    for (int b = 0; b < B; ++b)
      if (in[b]) {
        const int li = seg[b] - seg_lo;
        if (SMEM && li >= 0) {
          const double2 c0 = T[smem_slot32(li, 0)], c1 = T[smem_slot32(li, 1)];
          tA[b] = c0.x;
          tB[b] = c0.y;
          tC[b] = c1.x;
          tD[b] = c1.y;
        } else {
          ld256(P.fd.rec + 4 * (size_t)seg[b], tA[b], tB[b], tC[b], tD[b]);
        }
      }
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
  // skin shells: fp32 filter, batched; a pass is rare
  const float4 af = make_float4((float)ax, (float)ay, (float)az, 0.f);
  const float hi = P.band_hi;
  for (int k0 = nin; k0 < n; k0 += 4) {
    float4 pf[4];
    int jj[4];
#pragma unroll
    for (int b = 0; b < 4; ++b) {
      jj[b] = d + offs[min(k0 + b, n - 1)];
      pf[b] = __ldg(P.uf + jj[b]);
    }
    bool any = false, pass[4];
#pragma unroll
    for (int b = 0; b < 4; ++b) {
      const float fx = af.x - pf[b].x, fy = af.y - pf[b].y, fz = af.z - pf[b].z;
      pass[b] = k0 + b < n && fmaf(fz, fz, fmaf(fy, fy, fx * fx)) <= hi;
      any |= pass[b];
    }
    if (any) {
#pragma unroll
      for (int b = 0; b < 4; ++b)
        if (pass[b])
          acc += skin_density<FULL>(P, Pp, par, k0 + b, d, jj[b], __float_as_int(pf[b].w), ax,
                                    ay, az, m0, m1);
    }
  }
  if (FULL) P.rho[d] = acc;
  else red_add(&P.rho[d], acc);
  if (P.pmask) {
    P.pmask[2 * (size_t)d] = m0;
    P.pmask[2 * (size_t)d + 1] = m1;
  }
}

// -------------------------------------------------------------------- force
struct PairOut {
  double qx, qy, qz, phi;
};

// -fp of forces.cpp:164 times d, and phi, from one 64-byte force record
__device__ __forceinline__ PairOut pair_eval(const double* rec, double s, double ri, double ih,
                                             double dfsum, double dx, double dy, double dz) {
  double zA, zB, zC, zD, qA, qB, qC, qD;
  ld256(rec, zA, zB, zC, zD);
  ld256(rec + 4, qA, qB, qC, qD);
  const double s15 = 1.5 * s, s2 = s + s;
  const double z = fma(fma(fma(zA, s, zB), s, zC), s, zD);
  const double zs = fma(fma(zA, s15, zB), s2, zC);  // dz/ds
  const double ps = fma(fma(qA, s15, qB), s2, qC);  // drho/ds
  PairOut o;
  o.phi = z * ri;
  // phi' = (z' - phi)/r;  -fp = ((dFa + dFp) rho' + phi')/r;  d/dr = ih d/ds
  const double dphi = fma(zs, ih, -o.phi) * ri;
  const double mfp = fma(dfsum * ps, ih, dphi) * ri;
  o.qx = mfp * dx;
  o.qy = mfp * dy;
  o.qz = mfp * dz;
  return o;
}

template <bool FULL, int B>
__device__ __forceinline__ double force_site(const KP& P, KP* Pp, int par, int d, bool live) {
  const double4* __restrict__ pdf = P.pdf;
  const int* __restrict__ tgt = P.tgt;
  const long long S = P.S;
  double ax = kVacant, ay = 0, az = 0, adf = 0;
  if (live) ld256(pdf + d, ax, ay, az, adf);
  if (ax >= kVacantTest) {
    if (FULL && live) {
      P.frc[d] = 0.0;
      P.frc[S + d] = 0.0;
      P.frc[2 * S + d] = 0.0;
    }
    return 0.0;
  }
  const int n = FULL ? c_full_n[par] : c_half_n[par];
  const int nin = FULL ? c_full_nin[par] : c_half_nin[par];
  const int* offs = FULL ? c_full[par] : c_half[par];
  const double ih = P.ff.ih;
  double fx = 0.0, fy = 0.0, fz = 0.0, e = 0.0;
  auto accumulate = [&](const PairOut& o, int to) {
    fx -= o.qx;
    fy -= o.qy;
    fz -= o.qz;
    if (FULL) {
      e = fma(0.5, o.phi, e);
    } else {
      e += o.phi;
      red_add(&P.frc[to], o.qx);
      red_add(&P.frc[S + to], o.qy);
      red_add(&P.frc[2 * S + to], o.qz);
    }
  };
  for (int k0 = 0; k0 < nin; k0 += B) {
    int j[B], t[B], st[B], seg[B];
    double px[B], py[B], pz[B], pw[B], dx[B], dy[B], dz[B], s[B], ri[B];
#pragma unroll
    for (int b = 0; b < B; ++b) {
      j[b] = d + offs[min(k0 + b, nin - 1)];
      ld256(pdf + j[b], px[b], py[b], pz[b], pw[b]);
      t[b] = __ldg(tgt + j[b]);
    }
#pragma unroll
    for (int b = 0; b < B; ++b) {
      dx[b] = xsub(ax, px[b]);
      dy[b] = xsub(ay, py[b]);
      dz[b] = xsub(az, pz[b]);
      const double r2 = fma(dz[b], dz[b], fma(dy[b], dy[b], dx[b] * dx[b]));
      st[b] = k0 + b < nin ? decide<FULL>(P, par, k0 + b, j[b], ax, ay, az, px[b], py[b], pz[b],
                                          dx[b], dy[b], dz[b], r2)
                           : 0;
      if (st[b] == 2) {
        double q[4];
        if (guard_force(Pp, d, j[b], t[b], dx[b], dy[b], dz[b], adf + pw[b], FULL, q)) {
          fx -= q[0];
          fy -= q[1];
          fz -= q[2];
          e = FULL ? fma(0.5, q[3], e) : e + q[3];
        }
        st[b] = 0;
      }
      ri[b] = rsqrt(r2);
      seg[b] = seg_index(P.ff, r2 * ri[b], s[b]);
    }
#pragma unroll
    for (int b = 0; b < B; ++b) {
      if (!st[b]) continue;
      accumulate(pair_eval(P.ff.rec + 8 * (size_t)seg[b], s[b], ri[b], ih, adf + pw[b], dx[b],
                           dy[b], dz[b]),
                 t[b]);
    }
  }
  const float4 af = make_float4((float)ax, (float)ay, (float)az, 0.f);
  for (int k = nin; k < n; ++k) {
    const int jj = d + offs[k];
    const float4 pf = __ldg(P.uf + jj);
    const float gx = af.x - pf.x, gy = af.y - pf.y, gz = af.z - pf.z;
    if (fmaf(gz, gz, fmaf(gy, gy, gx * gx)) > P.band_hi) continue;
    double px, py, pz, pw;
    ld256(pdf + jj, px, py, pz, pw);
    const double ddx = xsub(ax, px), ddy = xsub(ay, py), ddz = xsub(az, pz);
    const double r2 = fma(ddz, ddz, fma(ddy, ddy, ddx * ddx));
    const int stt = decide<FULL>(P, par, k, jj, ax, ay, az, px, py, pz, ddx, ddy, ddz, r2);
    if (!stt) continue;
    const int tw = __float_as_int(pf.w);
    const int to = tw < 0 ? jj : tw;
    if (stt == 2) {
      double q[4];
      if (guard_force(Pp, d, jj, to, ddx, ddy, ddz, adf + pw, FULL, q)) {
        fx -= q[0];
        fy -= q[1];
        fz -= q[2];
        e = FULL ? fma(0.5, q[3], e) : e + q[3];
      }
      continue;
    }
    const double ri = rsqrt(r2);
    double s;
    const int sg = seg_index(P.ff, r2 * ri, s);
    accumulate(pair_eval(P.ff.rec + 8 * (size_t)sg, s, ri, ih, adf + pw, ddx, ddy, ddz), to);
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

// the force pass replaying the density pass's pair mask: no candidate
// filtering or cutoff decisions, only the in-cutoff pairs, two at a time
template <bool FULL>
__device__ __forceinline__ double force_site_mask(const KP& P, KP* Pp, int par, int d,
                                                  bool live) {
  const double4* __restrict__ pdf = P.pdf;
  const int* __restrict__ tgt = P.tgt;
  const long long S = P.S;
  double ax = kVacant, ay = 0, az = 0, adf = 0;
  if (live) ld256(pdf + d, ax, ay, az, adf);
  if (ax >= kVacantTest) {
    if (FULL && live) {
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
    int j[2], t[2], seg[2];
    double px[2], py[2], pz[2], pw[2], dx[2], dy[2], dz[2], s[2], ri[2];
#pragma unroll
    for (int b = 0; b < 2; ++b) {
      j[b] = d + offs[k[b]];
      ld256(pdf + j[b], px[b], py[b], pz[b], pw[b]);
      t[b] = __ldg(tgt + j[b]);
    }
#pragma unroll
    for (int b = 0; b < 2; ++b) {
      dx[b] = xsub(ax, px[b]);
      dy[b] = xsub(ay, py[b]);
      dz[b] = xsub(az, pz[b]);
      const double r2 = fma(dz[b], dz[b], fma(dy[b], dy[b], dx[b] * dx[b]));
      ri[b] = rsqrt(r2);
      seg[b] = seg_index(P.ff, r2 * ri[b], s[b]);
#ifdef CBX_DEBUG_BOUNDS
      if (j[b] < 0 || j[b] >= S || seg[b] < 0 || seg[b] > P.ff.nseg) {
        printf("force_mask oob: d=%d par=%d k=%d j=%d seg=%d r2=%g v=%d m=%llx %llx\n", d, par,
               k[b], j[b], seg[b], r2, (int)v[b], P.pmask[2 * (size_t)d],
               P.pmask[2 * (size_t)d + 1]);
        seg[b] = 0;
        j[b] = d;
      }
#endif
    }
    double zA[2], zB[2], zC[2], zD[2], qA[2], qB[2], qC[2], qD[2];
#pragma unroll
    for (int b = 0; b < 2; ++b) {
      const double* rec = P.ff.rec + 8 * (size_t)((P.xp & 1) ? 2000 + (k[b] & 7) : seg[b]);
      ld256(rec, zA[b], zB[b], zC[b], zD[b]);
      ld256(rec + 4, qA[b], qB[b], qC[b], qD[b]);
    }
#pragma unroll
    for (int b = 0; b < 2; ++b) {
      const double sb = s[b], s15 = 1.5 * sb, s2 = sb + sb;
      const double z = fma(fma(fma(zA[b], sb, zB[b]), sb, zC[b]), sb, zD[b]);
      const double zs = fma(fma(zA[b], s15, zB[b]), s2, zC[b]);  // dz/ds
      const double ps = fma(fma(qA[b], s15, qB[b]), s2, qC[b]);  // drho/ds
      const double phi = z * ri[b];
      // phi' = (z' - phi)/r;  -fp = ((dFa + dFp) rho' + phi')/r;  d/dr = ih d/ds
      const double dphi = fma(zs, ih, -phi) * ri[b];
      const double mfp = v[b] ? fma((adf + pw[b]) * ps, ih, dphi) * ri[b] : 0.0;
      const double qx = mfp * dx[b], qy = mfp * dy[b], qz = mfp * dz[b];
      fx -= qx;
      fy -= qy;
      fz -= qz;
      if (FULL) {
        e = fma(0.5, v[b] ? phi : 0.0, e);
      } else if (v[b]) {
        e += phi;
        if (!(P.xp & 2)) {
          red_add(&P.frc[t[b]], qx);
          red_add(&P.frc[S + t[b]], qy);
          red_add(&P.frc[2 * S + t[b]], qz);
        }
      }
    }
  }
  if (guard) {  // the guard pairs skipped by the density pass's mask
    const int n = FULL ? c_full_n[par] : c_half_n[par];
    for (int kk = 0; kk < n; ++kk) {
      const int jj = d + offs[kk];
      double px, py, pz, pw;
      ld256(pdf + jj, px, py, pz, pw);
      const double ddx = xsub(ax, px), ddy = xsub(ay, py), ddz = xsub(az, pz);
      const double r2 = fma(ddz, ddz, fma(ddy, ddy, ddx * ddx));
      if (decide<FULL>(P, par, kk, jj, ax, ay, az, px, py, pz, ddx, ddy, ddz, r2) != 2) continue;
      double q[4];
      if (guard_force(Pp, d, jj, __ldg(tgt + jj), ddx, ddy, ddz, adf + pw, FULL, q)) {
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

// masked offsets of the current pass staged per CTA (LDS instead of an
// indexed constant load); file scope so the address space is static
__shared__ int g_soffs[2][kMaskBits + 1];

// 64-byte spline records staged in shared memory: chunk c of record i at
// 16-byte slot 4 i + (c ^ ((i >> 1) & 3)).  A 128-byte wavefront serves 8
// distinct bank quads; record i lives in quad half (i & 1) and the XOR with
// bits 1-2 of i spreads chunk c of random records over all 8 quads.
__device__ __forceinline__ int smem_slot(int i, int c) { return 4 * i + (c ^ ((i >> 1) & 3)); }
__device__ __forceinline__ double2 smem_chunk(const double2* T, int i, int c) {
  return T[smem_slot(i, c)];
}

// 1/sqrt for r^2 in the normal range: the hardware approximation plus two
// Newton steps (relative error a few ulp, no special-case branch)
__device__ __forceinline__ double rsqrt_nr(double x) {
  double y;
  asm("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(x));
  const double h = 0.5 * x;
  y = y * fma(-h * y, y, 1.5);
  y = y * fma(-h * y, y, 1.5);
  return y;
}

// force pass, warp-uniform sweep: the warp walks the union of its lanes'
// pair masks, so at every step all lanes evaluate the same offset k --
// partner loads of a brick row are contiguous, the spline records of the
// lanes are the same or adjacent segments (one or two L1 lines instead of
// one line per lane), and offs[k] is a uniform constant load.  A lane whose
// own mask lacks k is predicated off (in a thermal lattice the union is
// nearly the intersection: the in-cutoff set is the same for every site).
__device__ __forceinline__ unsigned long long warp_or64(unsigned long long m) {
  const unsigned lo = __reduce_or_sync(0xffffffffu, (unsigned)m);
  const unsigned hi = __reduce_or_sync(0xffffffffu, (unsigned)(m >> 32));
  return ((unsigned long long)hi << 32) | lo;
}

template <bool FULL, int B>
__device__ __forceinline__ double force_site_union(const KP& P, KP* Pp, const int* s_offs,
                                                   int par, int d, bool live) {
  const double4* __restrict__ pdf = P.pdf;
  const int* __restrict__ tgt = P.tgt;
  const long long S = P.S;
  double ax = kVacant, ay = 0, az = 0, adf = 0;
  if (live) ld256(pdf + d, ax, ay, az, adf);
  const bool occ = ax < kVacantTest;
  if (!occ && FULL && live) {
    P.frc[d] = 0.0;
    P.frc[S + d] = 0.0;
    P.frc[2 * S + d] = 0.0;
  }
  unsigned long long m0 = 0, m1 = 0;
  if (occ) {
    m0 = P.pmask[2 * (size_t)d];
    m1 = P.pmask[2 * (size_t)d + 1];
  }
  const bool guard = (m1 & kGuardBit) != 0;
  m1 &= ~kGuardBit;
  unsigned long long u0 = warp_or64(m0), u1 = warp_or64(m1);
  const double ih = P.ff.ih;
  const double r2_idle = P.cut2_lo;  // an in-table distance for idle lanes
  double* __restrict__ fxp = P.frc;
  double* __restrict__ fyp = P.frc + S;
  double* __restrict__ fzp = P.frc + 2 * S;
  double fx = 0.0, fy = 0.0, fz = 0.0, e = 0.0;
  while (u0 | u1) {
    int k[B];
    bool v[B];
#pragma unroll
    for (int b = 0; b < B; ++b) {
      bool any = true;
      if (u0) {
        k[b] = __ffsll(u0) - 1;
        u0 &= u0 - 1;
      } else if (u1) {
        k[b] = 63 + __ffsll(u1);
        u1 &= u1 - 1;
      } else {
        k[b] = 0;
        any = false;
      }
      v[b] = any && (k[b] < 64 ? (m0 >> k[b]) & 1 : (m1 >> (k[b] - 64)) & 1);
    }
    // idle lanes read their own site (a valid, cached address) and a
    // valid table row; their results are discarded
    int j[B], t[B], seg[B];
    double px[B], py[B], pz[B], pw[B], s[B], ri[B];
#pragma unroll
    for (int b = 0; b < B; ++b) {
      j[b] = v[b] ? d + s_offs[k[b]] : d;
      ld256(pdf + j[b], px[b], py[b], pz[b], pw[b]);
      t[b] = __ldg(tgt + j[b]);
    }
    double dx[B], dy[B], dz[B];
#pragma unroll
    for (int b = 0; b < B; ++b) {
      dx[b] = xsub(ax, px[b]);
      dy[b] = xsub(ay, py[b]);
      dz[b] = xsub(az, pz[b]);
      double r2 = fma(dz[b], dz[b], fma(dy[b], dy[b], dx[b] * dx[b]));
      r2 = v[b] ? r2 : r2_idle;
      ri[b] = rsqrt(r2);
      seg[b] = seg_index(P.ff, r2 * ri[b], s[b]);
    }
    double zA[B], zB[B], zC[B], zD[B], qA[B], qB[B], qC[B], qD[B];
#pragma unroll
    for (int b = 0; b < B; ++b) {
      const double* rec = P.ff.rec + 8 * (size_t)seg[b];
      ld256(rec, zA[b], zB[b], zC[b], zD[b]);
      ld256(rec + 4, qA[b], qB[b], qC[b], qD[b]);
    }
#pragma unroll
    for (int b = 0; b < B; ++b) {
      const double sb = s[b], s15 = 1.5 * sb, s2 = sb + sb;
      const double z = fma(fma(fma(zA[b], sb, zB[b]), sb, zC[b]), sb, zD[b]);
      const double zs = fma(fma(zA[b], s15, zB[b]), s2, zC[b]);  // dz/ds
      const double ps = fma(fma(qA[b], s15, qB[b]), s2, qC[b]);  // drho/ds
      const double phi = v[b] ? z * ri[b] : 0.0;
      // phi' = (z' - phi)/r;  -fp = ((dFa + dFp) rho' + phi')/r;  d/dr = ih d/ds
      const double dphi = fma(zs, ih, -phi) * ri[b];
      const double mfp = v[b] ? fma((adf + pw[b]) * ps, ih, dphi) * ri[b] : 0.0;
      const double qx = mfp * dx[b], qy = mfp * dy[b], qz = mfp * dz[b];
      fx -= qx;
      fy -= qy;
      fz -= qz;
      if (FULL) {
        e = fma(0.5, phi, e);
      } else {
        e += phi;
        if (v[b]) {
          red_add(fxp + t[b], qx);
          red_add(fyp + t[b], qy);
          red_add(fzp + t[b], qz);
        }
      }
    }
  }
  const int* offs = FULL ? c_full[par] : c_half[par];
  if (guard) {  // the guard pairs skipped by the density pass's mask
    const int n = FULL ? c_full_n[par] : c_half_n[par];
    for (int kk = 0; kk < n; ++kk) {
      const int jj = d + offs[kk];
      double px, py, pz, pw;
      ld256(pdf + jj, px, py, pz, pw);
      const double ddx = xsub(ax, px), ddy = xsub(ay, py), ddz = xsub(az, pz);
      const double r2 = fma(ddz, ddz, fma(ddy, ddy, ddx * ddx));
      if (decide<FULL>(P, par, kk, jj, ax, ay, az, px, py, pz, ddx, ddy, ddz, r2) != 2) continue;
      double q[4];
      if (guard_force(Pp, d, jj, __ldg(tgt + jj), ddx, ddy, ddz, adf + pw, FULL, q)) {
        fx -= q[0];
        fy -= q[1];
        fz -= q[2];
        e = FULL ? fma(0.5, q[3], e) : e + q[3];
      }
    }
  }
  if (occ) {
    if (FULL) {
      P.frc[d] = fx;
      P.frc[S + d] = fy;
      P.frc[2 * S + d] = fz;
    } else {
      red_add(&P.frc[d], fx);
      red_add(&P.frc[S + d], fy);
      red_add(&P.frc[2 * S + d], fz);
    }
  }
  return e;
}

// force pass, warp-uniform sweep, software-pipelined over three stages so
// both memory round trips of a pair overlap other pairs' arithmetic:
//   stage 1  partner load (pdf, owner) of pair n
//   stage 2  geometry of pair a (loaded last iteration) -> spline record load
//   stage 3  force of pair b (record loaded last iteration), partner REDs
// All control flow is warp-uniform (the union of the lanes' masks).
struct PipePartner {
  double px, py, pz, pw;
  int t;
  bool v;
};
struct PipePair {
  double dx, dy, dz, pw, s, ri;
  double zA, zB, zC, zD, qA, qB, qC, qD;
  int t;
  bool v;
};

template <bool FULL>
__device__ __forceinline__ double force_site_pipe(const KP& P, KP* Pp, int par, int d,
                                                  bool live) {
  const double4* __restrict__ pdf = P.pdf;
  const int* __restrict__ tgt = P.tgt;
  const long long S = P.S;
  double ax = kVacant, ay = 0, az = 0, adf = 0;
  if (live) ld256(pdf + d, ax, ay, az, adf);
  const bool occ = ax < kVacantTest;
  if (!occ && FULL && live) {
    P.frc[d] = 0.0;
    P.frc[S + d] = 0.0;
    P.frc[2 * S + d] = 0.0;
  }
  unsigned long long m0 = 0, m1 = 0;
  if (occ) {
    m0 = P.pmask[2 * (size_t)d];
    m1 = P.pmask[2 * (size_t)d + 1];
  }
  const bool guard = (m1 & kGuardBit) != 0;
  m1 &= ~kGuardBit;
  unsigned long long u0 = warp_or64(m0), u1 = warp_or64(m1);
  const double ih = P.ff.ih;
  const double r2_idle = P.cut2_lo;  // an in-table distance for idle lanes
  double* __restrict__ fxp = P.frc;
  double* __restrict__ fyp = P.frc + S;
  double* __restrict__ fzp = P.frc + 2 * S;
  double fx = 0.0, fy = 0.0, fz = 0.0, e = 0.0;

  // the union as 32-bit words, consumed from the lowest (uniform control)
  unsigned cu = (unsigned)u0, co = (unsigned)m0;
  unsigned pu1 = (unsigned)(u0 >> 32), po1 = (unsigned)(m0 >> 32);
  unsigned pu2 = (unsigned)u1, po2 = (unsigned)m1;
  unsigned pu3 = (unsigned)(u1 >> 32), po3 = (unsigned)(m1 >> 32);
  int base = 0;
  const int* s_offs = g_soffs[par];
  auto fetch = [&](PipePartner& q) -> bool {  // stage 1 (uniform result)
    while (cu == 0) {
      if (base == 96) return false;
      cu = pu1;
      co = po1;
      pu1 = pu2;
      po1 = po2;
      pu2 = pu3;
      po2 = po3;
      pu3 = 0;
      base += 32;
    }
    const int bit = __ffs(cu) - 1;
    cu &= cu - 1;
    const int k = base + bit;
    q.v = (co >> bit) & 1;
    const int j = q.v ? d + s_offs[(P.xp & 16) ? 0 : k] : d;  // idle lanes read their own site
    ld256(pdf + j, q.px, q.py, q.pz, q.pw);
    q.t = __ldg(tgt + j);
    return true;
  };
  auto geometry = [&](const PipePartner& q, PipePair& c) {  // stage 2
    c.v = q.v;
    c.t = q.t;
    c.pw = q.pw;
    c.dx = xsub(ax, q.px);
    c.dy = xsub(ay, q.py);
    c.dz = xsub(az, q.pz);
    double r2 = fma(c.dz, c.dz, fma(c.dy, c.dy, c.dx * c.dx));
    r2 = c.v ? r2 : r2_idle;
    c.ri = rsqrt_nr(r2);
    const int seg = seg_index(P.ff, r2 * c.ri, c.s);
    const double* rec = P.ff.rec + 8 * (size_t)((P.xp & 32) ? 100 : seg);
    ld256(rec, c.zA, c.zB, c.zC, c.zD);
    ld256(rec + 4, c.qA, c.qB, c.qC, c.qD);
  };
  auto finish = [&](const PipePair& b) {  // stage 3
    const double sb = b.s, s15 = 1.5 * sb, s2 = sb + sb;
    const double z = fma(fma(fma(b.zA, sb, b.zB), sb, b.zC), sb, b.zD);
    const double zs = fma(fma(b.zA, s15, b.zB), s2, b.zC);  // dz/ds
    const double ps = fma(fma(b.qA, s15, b.qB), s2, b.qC);  // drho/ds
    const double phi = b.v ? z * b.ri : 0.0;
    // phi' = (z' - phi)/r;  -fp = ((dFa + dFp) rho' + phi')/r;  d/dr = ih d/ds
    const double dphi = fma(zs, ih, -phi) * b.ri;
    const double mfp = b.v ? fma((adf + b.pw) * ps, ih, dphi) * b.ri : 0.0;
    const double qx = mfp * b.dx, qy = mfp * b.dy, qz = mfp * b.dz;
    fx -= qx;
    fy -= qy;
    fz -= qz;
    if (FULL) {
      e = fma(0.5, phi, e);
    } else {
      e += phi;
      if (b.v && !(P.xp & 2)) {
        red_add(fxp + b.t, qx);
        red_add(fyp + b.t, qy);
        red_add(fzp + b.t, qz);
      }
    }
  };

  PipePartner a, n;
  PipePair b;
  bool a_ok = fetch(a), b_ok = false;
  // order inside an iteration: issue the next partner load, finish the
  // pair whose record arrived, then start the record load of the pair
  // whose partner arrived -- one PipePair live at a time
  while (a_ok || b_ok) {
    const bool n_ok = fetch(n);
    if (b_ok) finish(b);
    b_ok = a_ok;
    if (a_ok) geometry(a, b);
    a = n;
    a_ok = n_ok;
  }
  const int* offs = FULL ? c_full[par] : c_half[par];
  if (guard) {  // the guard pairs skipped by the density pass's mask
    const int n = FULL ? c_full_n[par] : c_half_n[par];
    for (int kk = 0; kk < n; ++kk) {
      const int jj = d + offs[kk];
      double px, py, pz, pw;
      ld256(pdf + jj, px, py, pz, pw);
      const double ddx = xsub(ax, px), ddy = xsub(ay, py), ddz = xsub(az, pz);
      const double r2 = fma(ddz, ddz, fma(ddy, ddy, ddx * ddx));
      if (decide<FULL>(P, par, kk, jj, ax, ay, az, px, py, pz, ddx, ddy, ddz, r2) != 2) continue;
      double q[4];
      if (guard_force(Pp, d, jj, __ldg(tgt + jj), ddx, ddy, ddz, adf + pw, FULL, q)) {
        fx -= q[0];
        fy -= q[1];
        fz -= q[2];
        e = FULL ? fma(0.5, q[3], e) : e + q[3];
      }
    }
  }
  if (occ) {
    if (FULL) {
      P.frc[d] = fx;
      P.frc[S + d] = fy;
      P.frc[2 * S + d] = fz;
    } else {
      red_add(&P.frc[d], fx);
      red_add(&P.frc[S + d], fy);
      red_add(&P.frc[2 * S + d], fz);
    }
  }
  return e;
}

// force pass, lean variant: one pair per iteration, no batching, so the
// register footprint allows 6-8 resident CTAs per SM (latency hidden by
// warps instead of by in-thread batching).  Warp-uniform union sweep.
template <bool FULL, bool SMEM>
__device__ __forceinline__ double force_site_lean(const KP& P, KP* Pp, int par, int d,
                                                  bool live, const double2* T = nullptr,
                                                  int seg_lo = 0) {
  const double4* __restrict__ pdf = P.pdf;
  const int* __restrict__ tgt = P.tgt;
  const long long S = P.S;
  double ax = kVacant, ay = 0, az = 0, adf = 0;
  if (live) ld256(pdf + d, ax, ay, az, adf);
  const bool occ = ax < kVacantTest;
  if (!occ && FULL && live) {
    P.frc[d] = 0.0;
    P.frc[S + d] = 0.0;
    P.frc[2 * S + d] = 0.0;
  }
  unsigned long long m0 = 0, m1 = 0;
  if (occ) {
    m0 = P.pmask[2 * (size_t)d];
    m1 = P.pmask[2 * (size_t)d + 1];
  }
  const bool guard = (m1 & kGuardBit) != 0;
  m1 &= ~kGuardBit;
  const unsigned long long u0 = warp_or64(m0), u1 = warp_or64(m1);
  unsigned cu = (unsigned)u0, co = (unsigned)m0;
  unsigned pu1 = (unsigned)(u0 >> 32), po1 = (unsigned)(m0 >> 32);
  unsigned pu2 = (unsigned)u1, po2 = (unsigned)m1;
  unsigned pu3 = (unsigned)(u1 >> 32), po3 = (unsigned)(m1 >> 32);
  int base = 0;
  const int* s_offs = g_soffs[par];
  const double ih = P.ff.ih;
  const double r2_idle = P.cut2_lo;
  double fx = 0.0, fy = 0.0, fz = 0.0, e = 0.0;
  for (;;) {
    while (cu == 0) {
      if (base == 96) break;
      cu = pu1;
      co = po1;
      pu1 = pu2;
      po1 = po2;
      pu2 = pu3;
      po2 = po3;
      pu3 = 0;
      base += 32;
    }
    if (cu == 0) break;
    const int bit = __ffs(cu) - 1;
    cu &= cu - 1;
    const bool v = (co >> bit) & 1;
    const int j = v ? d + s_offs[(P.xp & 16) ? 0 : base + bit] : d;
    double px, py, pz, pw;
    ld256(pdf + j, px, py, pz, pw);
    const int t = __ldg(tgt + j);
    const double dx = xsub(ax, px), dy = xsub(ay, py), dz = xsub(az, pz);
    double r2 = fma(dz, dz, fma(dy, dy, dx * dx));
    r2 = v ? r2 : r2_idle;
    const double ri = rsqrt_nr(r2);
    double sb;
    const int seg = seg_index(P.ff, r2 * ri, sb);
    double zA, zB, zC, zD, qA, qB, qC, qD;
    const int li = seg - seg_lo;
    if (SMEM && li >= 0) {
      const double2 c0 = smem_chunk(T, li, 0), c1 = smem_chunk(T, li, 1);
      const double2 c2 = smem_chunk(T, li, 2), c3 = smem_chunk(T, li, 3);
      zA = c0.x; zB = c0.y; zC = c1.x; zD = c1.y;
      qA = c2.x; qB = c2.y; qC = c3.x; qD = c3.y;
    } else {
      const double* rec = P.ff.rec + 8 * (size_t)seg;
      ld256(rec, zA, zB, zC, zD);
      ld256(rec + 4, qA, qB, qC, qD);
    }
    const double s15 = 1.5 * sb, s2 = sb + sb;
    const double z = fma(fma(fma(zA, sb, zB), sb, zC), sb, zD);
    const double zs = fma(fma(zA, s15, zB), s2, zC);  // dz/ds
    const double ps = fma(fma(qA, s15, qB), s2, qC);  // drho/ds
    const double phi = v ? z * ri : 0.0;
    const double dphi = fma(zs, ih, -phi) * ri;
    const double mfp = v ? fma((adf + pw) * ps, ih, dphi) * ri : 0.0;
    const double qx = mfp * dx, qy = mfp * dy, qz = mfp * dz;
    fx -= qx;
    fy -= qy;
    fz -= qz;
    if (FULL) {
      e = fma(0.5, phi, e);
    } else {
      e += phi;
      if (v && !(P.xp & 2)) {
        red_add(&P.frc[t], qx);
        red_add(&P.frc[S + t], qy);
        red_add(&P.frc[2 * S + t], qz);
      }
    }
  }
  const int* offs = FULL ? c_full[par] : c_half[par];
  if (guard) {  // the guard pairs skipped by the density pass's mask
    const int n = FULL ? c_full_n[par] : c_half_n[par];
    for (int kk = 0; kk < n; ++kk) {
      const int jj = d + offs[kk];
      double px, py, pz, pw;
      ld256(pdf + jj, px, py, pz, pw);
      const double ddx = xsub(ax, px), ddy = xsub(ay, py), ddz = xsub(az, pz);
      const double r2 = fma(ddz, ddz, fma(ddy, ddy, ddx * ddx));
      if (decide<FULL>(P, par, kk, jj, ax, ay, az, px, py, pz, ddx, ddy, ddz, r2) != 2) continue;
      double q[4];
      if (guard_force(Pp, d, jj, __ldg(tgt + jj), ddx, ddy, ddz, adf + pw, FULL, q)) {
        fx -= q[0];
        fy -= q[1];
        fz -= q[2];
        e = FULL ? fma(0.5, q[3], e) : e + q[3];
      }
    }
  }
  if (occ) {
    if (FULL) {
      P.frc[d] = fx;
      P.frc[S + d] = fy;
      P.frc[2 * S + d] = fz;
    } else {
      red_add(&P.frc[d], fx);
      red_add(&P.frc[S + d], fy);
      red_add(&P.frc[2 * S + d], fz);
    }
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

__device__ __forceinline__ bool brick_site(const Geo& G, int brick, int par, int& d) {
  const int nbx = (G.bx + kBrickX - 1) / kBrickX, nby = (G.by + kBrickY - 1) / kBrickY;
  const int bxi = brick % nbx, r = brick / nbx;
  const int byi = r % nby, bzi = r / nby;
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int cx = bxi * kBrickX + (lane & 7), cy = byi * kBrickY + (lane >> 3),
            cz = bzi * kBrickZ + w;
  const bool live = cx < G.bx && cy < G.by && cz < G.bz;
  d = live ? (int)(par * G.NC + cell_of(cx + G.g, cy + G.g, cz + G.g, G)) : 0;
  return live;
}

__host__ __device__ __forceinline__ int brick_count(const Geo& G) {
  return ((G.bx + kBrickX - 1) / kBrickX) * ((G.by + kBrickY - 1) / kBrickY) *
         ((G.bz + kBrickZ - 1) / kBrickZ);
}

// blocks [nsb, grid) run the clash-record pass of the same phase (Newton-3
// only: every update is an atomic add, so it may overlap the slot sweep)
constexpr int kClashBlocks128 = 32;

// groups of 128 threads (4 warps) of a large CTA, each on its own brick
__device__ __forceinline__ int next_brick_group8(int* ctr, int group, volatile int* slot) {
  asm volatile("bar.sync %0, 128;" ::"r"(group + 1));
  if ((threadIdx.x & 127) == 0) slot[group] = atomicAdd(ctr, 1);
  asm volatile("bar.sync %0, 128;" ::"r"(group + 1));
  return slot[group];
}

// density pass with the upper rho-spline window in shared memory (32-byte
// records): 512 threads = 4 groups of 4 warps, one CTA per SM
constexpr int kDensTabRecords = 3300;  // x 32 B = 105,600 B
template <bool FULL, int B, int NT>
__global__ void __launch_bounds__(NT, 1) k_density_smem(KP P, int nsb) {
  if (blockIdx.x >= nsb) {
    clash_body<0>(P, blockIdx.x - nsb, gridDim.x - nsb);
    return;
  }
  if (P.st->err) return;
  extern __shared__ __align__(16) unsigned char smem_tab[];
  __shared__ int s_slot[NT / 128];
  double2* T = reinterpret_cast<double2*>(smem_tab);
  const int nseg = P.fd.nseg;
  const int seg_lo = max(0, nseg + 1 - kDensTabRecords);
  const int nrec = nseg + 1 - seg_lo;
  const double2* src = reinterpret_cast<const double2*>(P.fd.rec + 4 * (size_t)seg_lo);
  for (int q = threadIdx.x; q < 2 * nrec; q += blockDim.x) T[smem_slot32(q >> 1, q & 1)] = __ldg(src + q);
  __syncthreads();
  const int group = threadIdx.x >> 7;
  const int lt = threadIdx.x & 127, lane = lt & 31, w = lt >> 5;
  const Geo& G = P.G;
  const int nbx = (G.bx + kBrickX - 1) / kBrickX, nby = (G.by + kBrickY - 1) / kBrickY;
  const int nb = brick_count(G);
  for (;;) {
    const int b = next_brick_group8(&P.work[0], group, s_slot);
    if (b >= nb) break;
    const int cx = (b % nbx) * kBrickX + (lane & 7), cy = ((b / nbx) % nby) * kBrickY + (lane >> 3),
              cz = (b / (nbx * nby)) * kBrickZ + w;
    const bool live = cx < G.bx && cy < G.by && cz < G.bz;
    const int c = live ? (int)cell_of(cx + G.g, cy + G.g, cz + G.g, G) : 0;
    for (int par = 0; par < 2; ++par)
      density_site<FULL, B, true>(P, P.dself, par, live ? (int)(par * G.NC + c) : 0, live, T,
                                  seg_lo);
  }
}

template <bool FULL, int B, int MINB>
__global__ void __launch_bounds__(128, MINB) k_density_fast(KP P, int nsb) {
  if (blockIdx.x >= nsb) {
    clash_body<0>(P, blockIdx.x - nsb, gridDim.x - nsb);
    return;
  }
  if (P.st->err) return;
  const int nb = brick_count(P.G);
  for (;;) {
    const int b = next_brick(&P.work[0]);
    if (b >= nb) break;
    for (int par = 0; par < 2; ++par) {
      int d;
      const bool live = brick_site(P.G, b, par, d);
      density_site<FULL, B>(P, P.dself, par, d, live);
    }
  }
}

template <bool FULL, int B>
__global__ void __launch_bounds__(128, 4) k_force_fast(KP P) {
  zero_pair_tail(P, gridDim.x * blockDim.x / 32);
  if (P.st->err || P.st->n_ovl) return;
  const int nb = brick_count(P.G);
  double e = 0.0;
  for (;;) {
    const int b = next_brick(&P.work[1]);
    if (b >= nb) break;
    for (int par = 0; par < 2; ++par) {
      int d;
      const bool live = brick_site(P.G, b, par, d);
      e += force_site<FULL, B>(P, P.dself, par, d, live);
    }
  }
  for (int o = 16; o > 0; o >>= 1) e += __shfl_xor_sync(0xffffffffu, e, o);
  if ((threadIdx.x & 31) == 0) P.part_pair[(blockIdx.x * blockDim.x + threadIdx.x) >> 5] = e;
}

// lean force pass with the upper spline window (records [seg_lo, nseg])
// in shared memory: 1024 threads, one CTA per SM, 8 groups of 4 warps each
// on their own brick.  Pairs below the window (cascade cores) read global.
constexpr int kLeanTabRecords = 3300;  // x 64 B = 211,200 B

template <bool FULL, int NT>
__global__ void __launch_bounds__(NT, 1) k_force_lean_smem(KP P, int nsb) {
  zero_pair_tail(P, nsb * blockDim.x / 32);
  if (blockIdx.x >= nsb) {
    clash_body<1>(P, blockIdx.x - nsb, gridDim.x - nsb);
    return;
  }
  if (P.st->err || P.st->n_ovl) return;
  extern __shared__ __align__(16) unsigned char smem_tab[];
  __shared__ int s_slot[8];
  double2* T = reinterpret_cast<double2*>(smem_tab);
  const int nseg = P.ff.nseg;  // records 0..nseg (padded)
  const int seg_lo = max(0, nseg + 1 - kLeanTabRecords);
  const int nrec = nseg + 1 - seg_lo;
  const double2* src = reinterpret_cast<const double2*>(P.ff.rec + 8 * (size_t)seg_lo);
  for (int q = threadIdx.x; q < 4 * nrec; q += blockDim.x)
    T[smem_slot(q >> 2, q & 3)] = __ldg(src + q);
  for (int i = threadIdx.x; i < 2 * (kMaskBits + 1); i += blockDim.x) {
    const int par = i / (kMaskBits + 1), k = i % (kMaskBits + 1);
    const int n = FULL ? c_full_n[par] : c_half_n[par];
    g_soffs[par][k] = k < n ? (FULL ? c_full[par][k] : c_half[par][k]) : 0;
  }
  __syncthreads();
  const int group = threadIdx.x >> 7;
  const int lt = threadIdx.x & 127, lane = lt & 31, w = lt >> 5;
  const Geo& G = P.G;
  const int nbx = (G.bx + kBrickX - 1) / kBrickX, nby = (G.by + kBrickY - 1) / kBrickY;
  const int nb = brick_count(G);
  double e = 0.0;
  for (;;) {
    const int b = next_brick_group8(&P.work[1], group, s_slot);
    if (b >= nb) break;
    const int cx = (b % nbx) * kBrickX + (lane & 7), cy = ((b / nbx) % nby) * kBrickY + (lane >> 3),
              cz = (b / (nbx * nby)) * kBrickZ + w;
    const bool live = cx < G.bx && cy < G.by && cz < G.bz;
    const int c = live ? (int)cell_of(cx + G.g, cy + G.g, cz + G.g, G) : 0;
    for (int par = 0; par < 2; ++par)
      e += force_site_lean<FULL, true>(P, P.dself, par, live ? (int)(par * G.NC + c) : 0, live,
                                       T, seg_lo);
  }
  for (int o = 16; o > 0; o >>= 1) e += __shfl_xor_sync(0xffffffffu, e, o);
  if ((threadIdx.x & 31) == 0) P.part_pair[(blockIdx.x * blockDim.x + threadIdx.x) >> 5] = e;
}

template <bool FULL, int MINB>
__global__ void __launch_bounds__(128, MINB) k_force_lean(KP P, int nsb) {
  zero_pair_tail(P, nsb * blockDim.x / 32);
  if (blockIdx.x >= nsb) {
    clash_body<1>(P, blockIdx.x - nsb, gridDim.x - nsb);
    return;
  }
  if (P.st->err || P.st->n_ovl) return;
  for (int i = threadIdx.x; i < 2 * (kMaskBits + 1); i += blockDim.x) {
    const int par = i / (kMaskBits + 1), k = i % (kMaskBits + 1);
    const int n = FULL ? c_full_n[par] : c_half_n[par];
    g_soffs[par][k] = k < n ? (FULL ? c_full[par][k] : c_half[par][k]) : 0;
  }
  __syncthreads();
  const int nb = brick_count(P.G);
  double e = 0.0;
  for (;;) {
    const int b = next_brick(&P.work[1]);
    if (b >= nb) break;
    for (int par = 0; par < 2; ++par) {
      int d;
      const bool live = brick_site(P.G, b, par, d);
      e += force_site_lean<FULL, false>(P, P.dself, par, d, live);
    }
  }
  for (int o = 16; o > 0; o >>= 1) e += __shfl_xor_sync(0xffffffffu, e, o);
  if ((threadIdx.x & 31) == 0) P.part_pair[(blockIdx.x * blockDim.x + threadIdx.x) >> 5] = e;
}

template <bool FULL>
__global__ void __launch_bounds__(128, 4) k_force_pipe(KP P, int nsb) {
  zero_pair_tail(P, nsb * blockDim.x / 32);
  if (blockIdx.x >= nsb) {
    clash_body<1>(P, blockIdx.x - nsb, gridDim.x - nsb);
    return;
  }
  if (P.st->err || P.st->n_ovl) return;
  for (int i = threadIdx.x; i < 2 * (kMaskBits + 1); i += blockDim.x) {
    const int par = i / (kMaskBits + 1), k = i % (kMaskBits + 1);
    const int n = FULL ? c_full_n[par] : c_half_n[par];
    g_soffs[par][k] = k < n ? (FULL ? c_full[par][k] : c_half[par][k]) : 0;
  }
  __syncthreads();
  const int nb = brick_count(P.G);
  double e = 0.0;
  for (;;) {
    const int b = next_brick(&P.work[1]);
    if (b >= nb) break;
    for (int par = 0; par < 2; ++par) {
      int d;
      const bool live = brick_site(P.G, b, par, d);
      e += force_site_pipe<FULL>(P, P.dself, par, d, live);
    }
  }
  for (int o = 16; o > 0; o >>= 1) e += __shfl_xor_sync(0xffffffffu, e, o);
  if ((threadIdx.x & 31) == 0) P.part_pair[(blockIdx.x * blockDim.x + threadIdx.x) >> 5] = e;
}

template <bool FULL, int B>
__global__ void __launch_bounds__(128, 4) k_force_union(KP P) {
  zero_pair_tail(P, gridDim.x * blockDim.x / 32);
  if (P.st->err || P.st->n_ovl) return;
  // the masked offsets (<= kMaskBits per parity) in shared memory: the
  // per-pair offset load is an LDS instead of an indexed constant load
  __shared__ int s_offs[2][kMaskBits + 1];
  for (int i = threadIdx.x; i < 2 * (kMaskBits + 1); i += blockDim.x) {
    const int par = i / (kMaskBits + 1), k = i % (kMaskBits + 1);
    const int n = FULL ? c_full_n[par] : c_half_n[par];
    s_offs[par][k] = k < n ? (FULL ? c_full[par][k] : c_half[par][k]) : 0;
  }
  __syncthreads();
  const int nb = brick_count(P.G);
  double e = 0.0;
  for (;;) {
    const int b = next_brick(&P.work[1]);
    if (b >= nb) break;
    for (int par = 0; par < 2; ++par) {
      int d;
      const bool live = brick_site(P.G, b, par, d);
      e += force_site_union<FULL, B>(P, P.dself, s_offs[par], par, d, live);
    }
  }
  for (int o = 16; o > 0; o >>= 1) e += __shfl_xor_sync(0xffffffffu, e, o);
  if ((threadIdx.x & 31) == 0) P.part_pair[(blockIdx.x * blockDim.x + threadIdx.x) >> 5] = e;
}

template <bool FULL>
__global__ void __launch_bounds__(128, 5) k_force_mask(KP P) {
  zero_pair_tail(P, gridDim.x * blockDim.x / 32);
  if (P.st->err || P.st->n_ovl) return;
  const int nb = brick_count(P.G);
  double e = 0.0;
  for (;;) {
    const int b = next_brick(&P.work[1]);
    if (b >= nb) break;
    for (int par = 0; par < 2; ++par) {
      int d;
      const bool live = brick_site(P.G, b, par, d);
      e += force_site_mask<FULL>(P, P.dself, par, d, live);
    }
  }
  for (int o = 16; o > 0; o >>= 1) e += __shfl_xor_sync(0xffffffffu, e, o);
  if ((threadIdx.x & 31) == 0) P.part_pair[(blockIdx.x * blockDim.x + threadIdx.x) >> 5] = e;
}


// force pass with the spline window in shared memory: 64-byte records of
// segments [seg_lo, nseg] are staged once per CTA, chunk c of record i at
// 16-byte slot 4 i + (c ^ (i & 3)) so random records spread over all banks;
// pairs below seg_lo (r < ~1.6 A, cascade cores only) read the global table.
constexpr int kSmemTabSegs = 3500;  // 3500 x 64 B = 224,000 B
__device__ __forceinline__ double2 tab_chunk(const double2* T, int i, int c) {
  return T[4 * i + (c ^ (i & 3))];
}

template <bool FULL>
__device__ __forceinline__ double force_site_smtab(const KP& P, KP* Pp, const double2* T,
                                                   int seg_lo, int par, int d, bool live) {
  const double4* __restrict__ pdf = P.pdf;
  const int* __restrict__ tgt = P.tgt;
  const long long S = P.S;
  double ax = kVacant, ay = 0, az = 0, adf = 0;
  if (live) ld256(pdf + d, ax, ay, az, adf);
  if (ax >= kVacantTest) {
    if (FULL && live) {
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
    int j[2], t[2], seg[2];
    double px[2], py[2], pz[2], pw[2], dx[2], dy[2], dz[2], s[2], ri[2];
#pragma unroll
    for (int b = 0; b < 2; ++b) {
      j[b] = d + offs[k[b]];
      ld256(pdf + j[b], px[b], py[b], pz[b], pw[b]);
      t[b] = __ldg(tgt + j[b]);
    }
#pragma unroll
    for (int b = 0; b < 2; ++b) {
      dx[b] = xsub(ax, px[b]);
      dy[b] = xsub(ay, py[b]);
      dz[b] = xsub(az, pz[b]);
      const double r2 = fma(dz[b], dz[b], fma(dy[b], dy[b], dx[b] * dx[b]));
      ri[b] = rsqrt(r2);
      seg[b] = seg_index(P.ff, r2 * ri[b], s[b]);
    }
#pragma unroll
    for (int b = 0; b < 2; ++b) {
      if (!v[b]) continue;
      double zA, zB, zC, zD, qA, qB, qC, qD;
      const int li = seg[b] - seg_lo;
      if (li >= 0) {
        const double2 c0 = tab_chunk(T, li, 0), c1 = tab_chunk(T, li, 1),
                      c2 = tab_chunk(T, li, 2), c3 = tab_chunk(T, li, 3);
        zA = c0.x; zB = c0.y; zC = c1.x; zD = c1.y; qA = c2.x; qB = c2.y; qC = c3.x; qD = c3.y;
      } else {
        const double* rec = P.ff.rec + 8 * (size_t)seg[b];
        ld256(rec, zA, zB, zC, zD);
        ld256(rec + 4, qA, qB, qC, qD);
      }
      (void)qD;
      const double sb = s[b], s15 = 1.5 * sb, s2 = sb + sb;
      const double z = fma(fma(fma(zA, sb, zB), sb, zC), sb, zD);
      const double zs = fma(fma(zA, s15, zB), s2, zC);
      const double ps = fma(fma(qA, s15, qB), s2, qC);
      const double phi = z * ri[b];
      const double dphi = fma(zs, ih, -phi) * ri[b];
      const double mfp = fma((adf + pw[b]) * ps, ih, dphi) * ri[b];
      const double qx = mfp * dx[b], qy = mfp * dy[b], qz = mfp * dz[b];
      fx -= qx;
      fy -= qy;
      fz -= qz;
      if (FULL) {
        e = fma(0.5, phi, e);
      } else {
        e += phi;
        red_add(&P.frc[t[b]], qx);
        red_add(&P.frc[S + t[b]], qy);
        red_add(&P.frc[2 * S + t[b]], qz);
      }
    }
  }
  if (guard) {
    const int n = FULL ? c_full_n[par] : c_half_n[par];
    for (int kk = 0; kk < n; ++kk) {
      const int jj = d + offs[kk];
      double px, py, pz, pw;
      ld256(pdf + jj, px, py, pz, pw);
      const double ddx = xsub(ax, px), ddy = xsub(ay, py), ddz = xsub(az, pz);
      const double r2 = fma(ddz, ddz, fma(ddy, ddy, ddx * ddx));
      if (decide<FULL>(P, par, kk, jj, ax, ay, az, px, py, pz, ddx, ddy, ddz, r2) != 2) continue;
      double q[4];
      if (guard_force(Pp, d, jj, __ldg(tgt + jj), ddx, ddy, ddz, adf + pw, FULL, q)) {
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

// 512 threads = 4 groups of 4 warps, each group on its own brick
__device__ __forceinline__ int next_brick_group(int* ctr, int group, volatile int* slot) {
  asm volatile("bar.sync %0, 128;" ::"r"(group + 1));
  if ((threadIdx.x & 127) == 0) slot[group] = atomicAdd(ctr, 1);
  asm volatile("bar.sync %0, 128;" ::"r"(group + 1));
  return slot[group];
}

template <bool FULL>
__global__ void __launch_bounds__(512, 1) k_force_smtab(KP P) {
  zero_pair_tail(P, gridDim.x * blockDim.x / 32);
  if (P.st->err || P.st->n_ovl) return;
  extern __shared__ __align__(16) unsigned char smem[];
  __shared__ int s_slot[4];
  double2* T = reinterpret_cast<double2*>(smem);
  const int nseg = P.ff.nseg;  // records 0..nseg (padded)
  const int seg_lo = max(0, nseg + 1 - kSmemTabSegs);
  const int nrec = nseg + 1 - seg_lo;
  for (int q = threadIdx.x; q < 4 * nrec; q += blockDim.x) {
    const int i = q >> 2, c = q & 3;
    T[4 * i + (c ^ (i & 3))] = reinterpret_cast<const double2*>(P.ff.rec + 8 * (size_t)(seg_lo + i))[c];
  }
  __syncthreads();
  const int group = threadIdx.x >> 7;
  const int nb = brick_count(P.G);
  double e = 0.0;
  for (;;) {
    const int b = next_brick_group(&P.work[1], group, s_slot);
    if (b >= nb) break;
    for (int par = 0; par < 2; ++par) {
      const int lt = threadIdx.x & 127;
      const int lane = lt & 31, w = lt >> 5;
      const Geo& G = P.G;
      const int nbx = (G.bx + kBrickX - 1) / kBrickX, nby = (G.by + kBrickY - 1) / kBrickY;
      const int cx = (b % nbx) * kBrickX + (lane & 7), cy = ((b / nbx) % nby) * kBrickY + (lane >> 3),
                cz = (b / (nbx * nby)) * kBrickZ + w;
      const bool live = cx < G.bx && cy < G.by && cz < G.bz;
      const int d = live ? (int)(par * G.NC + cell_of(cx + G.g, cy + G.g, cz + G.g, G)) : 0;
      e += force_site_smtab<FULL>(P, P.dself, T, seg_lo, par, d, live);
    }
  }
  for (int o = 16; o > 0; o >>= 1) e += __shfl_xor_sync(0xffffffffu, e, o);
  if ((threadIdx.x & 31) == 0) P.part_pair[(blockIdx.x * blockDim.x + threadIdx.x) >> 5] = e;
}

void launch_force_smtab(const KP& P, int mode, cudaStream_t s) {
  const size_t bytes = (size_t)kSmemTabSegs * 64;
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(k_force_smtab<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes);
    cudaFuncSetAttribute(k_force_smtab<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes);
    attr = true;
  }
  int sms = 148, dev = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const int g = max(1, min(sms, (brick_count(P.G) + 3) / 4));
  if (mode) k_force_smtab<true><<<g, 512, bytes, s>>>(P);
  else k_force_smtab<false><<<g, 512, bytes, s>>>(P);
}

int fast_grid(const KP& P, bool force, int mode) {
  int per_sm = 0;
  if (force) {  // one grid for both force variants: the partial-energy count must match
    int a = 0, b = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(
        &a, mode ? (const void*)k_force_mask<true> : (const void*)k_force_mask<false>, 128, 0);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(
        &b, mode ? (const void*)k_force_fast<true, 2> : (const void*)k_force_fast<false, 2>, 128,
        0);
    int c2 = 0, c4 = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(
        &c2, mode ? (const void*)k_force_union<true, 2> : (const void*)k_force_union<false, 2>,
        128, 0);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(
        &c4, mode ? (const void*)k_force_union<true, 4> : (const void*)k_force_union<false, 4>,
        128, 0);
    int c5 = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(
        &c5, mode ? (const void*)k_force_pipe<true> : (const void*)k_force_pipe<false>, 128, 0);
    int c6 = 0, c8 = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(
        &c6, mode ? (const void*)k_force_lean<true, 6> : (const void*)k_force_lean<false, 6>, 128, 0);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(
        &c8, mode ? (const void*)k_force_lean<true, 8> : (const void*)k_force_lean<false, 8>, 128, 0);
    per_sm = max(max(max(a, b), max(c2, c4)), max(c5, max(c6, c8)));
  }
  if (!force)
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(
        &per_sm, mode ? (const void*)k_density_fast<true, 2, 6> : (const void*)k_density_fast<false, 2, 6>,
        128, 0);
  int sms = 148;
  int dev = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const int blocks = sms * (per_sm > 0 ? per_sm : 1);
  return max(1, min(blocks, brick_count(P.G)));
}

bool launch_density_fast(const KP& P, int mode, int grid, cudaStream_t s) {
  static const int dsm = [] {  // 2: lean, spline window in shared memory (default)
    const char* e = getenv("CBX_DENSITY_SMEM");
    return e ? atoi(e) : 2;
  }();
  if (dsm) {
    const size_t bytes = (size_t)kDensTabRecords * 32;
    static bool attr = false;
    if (!attr) {
      cudaFuncSetAttribute(k_density_smem<false, 4, 512>,
                           cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes);
      cudaFuncSetAttribute(k_density_smem<true, 4, 512>,
                           cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes);
      cudaFuncSetAttribute(k_density_smem<false, 1, 1024>,
                           cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes);
      cudaFuncSetAttribute(k_density_smem<true, 1, 1024>,
                           cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes);
      attr = true;
    }
    int sms = 148, dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    const int g = max(1, min(sms, (brick_count(P.G) + 3) / 4));
    if (dsm == 2) {  // lean: one candidate per iteration, 1024 threads
      const int g8 = max(1, min(sms, (brick_count(P.G) + 7) / 8));
      if (mode) k_density_smem<true, 1, 1024><<<g8, 1024, bytes, s>>>(P, g8);
      else k_density_smem<false, 1, 1024><<<g8 + 4, 1024, bytes, s>>>(P, g8);
    } else {
      if (mode) k_density_smem<true, 4, 512><<<g, 512, bytes, s>>>(P, g);
      else k_density_smem<false, 4, 512><<<g + 8, 512, bytes, s>>>(P, g);
    }
    return !mode;
  }
  static const int batch = [] {
    const char* e = getenv("CBX_DENSITY_BATCH");
    return e ? atoi(e) : 4;
  }();
  const int ex = mode ? 0 : kClashBlocks128;  // fused clash pass (Newton-3)
  if (batch == 4) {
    if (mode) k_density_fast<true, 4, 4><<<grid, 128, 0, s>>>(P, grid);
    else k_density_fast<false, 4, 4><<<grid + ex, 128, 0, s>>>(P, grid);
  } else {
    if (mode) k_density_fast<true, 2, 6><<<grid, 128, 0, s>>>(P, grid);
    else k_density_fast<false, 2, 6><<<grid + ex, 128, 0, s>>>(P, grid);
  }
  return ex != 0;
}
bool launch_force_fast(const KP& P, int mode, int grid, cudaStream_t s) {
  if (P.use_mask && (P.xp & 4)) {
    launch_force_smtab(P, mode, s);
    return false;
  }
  if (P.use_mask && (P.xp & 8)) {  // per-lane mask walk (previous variant)
    if (mode) k_force_mask<true><<<grid, 128, 0, s>>>(P);
    else k_force_mask<false><<<grid, 128, 0, s>>>(P);
    return false;
  }
  static const int pipe = [] {
    const char* e = getenv("CBX_FORCE_PIPE");
    return e ? atoi(e) : 1;
  }();
  static const int lean = [] {  // 1: shared-memory spline window (default)
    const char* e = getenv("CBX_FORCE_LEAN");
    return e ? atoi(e) : 1;
  }();
  if (P.use_mask && lean == 1) {
    const size_t bytes = (size_t)kLeanTabRecords * 64;
    static bool attr = false;
    if (!attr) {
      cudaFuncSetAttribute(k_force_lean_smem<false, 1024>,
                           cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes);
      cudaFuncSetAttribute(k_force_lean_smem<true, 1024>,
                           cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes);
      cudaFuncSetAttribute(k_force_lean_smem<false, 768>,
                           cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes);
      cudaFuncSetAttribute(k_force_lean_smem<true, 768>,
                           cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes);
      attr = true;
    }
    int sms = 148, dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    const int g = max(1, min(sms, (brick_count(P.G) + 7) / 8));
    static const int nt = [] {
      const char* e = getenv("CBX_LEAN_THREADS");
      return e ? atoi(e) : 1024;
    }();
    if (nt == 768) {
      const int g6 = max(1, min(sms, (brick_count(P.G) + 5) / 6));
      if (mode) k_force_lean_smem<true, 768><<<g6, 768, bytes, s>>>(P, g6);
      else k_force_lean_smem<false, 768><<<g6 + 4, 768, bytes, s>>>(P, g6);
    } else {
      if (mode) k_force_lean_smem<true, 1024><<<g, 1024, bytes, s>>>(P, g);
      else k_force_lean_smem<false, 1024><<<g + 4, 1024, bytes, s>>>(P, g);
    }
    return !mode;
  }
  if (P.use_mask && lean) {
    const int ex = mode ? 0 : kClashBlocks128;
    if (lean == 8) {
      if (mode) k_force_lean<true, 8><<<grid, 128, 0, s>>>(P, grid);
      else k_force_lean<false, 8><<<grid + ex, 128, 0, s>>>(P, grid);
    } else {
      if (mode) k_force_lean<true, 6><<<grid, 128, 0, s>>>(P, grid);
      else k_force_lean<false, 6><<<grid + ex, 128, 0, s>>>(P, grid);
    }
    return !mode;
  }
  if (P.use_mask && pipe) {
    if (mode) k_force_pipe<true><<<grid, 128, 0, s>>>(P, grid);
    else k_force_pipe<false><<<grid + kClashBlocks128, 128, 0, s>>>(P, grid);
    return !mode;
  }
  if (P.use_mask) {
    static const int ub = [] {
      const char* e = getenv("CBX_UNION_BATCH");
      return e ? atoi(e) : 2;
    }();
    if (ub == 4) {
      if (mode) k_force_union<true, 4><<<grid, 128, 0, s>>>(P);
      else k_force_union<false, 4><<<grid, 128, 0, s>>>(P);
    } else {
      if (mode) k_force_union<true, 2><<<grid, 128, 0, s>>>(P);
      else k_force_union<false, 2><<<grid, 128, 0, s>>>(P);
    }
    return false;
  }
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
  return false;
}
