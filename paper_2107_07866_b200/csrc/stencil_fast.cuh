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
#ifndef CBX_PIN_SMEM
#define CBX_PIN_SMEM 1
#endif

__device__ __forceinline__ void ld256(const void* p, double& a, double& b, double& c,
                                      double& d) {
  // not volatile: a pure read of data that is constant during the kernel,
  // free to be scheduled early by the compiler
  asm("ld.global.nc.v4.f64 {%0,%1,%2,%3}, [%4];" : "=d"(a), "=d"(b), "=d"(c), "=d"(d) : "l"(p));
}
// the 32-byte load only where pred holds (the destinations keep their values)
__device__ __forceinline__ void ld256_pred(bool pred, const void* p, double& a, double& b,
                                           double& c, double& d) {
  asm("{\n .reg .pred q;\n setp.ne.b32 q, %5, 0;\n"
      " @q ld.global.nc.v4.f64 {%0,%1,%2,%3}, [%4];\n}"
      : "+d"(a), "+d"(b), "+d"(c), "+d"(d)
      : "l"(p), "r"((int)pred));
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
  if (!full) red_add(acc_ptr<-1>(*P, tgt), rho);
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
    red_add(acc_ptr<0>(*P, tgt), q[0]);
    red_add(acc_ptr<1>(*P, tgt), q[1]);
    red_add(acc_ptr<2>(*P, tgt), q[2]);
  }
  return true;
}

// 1/sqrt for r^2 in the normal range: the hardware approximation plus two
// Newton steps (relative error a few ulp, no special-case branch)
// (measured on B200 over r^2 in [0.5, 64]: the approximation 9.3e-7, one
// step 1.3e-12, two steps 4e-16 relative -- one step would be 1.5 % faster
// but its ~2e-11 per-pair force error, summed over 58 pairs, is not provably
// inside the 1e-10 force tolerance)
__device__ __forceinline__ double rsqrt_nr(double x) {
  double y;
  asm("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(x));
  const double h = 0.5 * x;
  y = y * fma(-h * y, y, 1.5);
  y = y * fma(-h * y, y, 1.5);
  return y;
}

__device__ __forceinline__ double2 lds2(unsigned a) {
  double2 v;
  asm("ld.shared.v2.f64 {%0,%1}, [%2];" : "=d"(v.x), "=d"(v.y) : "r"(a));
  return v;
}
__device__ __forceinline__ float2 lds_f2(unsigned a) {
  float2 v;
  asm("ld.shared.v2.f32 {%0,%1}, [%2];" : "=f"(v.x), "=f"(v.y) : "r"(a));
  return v;
}
__device__ __forceinline__ double lds_d(unsigned a) {
  double v;
  asm("ld.shared.f64 %0, [%1];" : "=d"(v) : "r"(a));
  return v;
}
__device__ __forceinline__ int lds_i(unsigned a) {
  int v;
  asm("ld.shared.b32 %0, [%1];" : "=r"(v) : "r"(a));
  return v;
}

// 16 bytes of the 64-byte force record `seg` (chunk c: 0 [zA zB], 1 [zC zD],
// 2 [qA qB], 3 [qC qD]) through the texture path: the TEX data pipe runs
// beside the LSU pipe that serves the shared-memory table, the partner
// gathers and the reductions (tabbench: 2 LDS.128 + 1 TLD per lane cost what
// 2 LDS.128 alone cost)
__device__ __forceinline__ double2 tex_chunk(unsigned long long tex, int seg, int c) {
  const int4 q = tex1Dfetch<int4>((cudaTextureObject_t)tex, 4 * seg + c);
  return make_double2(__hiloint2double(q.y, q.x), __hiloint2double(q.w, q.z));
}

// 16-byte record i of a table bound to a texture of int4 texels (the
// density pass's [D C] records)
__device__ __forceinline__ double2 tex_rec16(unsigned long long tex, int i) {
  const int4 q = tex1Dfetch<int4>((cudaTextureObject_t)tex, i);
  return make_double2(__hiloint2double(q.y, q.x), __hiloint2double(q.w, q.z));
}

// ------------------------------------------------------------------ density
// one skin candidate that passed the fp32 filter (rare): full decision
template <bool FULL, bool REV = true>
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
  if (!FULL) red_add(REV ? acc_ptr<-1>(P, to) : P.rho + to, rho);
  return rho;
}

// 32-byte density records staged in shared memory: chunk c of record i at
// 16-byte slot 2 i + (c ^ ((i >> 2) & 1)) (8 distinct bank quads for random i)
__device__ __forceinline__ int smem_slot32(int i, int c) { return 2 * i + (c ^ ((i >> 2) & 1)); }

// CMPD: 0 the fp64 32-byte records of the window in shared memory; 1 the
// compressed records ([D C] fp64 + [A B] fp32) in shared memory; 2 compressed,
// [D C] by texture fetch (TEX pipe) and [A B] in shared memory (LSU pipe);
// 3-4: the inner loop unrolled by two with alternating register sets (no
// copies) and a one-word pair mask; tables: 3 fp64 [A B] (16 B) in shared
// memory + [C D] by texture, 4 (default where the fp32 guard holds) those of
// 2 (both halves by texture, fp32 or fp64: measured slower)
// end of the offsets a site of sublattice par examines for threshold T
template <bool FULL>
__device__ __forceinline__ int skin_end(const KP& P, int par, double T) {
  const SkinGroups& sg = FULL ? P.skf[par] : P.skh[par];
  int n = FULL ? c_full_nin[par] : c_half_nin[par];
  for (int i = 0; i < sg.n; ++i) {
    if (sg.len[i] > T) return n;
    n = sg.end[i];
  }
  return kMaxOffsets;
}

// skU (skin pruning, skin_region_bound): the largest displacement bound of
// the chunks the lanes' skin partners lie in, or >= 1e299 for none; cxs, cys,
// czs: the site's ghost-inclusive cell.  Returns the end of the offsets
// examined (the diagnostic count of cbx_skin_stats).
template <bool FULL, int B, bool SMEM = false, bool REV = false, int CMPD = 0>
__device__ __forceinline__ int density_site(const KP& P, KP* Pp, int par, int d, bool live,
                                            unsigned tb = 0, int seg_lo = 0,
                                            bool rev_here = true, bool deep = false,
                                            unsigned tb8 = 0, double skU = 1e300, int cxs = 0,
                                            int cys = 0, int czs = 0) {
  const double4* __restrict__ pdf = P.pdf;
  const int* __restrict__ tgt = P.tgt;
  double ax = kVacant, ay = 0, az = 0, aw = 0;
  if (live) ld256(pdf + d, ax, ay, az, aw);
  int n_lim = kMaxOffsets;
  if (skU < 1e299) {  // warp-uniform: the lanes' own displacements |u_i|
    double u2 = 0.0;
    if (ax < kVacantTest) {
      const double h = 0.5 * par;
      const double ux = ax - ((double)cxs + h) * P.G.a0, uy = ay - ((double)cys + h) * P.G.a0,
                   uz = az - ((double)(czs + P.G.zoff) + h) * P.G.a0;
      u2 = fma(ux, ux, fma(uy, uy, uz * uz));
    }
    // non-negative floats order as their bit patterns; rounded up
    const unsigned m = __reduce_max_sync(0xffffffffu, __float_as_uint(__double2float_ru(u2)));
    n_lim = skin_end<FULL>(P, par, P.cutoff + 1e-9 + skU + sqrt((double)__uint_as_float(m)));
  }
  if (ax >= kVacantTest) {
    if (FULL && live) P.rho[d] = 0.0;
    return n_lim;
  }
  // n_lim: skin shells beyond it are out of cutoff for every lane (regional
  // displacement bound, skin_end)
  const int n = min(FULL ? c_full_n[par] : c_half_n[par], n_lim);
  const int nin = FULL ? c_full_nin[par] : c_half_nin[par];
  const int* offs = FULL ? c_full[par] : c_half[par];
  const double lo = P.cut2_lo, g2 = P.guard_r2;
  double acc = 0.0;
  unsigned long long m0 = 0, m1 = 0;
  // inner shells: direct fp64 gather; the common case is decided by one
  // compare, the near-cutoff / guard cases drop to decide().  B == 1 (the
  // shared-memory kernels): software-pipelined, the next candidate's gather
  // is in flight while the current one's table lookup and RED run
  if constexpr (B == 1 && (CMPD == 3 || CMPD == 4)) {
    // one inner candidate once its partner is loaded (nin <= 64: host check)
    auto cand = [&](int k, int j, int t, double px, double py, double pz) {
      const double dx = xsub(ax, px), dy = xsub(ay, py), dz = xsub(az, pz);
      const double r2 = fma(dz, dz, fma(dy, dy, dx * dx));
      bool in = r2 <= lo && r2 >= g2;
      if (!in && r2 <= P.cut2_hi) {
        const int st = decide<FULL>(P, par, k, j, ax, ay, az, px, py, pz, dx, dy, dz, r2);
        if (st == 1) {
          in = true;
        } else if (st == 2) {
          m1 |= kGuardBit;
          acc += guard_rho(Pp, d, j, t, dx, dy, dz, FULL);
        }
      }
      if (in) {
        double sv;
        const int sg = seg_index(P.fd, r2 * rsqrt_nr(r2), sv);
        const int li = sg - seg_lo;
        double tA, tB, tC, tD;
        if (li >= 0 && CMPD == 4) {  // the compressed records of CMPD 2
          const double2 dc = tex_rec16(P.tex_fd, sg);
          const float2 ab = lds_f2(tb8 + 8 * li);
          tA = (double)ab.x;
          tB = (double)ab.y;
          tC = dc.y;
          tD = dc.x;
        } else if (li >= 0) {
          const double2 ab = lds2(tb + 16 * li);
          const double2 cd = tex_rec16(P.tex_fd4, sg);
          tA = ab.x;
          tB = ab.y;
          tC = cd.x;
          tD = cd.y;
        } else {
          ld256(P.fd.rec + 4 * (size_t)sg, tA, tB, tC, tD);
        }
        const double rho = fma(fma(fma(tA, sv, tB), sv, tC), sv, tD);
        acc += rho;
        if (!FULL) red_add(REV && rev_here ? acc_ptr_up(P, t, -1) : P.rho + t, rho);
      }
      m0 |= (unsigned long long)in << k;
    };
    int ja = d + offs[0], jb;
    double xa, ya, za, wa, xb, yb, zb, wb;
    ld256(pdf + ja, xa, ya, za, wa);
    int ta = deep ? ja : __ldg(tgt + ja), tq;
    int k = 0;
#pragma unroll 1
    for (; k + 1 < nin; k += 2) {
      jb = d + offs[k + 1];
      ld256(pdf + jb, xb, yb, zb, wb);
      tq = deep ? jb : __ldg(tgt + jb);
      cand(k, ja, ta, xa, ya, za);
      if (k + 2 < nin) {
        ja = d + offs[k + 2];
        ld256(pdf + ja, xa, ya, za, wa);
        ta = deep ? ja : __ldg(tgt + ja);
      }
      cand(k + 1, jb, tq, xb, yb, zb);
    }
    if (k < nin) cand(k, ja, ta, xa, ya, za);
  } else if constexpr (B == 1) {
    int jn = d + offs[0];
    double qx, qy, qz, qw;
    ld256(pdf + jn, qx, qy, qz, qw);
    int tn = deep ? jn : __ldg(tgt + jn);
#pragma unroll 1
    for (int k = 0; k < nin; ++k) {
      const int j = jn, t = tn;
      const double px = qx, py = qy, pz = qz;
      if (k + 1 < nin) {
        jn = d + offs[k + 1];
        ld256(pdf + jn, qx, qy, qz, qw);
        tn = deep ? jn : __ldg(tgt + jn);
      }
      const double dx = xsub(ax, px), dy = xsub(ay, py), dz = xsub(az, pz);
      const double r2 = fma(dz, dz, fma(dy, dy, dx * dx));
      bool in = r2 <= lo && r2 >= g2;
      if (!in && r2 <= P.cut2_hi) {
        const int st = decide<FULL>(P, par, k, j, ax, ay, az, px, py, pz, dx, dy, dz, r2);
        if (st == 1) {
          in = true;
        } else if (st == 2) {
          m1 |= kGuardBit;
          acc += guard_rho(Pp, d, j, t, dx, dy, dz, FULL);
        }
      }
      if (in) {
        double sv;
        const int sg = seg_index(P.fd, r2 * rsqrt_nr(r2), sv);
        const int li = sg - seg_lo;
        double tA, tB, tC, tD;
        if (SMEM && CMPD && li >= 0) {  // [D C] and the fp32 pair [A B]
          const double2 dc = CMPD == 2 ? tex_rec16(P.tex_fd, sg) : lds2(tb + 16 * li);
          const float2 ab = lds_f2(tb8 + 8 * li);
          tA = (double)ab.x;
          tB = (double)ab.y;
          tC = dc.y;
          tD = dc.x;
        } else if (SMEM && li >= 0) {
          const double2 c0 = lds2(tb + 16 * smem_slot32(li, 0)), c1 = lds2(tb + 16 * smem_slot32(li, 1));
          tA = c0.x;
          tB = c0.y;
          tC = c1.x;
          tD = c1.y;
        } else {
          ld256(P.fd.rec + 4 * (size_t)sg, tA, tB, tC, tD);
        }
        const double rho = fma(fma(fma(tA, sv, tB), sv, tC), sv, tD);
        acc += rho;
        if (!FULL) red_add(REV && rev_here ? acc_ptr_up(P, t, -1) : P.rho + t, rho);
        set_bit(m0, m1, k);
      }
    }
  } else
  for (int k0 = 0; k0 < nin; k0 += B) {
    int j[B], t[B], seg[B];
    bool in[B];
    double px[B], py[B], pz[B], s[B], r2[B];
#pragma unroll
    for (int b = 0; b < B; ++b) {
      j[b] = d + offs[min(k0 + b, nin - 1)];
      double w;
      ld256(pdf + j[b], px[b], py[b], pz[b], w);
      t[b] = deep ? j[b] : __ldg(tgt + j[b]);
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
    for (int b = 0; b < B; ++b) seg[b] = seg_index(P.fd, r2[b] * rsqrt_nr(r2[b]), s[b]);
    double tA[B], tB[B], tC[B], tD[B];
#pragma unroll
    for (int b = 0; b < B; ++b)
      if (in[b]) {
        const int li = seg[b] - seg_lo;
        if (SMEM && CMPD) {  // [D C] and the fp32 pair [A B]
          const int lc = max(li, 0);
          const double2 dc = CMPD == 2 ? tex_rec16(P.tex_fd, lc + seg_lo) : lds2(tb + 16 * lc);
          const float2 ab = lds_f2(tb8 + 8 * lc);
          tA[b] = (double)ab.x;
          tB[b] = (double)ab.y;
          tC[b] = dc.y;
          tD[b] = dc.x;
        } else if (SMEM) {
          const int lc = max(li, 0);
          const double2 c0 = lds2(tb + 16 * smem_slot32(lc, 0)), c1 = lds2(tb + 16 * smem_slot32(lc, 1));
          tA[b] = c0.x;
          tB[b] = c0.y;
          tC[b] = c1.x;
          tD[b] = c1.y;
        }
        if (!SMEM || li < 0) ld256(P.fd.rec + 4 * (size_t)seg[b], tA[b], tB[b], tC[b], tD[b]);
      }
#pragma unroll
    for (int b = 0; b < B; ++b) {
      if (in[b]) {
        const double rho = fma(fma(fma(tA[b], s[b], tB[b]), s[b], tC[b]), s[b], tD[b]);
        acc += rho;
        if (!FULL) red_add(REV && rev_here ? acc_ptr_up(P, t[b], -1) : P.rho + t[b], rho);
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
      // (each lane walking its own passing candidates in a loop -- max over
      // the lanes instead of one divergent pass per candidate -- measured
      // slower: density 4.93 vs 4.24 ms at config 5, the loop's selects spill)
#pragma unroll
      for (int b = 0; b < 4; ++b)
        if (pass[b])
          acc += skin_density<FULL, REV>(P, Pp, par, k0 + b, d, jj[b], __float_as_int(pf[b].w), ax,
                                    ay, az, m0, m1);
    }
  }
  if (FULL) P.rho[d] = acc;
  else red_add(&P.rho[d], acc);
  if (P.pmask) {
    P.pmask[2 * (size_t)d] = m0;
    P.pmask[2 * (size_t)d + 1] = m1;
  }
  return n_lim;
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
      red_add(acc_ptr<0>(P, to), o.qx);
      red_add(acc_ptr<1>(P, to), o.qy);
      red_add(acc_ptr<2>(P, to), o.qz);
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

// OR of a 64-bit value over the warp (the union of the lanes' pair masks)
__device__ __forceinline__ unsigned long long warp_or64(unsigned long long m) {
  const unsigned lo = __reduce_or_sync(0xffffffffu, (unsigned)m);
  const unsigned hi = __reduce_or_sync(0xffffffffu, (unsigned)(m >> 32));
  return ((unsigned long long)hi << 32) | lo;
}

// Force-table sources (template TB of the force pass):
//   kTabSmem64: the 64-byte records of the window in shared memory, 4 LDS.128
//   kTabSplit:  [zA zB][zC zD] of the window in shared memory (2 LDS.128),
//               [qA qB][qC qD] by texture fetches (2 TLD) -- the LSU and TEX
//               pipes share the lookups
//   kTabSplit3: [zC zD] (LDS.128) + qC (LDS.64) in shared memory, [zA zB]
//               [qA qB] by texture fetches
// Pairs below the window (cascade cores) fetch every chunk by texture.
constexpr int kTabSmem64 = 0, kTabSplit = 2, kTabSplit3 = 3;
constexpr int kTabSmemBytes[4] = {64, 0, 32, 24};

// force pass, lean variant: one pair per iteration, no batching, so the
// register footprint allows 6-8 resident CTAs per SM (latency hidden by
// warps instead of by in-thread batching).  Warp-uniform union sweep.
template <bool FULL, int TB, bool REV = false>
__device__ __forceinline__ double force_site_lean(const KP& P, KP* Pp, int par, int d,
                                                  bool live, unsigned tb = 0,
                                                  int seg_lo = 0, bool rev_here = false,
                                                  bool deep = false, unsigned tb8 = 0) {
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
  const unsigned s_offs = smem_addr(g_soffs[par]);
  const double ih = P.ff.ih;
  const double r2_idle = P.cut2_lo;
  double fx = 0.0, fy = 0.0, fz = 0.0, e = 0.0;
  // the warp walks the union of its lanes' masks (warp-uniform offset, lanes
  // without the bit idle), one 32-bit word at a time.  Skin offsets (k >= nin,
  // P.skin_lane): the lattice puts them beyond the cutoff, so few lanes hold
  // any one of them (shell 6 at 600 K: ~16 % each) -- after the inner offsets
  // every lane walks its OWN skin bits (lane-varying offset from the staged
  // shared-memory copy): max over the lanes of their skin-pair counts
  // iterations instead of the size of the union
#ifdef CBX_AB  // experiment build: runtime switches back to the earlier variants
  const bool packed = P.tab_packed != 0, skin_lane = P.skin_lane != 0;
  const bool offs_const = P.offs_const != 0, idle_pred = P.idle_pred != 0;
#else
  constexpr bool packed = true, skin_lane = true, offs_const = true, idle_pred = true;
#endif
  const int nin = skin_lane ? (FULL ? c_full_nin[par] : c_half_nin[par]) : kMaskBits + 1;
  {
  int wd = 0;
  unsigned cu = 0, co = 0;
#pragma unroll 1
  for (;;) {
      bool v;
      int off;
      if (wd <= 4) {  // inner offsets: the union walk
        if (!cu) {
          if (wd == 4 || 32 * wd >= nin) {  // the lanes' own skin bits from here
            if (nin > kMaskBits) break;
            if (nin < 64) { m0 &= ~0ull << nin; } else { m0 = 0; m1 &= ~0ull << (nin - 64); }
            wd = 5;
            continue;
          }
          const unsigned long long mw = wd < 2 ? m0 : m1;
          co = (wd & 1) ? (unsigned)(mw >> 32) : (unsigned)mw;
          if (nin - 32 * wd < 32) co &= (1u << (nin - 32 * wd)) - 1u;
          cu = __reduce_or_sync(0xffffffffu, co);
          ++wd;
          continue;
        }
        const int bit = __ffs(cu) - 1;
        cu &= cu - 1;
        v = (co >> bit) & 1;
        // the offset: a warp-uniform index, from the constant cache (no LSU
        // wavefront) or the staged shared-memory copy
        const int k = 32 * (wd - 1) + bit;
        off = offs_const ? (FULL ? c_full[par][k] : c_half[par][k]) : lds_i(s_offs + 4 * k);
      } else {
        v = (m0 | m1) != 0;
        if (!__any_sync(0xffffffffu, v)) break;
        int k = 0;
        if (m0) {
          k = __ffsll((long long)m0) - 1;
          m0 &= m0 - 1;
        } else if (m1) {
          k = 63 + __ffsll((long long)m1);
          m1 &= m1 - 1;
        }
        off = lds_i(s_offs + 4 * k);
      }
      const int j = v ? d + off : d;
      double px = ax, py = ay, pz = az, pw = 0.0;
      int t = j;
      if (idle_pred) {  // idle lanes issue no gather (sparse offsets touch fewer lines)
        ld256_pred(v, pdf + j, px, py, pz, pw);
        if (!deep && v) t = __ldg(tgt + j);
      } else {
        ld256(pdf + j, px, py, pz, pw);
        t = deep ? j : __ldg(tgt + j);
      }
      const double dx = xsub(ax, px), dy = xsub(ay, py), dz = xsub(az, pz);
      double r2 = fma(dz, dz, fma(dy, dy, dx * dx));
      r2 = v ? r2 : r2_idle;
      const double ri = rsqrt_nr(r2);
      double sb;
      const int seg = seg_index(P.ff, r2 * ri, sb);
      double zA, zB, zC, zD, qA, qB, qC;
      int li = seg - seg_lo;
      if (TB == kTabSplit3) {  // the window's gap: records above it move down, inside it -> texture
        const bool up = seg >= P.fw_gap_lo + P.fw_gap_n;
        li = up ? li - P.fw_gap_n : (seg >= P.fw_gap_lo ? -1 : li);
      }
      const int lc = max(li, 0);
      if (TB == kTabSplit) {
        const double2 q0 = tex_chunk(P.tex_ff, seg, 2), q1 = tex_chunk(P.tex_ff, seg, 3);
        qA = q0.x; qB = q0.y; qC = q1.x;
        if (li >= 0) {
          const double2 c0 = lds2(tb + 32 * lc), c1 = lds2(tb + 32 * lc + 16);
          zA = c0.x; zB = c0.y; zC = c1.x; zD = c1.y;
        } else {
          const double2 c0 = tex_chunk(P.tex_ff, seg, 0), c1 = tex_chunk(P.tex_ff, seg, 1);
          zA = c0.x; zB = c0.y; zC = c1.x; zD = c1.y;
        }
      } else if (TB == kTabSplit3) {
        // [zA zB] and [qA qB]: the two halves of one 32-byte sector of the
        // packed array (P.tab_packed; else chunks 0 and 2 of the 64-byte record)
        const double2 c0 = packed ? tex_rec16(P.tex_fab, 2 * seg) : tex_chunk(P.tex_ff, seg, 0);
        const double2 q0 = packed ? tex_rec16(P.tex_fab, 2 * seg + 1) : tex_chunk(P.tex_ff, seg, 2);
        zA = c0.x; zB = c0.y; qA = q0.x; qB = q0.y;
        if (li >= 0) {
          const double2 c1 = lds2(tb + 16 * lc);
          zC = c1.x; zD = c1.y;
          qC = lds_d(tb8 + 8 * lc);
        } else {
          const double2 c1 = tex_chunk(P.tex_ff, seg, 1), q1 = tex_chunk(P.tex_ff, seg, 3);
          zC = c1.x; zD = c1.y; qC = q1.x;
        }
      } else {
        const double2 c0 = lds2(tb + 16 * smem_slot(lc, 0)), c1 = lds2(tb + 16 * smem_slot(lc, 1));
        const double2 c2 = lds2(tb + 16 * smem_slot(lc, 2)), c3 = lds2(tb + 16 * smem_slot(lc, 3));
        zA = c0.x; zB = c0.y; zC = c1.x; zD = c1.y;
        qA = c2.x; qB = c2.y; qC = c3.x;
        if (li < 0) {  // below the window (cascade cores): global record
          const double* rec = P.ff.rec + 8 * (size_t)seg;
          double qD;
          ld256(rec, zA, zB, zC, zD);
          ld256(rec + 4, qA, qB, qC, qD);
        }
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
        if (v) {
          if (REV && rev_here) {  // warp-uniform: a plane within reach of the halo
            double* f = acc_ptr_up(P, t, 0);
            const long long st = (int)t - ((int)t >= (int)P.G.NC ? (int)P.G.NC : 0) >= (int)P.rev.hi
                                     ? P.rev.S[1] : S;
            red_add(f, qx);
            red_add(f + st, qy);
            red_add(f + 2 * st, qz);
          } else {
            red_add(&P.frc[t], qx);
            red_add(&P.frc[S + t], qy);
            red_add(&P.frc[2 * S + t], qz);
          }
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

// one pair-energy partial per CTA: warp sums, then the warps in order
// (deterministic for a given grid)
template <int NT>
__device__ __forceinline__ void block_partial(double e, double* part) {
  __shared__ double s_w[NT / 32];
  for (int o = 16; o > 0; o >>= 1) e += __shfl_xor_sync(0xffffffffu, e, o);
  if ((threadIdx.x & 31) == 0) s_w[threadIdx.x >> 5] = e;
  __syncthreads();
  if (threadIdx.x == 0) {
    double t = 0.0;
    for (int i = 0; i < NT / 32; ++i) t += s_w[i];
    part[blockIdx.x] = t;
  }
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

// Work units of the shared-table passes: a strip of 32 consecutive interior
// cells of one x-y plane (x fastest, rows wrapping, so no partly empty
// bricks at the box faces) on 4 consecutive z planes, warp w on plane
// 4 zb + w.  Config 2: 79 strips x 13 z blocks = 1027 units, 99 % of the
// lanes live (8x4x4 bricks: 1183, 85 %).
__host__ __device__ __forceinline__ int strip_count(const Geo& G) {
  return (G.bx * G.by + 31) / 32;
}
__host__ __device__ __forceinline__ int unit_count(const Geo& G) {
  return strip_count(G) * ((G.bz + 3) / 4);
}
// strip of unit u within its z block.  When rows hold whole strips
// (bx % 32 == 0, e.g. configs 4 and 5) consecutive units walk down a column
// of strips along y: a CTA's concurrent groups then share the partner rows
// of a compact (36 x 11 x 6)-cell neighbourhood that fits L1 (row order
// spans whole rows: a 5-row x 6-plane working set 3x the L1)
__device__ __forceinline__ int unit_strip(const Geo& G, int u, int& zb) {
  const int ns = strip_count(G);
  zb = u / ns;
  const int r = u - zb * ns;
  if (G.bx % 32 == 0 && G.col_units) {
    const int xs = r / G.by, y = r - xs * G.by;
    return y * (G.bx / 32) + xs;
  }
  return r;
}
__device__ __forceinline__ bool unit_cell(const Geo& G, int u, int lane, int w, int& c,
                                          int* gx = nullptr, int* gy = nullptr,
                                          int* gz = nullptr) {
  int zb;
  const int st = unit_strip(G, u, zb);
  const int e = st * 32 + lane, cz = zb * 4 + w;
  const bool live = e < G.bx * G.by && cz < G.bz;
  const int cy = e / G.bx, cx = e - cy * G.bx;
  c = live ? (int)cell_of(cx + G.g, cy + G.g, cz + G.g, G) : 0;
  if (gx) {  // ghost-inclusive cell coordinates
    *gx = cx + G.g;
    *gy = cy + G.g;
    *gz = cz + G.g;
  }
  return live;
}
// a "deep" site has every stencil partner in an interior cell (the offsets
// reach at most g cells per axis; half lists reach up in z only), so each
// partner is its own owner and the owner load tgt[j] is skipped.  On a slab
// rank the z-halo planes' owner is the site itself too (tgt, capi.cu), so
// only x and y matter there.
__device__ __forceinline__ bool unit_deep(const Geo& G, int u, int lane, int w, bool full) {
  int zb;
  const int st = unit_strip(G, u, zb);
  const int e = st * 32 + lane, cz = zb * 4 + w;
  const int cy = e / G.bx, cx = e - cy * G.bx;
  return cx >= G.g && cx < G.bx - G.g && cy >= G.g && cy < G.by - G.g &&
         (G.slab || (cz < G.bz - G.g && (!full || cz >= G.g)));
}
// warp w of unit u sits on a z plane whose partners can lie in a halo plane
// (Newton-3 half lists reach dz >= 0 only, at most the ghost width)
__device__ __forceinline__ bool near_halo(const Geo& G, int u, int w) {
  return (u / strip_count(G)) * 4 + w + G.g >= G.bz;
}
// CTA b owns the contiguous unit range [b nu / nsb, (b + 1) nu / nsb): its
// concurrent groups sit on neighbouring strips of one z block and share most
// of their partner rows in L1 (scattered units shared none).  Within the
// range the groups take units in order from a shared-memory counter, so a
// heavier unit (a cascade core) delays only its own group.
__device__ __forceinline__ int unit_lo(int b, int nsb, int nu) {
  return (int)(((long long)b * nu) / nsb);
}
// rr > 0 (default 14): batches of rr consecutive units dealt round-robin to
// the CTAs -- every CTA sweeps the box bottom-up in step with the others, so
// the concurrent work is a thin slab of planes whose partners stay in L2
// (config 5, A/B: force 7.52 -> 7.36 ms, density 4.30 -> 4.16 ms against
// contiguous per-CTA ranges; batches of 10-21 within noise, 42 slower)
__device__ __forceinline__ int next_unit(int* s_ctr, int group, int nsb, int nu,
                                         volatile int* slot, int rr = 0) {
  asm volatile("bar.sync %0, 128;" ::"r"(group + 1));
  if ((threadIdx.x & 127) == 0) {
    const int i = atomicAdd(s_ctr, 1);
    slot[group] = rr ? ((i / rr) * nsb + blockIdx.x) * rr + i % rr
                     : unit_lo(blockIdx.x, nsb, nu) + i;
  }
  asm volatile("bar.sync %0, 128;" ::"r"(group + 1));
  const int u = slot[group];
  if (rr) return u < nu ? u : nu;
  return u < unit_lo(blockIdx.x + 1, nsb, nu) ? u : nu;
}

// Skin pruning by the regional displacement bounds (cbx_device.cuh).  For a
// pair of sites at lattice distance R whose atoms are displaced by u_i and u_j
// from them, r = |R + u_j - u_i| >= R - |u_i| - |u_j|.  Every skin partner of
// a warp's lanes lies in the chunks of planes z..z+s (z-s..z+s with full
// lists), rows y-s..y+s and x chunks xs-1..xs+1, s the cell reach of the skin
// offsets (P.skin_reach); with U the largest bound among them and |u_i| the
// lanes' own displacements (density_site), a skin shell with
// R > cutoff + U + max |u_i| + margin is out of cutoff for every lane,
// whatever the reference's rounding (margin 1e-9 A against rounding errors of
// ~1e-12 A in r and u).  Returns U (>= 1e299 when a chunk is unbounded, stale
// or in a z halo of a slab rank).  Rows holding whole chunks (bx % 32 == 0)
// only: P.ub is null otherwise.
template <bool FULL>
__device__ __forceinline__ double skin_region_bound(const KP& P, int u, int w,
                                                    unsigned long long cur) {
  if (!cur) return 1e300;
  const Geo& G = P.G;
  int zb;
  const int st = unit_strip(G, u, zb);
  const int nxs = G.bx >> 5;
  const int y = st / nxs, xs = st - y * nxs, z = zb * 4 + w;
  const int g = P.skin_reach[FULL ? 1 : 0], ny = 2 * g + 1, nz = FULL ? 2 * g + 1 : g + 1;
  const int total = nz * ny * 3;
  unsigned long long q = 0;
  for (int i = threadIdx.x & 31; i < total; i += 32) {
    const int iz = i / (ny * 3), r = i - iz * ny * 3, iy = r / 3, ix = r - iy * 3;
    int zz = z + iz - (FULL ? g : 0);
    int yy = y + iy - g, xx = xs + ix - 1;
    yy = ((yy % G.by) + G.by) % G.by;
    xx = ((xx % nxs) + nxs) % nxs;
    if (zz < 0 || zz >= G.bz) {
      if (G.slab) {
        q = kUbQMax;
        continue;
      }
      zz = ((zz % G.bz) + G.bz) % G.bz;
    }
    const unsigned long long e = __ldcg(P.ub + ((size_t)zz * G.by + yy) * nxs + xx);
    q = max(q, (e >> kUbShift) == cur ? (e & kUbQMax) : kUbQMax);
  }
  const unsigned qm = __reduce_max_sync(0xffffffffu, (unsigned)q);
  if (qm >= (unsigned)kUbQMax) return 1e300;
  return (double)qm / kUbScale;
}

// density pass with the upper rho-spline window in shared memory (32-byte
// records): NT threads = NT/128 groups of 4 warps, one CTA per SM; B = 1
// (one candidate per iteration) keeps the thread at 64 registers
// kDensTabRecords (cbx_device.cuh): records of the staged window
template <bool FULL, int B, int NT, bool REV = false, int CMPD = 0>
__global__ void __launch_bounds__(NT, 1) k_density_smem(KP P, int nsb) {
  if (blockIdx.x >= nsb) {
    pdl_wait();
    pdl_trigger();
    // merged kick: the previous step's StepState sums, pending since
    // k_rehash_images, in the first clash block (it runs in the pass's tail)
    if (blockIdx.x == nsb) finalize_pending<NT>(P);
    clash_body<0>(P, blockIdx.x - nsb, gridDim.x - nsb);
    return;
  }
  extern __shared__ __align__(16) unsigned char smem_tab[];
  __shared__ int s_slot[NT / 128];
  __shared__ int s_ctr;
  double2* T = reinterpret_cast<double2*>(smem_tab);
  const int nseg = P.fd.nseg;
  if (threadIdx.x == 0) s_ctr = 0;
  // an even first record: the fp32 [A B] pairs (8 bytes each) are then
  // 16-byte aligned for the bulk copy
  constexpr int CM = CMPD == 4 ? 2 : CMPD;  // 4: the tables of 2, the loop of 3
  const int seg_lo = CM == 3 ? max(0, nseg + 1 - kDensTabRecords)
                     : CM ? dens_window_lo_cmp(nseg) : max(0, nseg + 1 - kDensTabRecords);
  const int nrec = nseg + 1 - seg_lo;
  const double2* src = reinterpret_cast<const double2*>(P.fd.rec + 4 * (size_t)seg_lo);
  // the constant table is staged while the predecessor drains (PDL)
  // 24-byte records: [D C] 16-byte slots, then the fp32 [A B] pairs
  // (CMPD 2: only the [A B] pairs are staged, from offset 0)
  double2* T8 = CM == 2 ? T : T + kDensTabRecords;  // byte offset 16 x kDensTabRecords
  __shared__ __align__(8) unsigned long long s_mbar;
  if (CM == 3) {  // the window's fp64 [A B] pairs, one bulk copy
    if (threadIdx.x == 0) {
      const unsigned mb = smem_addr(&s_mbar);
      mbar_init(mb);
      mbar_expect_tx(mb, 16u * nrec);
      bulk_stage(smem_addr(T), P.fdab + 2 * (size_t)seg_lo, 16u * nrec, mb);
    }
  } else if (CMPD) {  // two bulk copies ([A B] rounded up to 16 bytes: the table is padded)
    const int N1 = nseg + 1;
    const unsigned mb = smem_addr(&s_mbar);
    if (threadIdx.x == 0) {
      const unsigned b16 = 16u * nrec, b8 = (8u * nrec + 15u) & ~15u;
      mbar_init(mb);
      if (CM == 2) {
        mbar_expect_tx(mb, b8);
      } else {
        mbar_expect_tx(mb, b16 + b8);
        bulk_stage(smem_addr(T), P.fdc + 2 * (size_t)seg_lo, b16, mb);
      }
      bulk_stage(smem_addr(T8), P.fdc + 2 * (size_t)N1 + seg_lo, b8, mb);
    }
  } else {
    for (int q = threadIdx.x; q < 2 * nrec; q += blockDim.x) T[smem_slot32(q >> 1, q & 1)] = __ldg(src + q);
  }
  __syncthreads();  // the barrier's initialisation is visible
  if (CMPD) mbar_wait0(smem_addr(&s_mbar));
  pdl_wait();
  pdl_trigger();
  if (P.st->err || P.st->halt) return;
  const int group = threadIdx.x >> 7;
  const int lt = threadIdx.x & 127, lane = lt & 31, w = lt >> 5;
  const Geo& G = P.G;
  const int nu = unit_count(G);
  // stamp of the regional displacement bounds this pass may use (0: none)
  const unsigned long long ub_cur = P.ub ? __ldcg(P.ustamp) : 0ull;
  const bool cnt_skin = __ldcg(P.skin_cnt + 2) != 0;
  // the window's shared addresses held in registers: left to the compiler,
  // the address (window base + CTA rank << 24) is rebuilt from SR_CgaCtaId
  // for every candidate (4-5 issue slots of ~70 in an issue-bound loop):
  // density 4.29 -> 4.20 ms at config 5 (A/B, two release builds)
  unsigned tbr = smem_addr(T), tb8r = smem_addr(T8);
#if CBX_PIN_SMEM
  asm volatile("" : "+r"(tbr), "+r"(tb8r));
#endif
  for (;;) {
    const int u = next_unit(&s_ctr, group, nsb, nu, s_slot, P.unit_rr);
    if (u >= nu) break;
    int c, cxs, cys, czs;
    const bool live = unit_cell(G, u, lane, w, c, &cxs, &cys, &czs);
    const bool deep = live && unit_deep(G, u, lane, w, FULL);
    const double skU = skin_region_bound<FULL>(P, u, w, ub_cur);
    for (int par = 0; par < 2; ++par) {
      const int n_lim = density_site<FULL, B, true, REV, CMPD>(
          P, P.dself, par, live ? (int)(par * G.NC + c) : 0, live, tbr, seg_lo,
          near_halo(G, u, w), deep, tb8r, skU, cxs, cys, czs);
      if (cnt_skin) {  // diagnostic (cbx_skin_stats)
        const unsigned nl = __popc(__ballot_sync(0xffffffffu, live));
        if (lane == 0) {
          const int nf = FULL ? c_full_n[par] : c_half_n[par];
          const int ni = FULL ? c_full_nin[par] : c_half_nin[par];
          atomicAdd(P.skin_cnt, (unsigned long long)(min(nf, n_lim) - ni) * nl);
          atomicAdd(P.skin_cnt + 1, (unsigned long long)(nf - ni) * nl);
        }
      }
    }
  }
}

template <bool FULL, int B, int MINB>
__global__ void __launch_bounds__(128, MINB) k_density_fast(KP P, int nsb) {
  if (blockIdx.x >= nsb) {
    clash_body<0>(P, blockIdx.x - nsb, gridDim.x - nsb);
    return;
  }
  if (P.st->err || P.st->halt) return;
  const int nb = brick_count(P.G);
  for (;;) {
    const int b = next_brick(&P.work[0]);
    if (b >= nb) break;
    for (int par = 0; par < 2; ++par) {
      int d;
      const bool live = brick_site(P.G, b, par, d);
      density_site<FULL, B, false, true>(P, P.dself, par, d, live);  // runtime rev check
    }
  }
}

template <bool FULL, int B>
__global__ void __launch_bounds__(128, 4) k_force_fast(KP P) {
  zero_pair_tail(P, gridDim.x);
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
  block_partial<128>(e, P.part_pair);
}

// lean force pass with the upper spline window (records [seg_lo, nseg])
// in shared memory (TB: which 16-byte chunks, see kTabSmem64 / kTabSplit /
// kTabSplit3): 1024 threads, one CTA per SM, 8 groups of 4 warps each on
// their own unit.  Pairs below the window (cascade cores) read global /
// texture records.
// kLeanTabRecords (cbx_device.cuh): x 64 B = 211,200 B; split: x 32 B / x 24 B

__host__ __device__ __forceinline__ int force_window_lo(int nseg, int tb) {
  const int lo = nseg + 1 - kLeanTabRecords;
  // the split-3 window starts on an even record: its 8-byte qC array is then
  // 16-byte aligned for the bulk copy
  return tb == kTabSplit3 ? ((lo > 0 ? lo : 0) + 1) & ~1 : (lo > 0 ? lo : 0);
}

template <bool FULL, int NT, int TB, bool REV = false>
__global__ void __launch_bounds__(NT, 1) k_force_lean_smem(KP P, int nsb) {
  if (blockIdx.x >= nsb) {
    pdl_wait();
    pdl_trigger();
    // the unused pair partials (read by k_finalize over the full capacity)
    // are zeroed by an extra block, not by a unit CTA
    if (blockIdx.x == nsb) {
      for (int i = nsb + threadIdx.x; i < P.n_pair_part; i += blockDim.x) P.part_pair[i] = 0.0;
    }
    clash_body<1>(P, blockIdx.x - nsb, gridDim.x - nsb);
    return;
  }
  extern __shared__ __align__(16) unsigned char smem_tab[];
  __shared__ int s_slot[8];
  __shared__ int s_ctr;
  double2* T = reinterpret_cast<double2*>(smem_tab);
  const int nseg = P.ff.nseg;  // records 0..nseg (padded)
  if (threadIdx.x == 0) s_ctr = 0;
  // split-3: the window [fw_lo, nseg] minus the gap [fw_gap_lo, fw_gap_lo +
  // fw_gap_n) between two neighbour shells (capi.cu, force_window_setup)
  const int seg_lo = TB == kTabSplit3 ? P.fw_lo : force_window_lo(nseg, TB);
  const int gap_n = TB == kTabSplit3 ? P.fw_gap_n : 0;
  const int nrec = nseg + 1 - seg_lo - gap_n;
  const unsigned tb8 = smem_addr(T) + 16u * (TB == kTabSplit3 ? P.fw_cap : kLeanTabRecords);  // split-3: the qC array
  __shared__ __align__(8) unsigned long long s_mbar;
  if (TB != kTabSmem64) {  // bulk copies of the window's chunks, one thread
    if (threadIdx.x == 0) {
      const unsigned mb = smem_addr(&s_mbar);
      mbar_init(mb);
      if (TB == kTabSplit) {
        mbar_expect_tx(mb, 32u * nrec);
        bulk_stage(smem_addr(T), P.ffz + 4 * (size_t)seg_lo, 32u * nrec, mb);
      } else {
        // records below the gap (n1, even) and above it (n2)
        const int n1 = gap_n ? P.fw_gap_lo - seg_lo : nrec, n2 = nrec - n1;
        const int up = gap_n ? P.fw_gap_lo + gap_n : 0;  // first record above the gap
        const unsigned b1 = (8u * n1 + 15u) & ~15u, b2 = (8u * n2 + 15u) & ~15u;
        mbar_expect_tx(mb, 16u * nrec + b1 + (n2 ? b2 : 0u));
        bulk_stage(smem_addr(T), P.ffzc + 2 * (size_t)seg_lo, 16u * n1, mb);
        bulk_stage(tb8, P.ffqc + seg_lo, b1, mb);
        if (n2) {
          bulk_stage(smem_addr(T) + 16u * n1, P.ffzc + 2 * (size_t)up, 16u * n2, mb);
          bulk_stage(tb8 + 8u * n1, P.ffqc + up, b2, mb);
        }
      }
    }
  } else {
    const double2* src = reinterpret_cast<const double2*>(P.ff.rec + 8 * (size_t)seg_lo);
    for (int q = threadIdx.x; q < 4 * nrec; q += blockDim.x)
      T[smem_slot(q >> 2, q & 3)] = __ldg(src + q);
  }
  for (int i = threadIdx.x; i < 2 * (kMaskBits + 1); i += blockDim.x) {
    const int par = i / (kMaskBits + 1), k = i % (kMaskBits + 1);
    const int n = FULL ? c_full_n[par] : c_half_n[par];
    g_soffs[par][k] = k < n ? (FULL ? c_full[par][k] : c_half[par][k]) : 0;
  }
  __syncthreads();  // the barrier's initialisation is visible
  if (TB != kTabSmem64) mbar_wait0(smem_addr(&s_mbar));
  pdl_wait();
  pdl_trigger();
  if (P.mark_k2 && blockIdx.x == 0 && threadIdx.x == 0) P.st->k2_pending = 1;  // merged kick
  if (FULL) zero_pair_tail(P, nsb);  // no extra blocks in this launch
  if (P.st->err || P.st->n_ovl) return;
  const int group = threadIdx.x >> 7;
  const int lt = threadIdx.x & 127, lane = lt & 31, w = lt >> 5;
  const Geo& G = P.G;
  const int nu = unit_count(G);
  double e = 0.0;
  // (holding the window addresses in registers as k_density_smem does costs
  // this pass more than the rebuilt addresses: force 6.63 vs 6.36 ms, A/B)
  const unsigned tbr = smem_addr(T), tb8r = tb8;
  for (;;) {
    const int u = next_unit(&s_ctr, group, nsb, nu, s_slot, P.unit_rr);
    if (u >= nu) break;
    int c;
    const bool live = unit_cell(G, u, lane, w, c);
    const bool deep = live && unit_deep(G, u, lane, w, FULL);
    for (int par = 0; par < 2; ++par)
      e += force_site_lean<FULL, TB, REV>(P, P.dself, par, live ? (int)(par * G.NC + c) : 0,
                                          live, tbr, seg_lo, near_halo(G, u, w), deep,
                                          tb8r);
  }
  block_partial<NT>(e, P.part_pair);
}

// persistent grid of the 128-thread kernels (density fallback, decision-
// path force pass): resident CTAs, at most one per brick
int fast_grid(const KP& P, bool force, int mode) {
  int per_sm = 0;
  if (force)
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(
        &per_sm, mode ? (const void*)k_force_fast<true, 2> : (const void*)k_force_fast<false, 2>,
        128, 0);
  else
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(
        &per_sm, mode ? (const void*)k_density_fast<true, 4, 4>
                      : (const void*)k_density_fast<false, 4, 4>,
        128, 0);
  int sms = 148;
  int dev = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const int blocks = sms * (per_sm > 0 ? per_sm : 1);
  return max(1, min(blocks, brick_count(P.G)));
}

static int sm_count() {
  int sms = 148, dev = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  return sms;
}

// the shared-memory density pass for one table layout (CMPD, see
// density_site); returns true when the clash-record pass ran in the launch
template <int CMPD>
bool launch_density_smem(const KP& P, int mode, cudaStream_t s) {
  const size_t bytes =
      (size_t)kDensTabRecords * (CMPD == 3 ? 16 : CMPD >= 2 ? 8 : CMPD == 1 ? 24 : 32);
  static bool attr = false;
  if (!attr) {
    for (const void* k : {(const void*)k_density_smem<false, 1, 1024, false, CMPD>,
                          (const void*)k_density_smem<true, 1, 1024, false, CMPD>,
                          (const void*)k_density_smem<false, 1, 1024, true, CMPD>,
                          (const void*)k_density_smem<false, 1, 896, false, CMPD>})
      cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes);
    attr = true;
  }
  const int g = max(1, min(sm_count(), unit_count(P.G)));
  static const int nt_env = ab_flag("CBX_DENSITY_NT", 0);  // overrides the rule below
  // at most 7 units per CTA: 7 groups with 72 registers (as the force pass)
  const int nt = nt_env ? nt_env : ((unit_count(P.G) + g - 1) / g <= 7 ? 896 : 1024);
  if (nt == 896 && !mode && !P.rev.on) {
    launch_pdl(k_density_smem<false, 1, 896, false, CMPD>, g + 4, 896, bytes, s, P, g);
    return true;
  }
  if (mode) launch_pdl(k_density_smem<true, 1, 1024, false, CMPD>, g, 1024, bytes, s, P, g);
  else if (P.rev.on)
    launch_pdl(k_density_smem<false, 1, 1024, true, CMPD>, g + 4, 1024, bytes, s, P, g);
  else launch_pdl(k_density_smem<false, 1, 1024, false, CMPD>, g + 4, 1024, bytes, s, P, g);
  return !mode;
}
int density_table_mode(const KP& P) {
  // default: the unrolled inner loop (needs the inner offsets in one 64-bit
  // mask word) with the compressed records where the local fp32 guard held
  // (P.fdc: [D C] by texture, fp32 [A B] in shared memory -- 4), else fp64
  // [A B] in shared memory and [C D] by texture (3).  Measured at config 5
  // (A/B, same box): 4: 4.31 ms; both halves by texture: 4.33; 3: 4.63;
  // fp64 both by texture: 4.67; 2 (round-2 loop, tables of 4): 4.54
  static const int tm = ab_flag("CBX_DENSITY_TAB", -1);
  if (tm < 0) return P.nin64 ? (P.fdc ? 4 : 3) : (P.fdc ? 2 : 0);
  if (tm == 3) return P.nin64 ? 3 : 0;
  if (tm == 4) return P.nin64 && P.fdc ? 4 : 0;
  return tm && P.fdc ? tm : 0;
}

// density pass: the lean 1024-thread kernel with the rho-spline window in
// shared memory (default); CBX_DENSITY_SMEM=0 (A/B build) selects the
// 128-thread batched kernel.  Returns true when the clash-record pass ran in
// the same launch.
bool launch_density_fast(const KP& P, int mode, int grid, cudaStream_t s) {
  static const int dsm = ab_flag("CBX_DENSITY_SMEM", 1);
  if (dsm) {
    const int tm = density_table_mode(P);
    if (tm == 3) return launch_density_smem<3>(P, mode, s);
    if (tm == 4) return launch_density_smem<4>(P, mode, s);
    if (tm == 2) return launch_density_smem<2>(P, mode, s);
    if (tm == 1) return launch_density_smem<1>(P, mode, s);
    return launch_density_smem<0>(P, mode, s);
  }
  const int ex = mode ? 0 : kClashBlocks128;  // fused clash pass (Newton-3)
  if (mode) k_density_fast<true, 4, 4><<<grid, 128, 0, s>>>(P, grid);
  else k_density_fast<false, 4, 4><<<grid + ex, 128, 0, s>>>(P, grid);
  return ex != 0;
}

// force pass: with a valid pair mask the lean mask-replay kernel with the
// force spline window in shared memory (+ texture chunks); otherwise
// (positions changed since the density pass) the decision path, which
// re-derives every pair
template <int TB>
void launch_force_lean(const KP& P, int mode, cudaStream_t s) {
  const size_t bytes =
      (size_t)(TB == kTabSplit3 ? P.fw_cap : kLeanTabRecords) * kTabSmemBytes[TB] + 16;
  static size_t attr_bytes = 0;  // the largest size the kernels were set up for
  if (attr_bytes < bytes) {
    attr_bytes = bytes;
    // default carveout: the driver takes the smallest shared-memory split
    // that fits the table and leaves the rest of the SM's 256 KB as L1 for
    // the partner gathers and the texture fetches
    for (const void* k : {(const void*)k_force_lean_smem<false, 1024, TB, false>,
                          (const void*)k_force_lean_smem<true, 1024, TB, false>,
                          (const void*)k_force_lean_smem<false, 1024, TB, true>,
                          (const void*)k_force_lean_smem<false, 896, TB, false>,
                          (const void*)k_force_lean_smem<false, 896, TB, true>})
      cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes);
  }
  const int g = max(1, min(sm_count(), unit_count(P.G)));
  // at most 7 units per CTA (one wave, e.g. config 2): 7 groups of 128
  // threads with 72 registers instead of 8 with 64 (CBX_FORCE_NT overrides)
  static const int nt_env = ab_flag("CBX_FORCE_NT", 0);
  // more than 7 units per CTA: 1024 threads (64 registers, some spills) --
  // since the round-robin unit batches and the predicated idle gathers,
  // 7.12 vs 7.44 ms at config 5 (steps 4-13; 7.36 vs 7.72 at steps 51-60);
  // round 1's order measured 896 ahead (7.27 vs 7.38-7.54)
  const int nt = nt_env ? nt_env : ((unit_count(P.G) + g - 1) / g <= 7 ? 896 : 1024);
  if (nt == 896 && !mode) {
    if (P.rev.on)
      launch_pdl(k_force_lean_smem<false, 896, TB, true>, g + 4, 896, bytes, s, P, g);
    else launch_pdl(k_force_lean_smem<false, 896, TB, false>, g + 4, 896, bytes, s, P, g);
    return;
  }
  if (mode) launch_pdl(k_force_lean_smem<true, 1024, TB, false>, g, 1024, bytes, s, P, g);
  else if (P.rev.on)
    launch_pdl(k_force_lean_smem<false, 1024, TB, true>, g + 4, 1024, bytes, s, P, g);
  else launch_pdl(k_force_lean_smem<false, 1024, TB, false>, g + 4, 1024, bytes, s, P, g);
}
int force_table_mode() {
  static const int tb = ab_flag("CBX_FORCE_TAB", kTabSplit3);
  return tb;
}
bool launch_force_fast(const KP& P, int mode, int grid, cudaStream_t s) {
  if (P.use_mask) {
    const int tb = force_table_mode();
    if (tb == kTabSplit3) launch_force_lean<kTabSplit3>(P, mode, s);
    else if (tb == kTabSmem64) launch_force_lean<kTabSmem64>(P, mode, s);
    else launch_force_lean<kTabSplit>(P, mode, s);
    return !mode;
  }
  if (mode) k_force_fast<true, 2><<<grid, 128, 0, s>>>(P);
  else k_force_fast<false, 2><<<grid, 128, 0, s>>>(P);
  return false;
}
