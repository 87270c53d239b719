// finalize.cuh -- the StepState sums (sim.cpp:237-246, 262-270): deterministic
// sums of the per-block / per-record partials into DevStatus, and the
// deferred form run by an otherwise idle block of a later kernel.  Header
// templates: store_kernels.cu (k_kick2, k_kick_drift, k_finalize*) and the
// density pass (eam_kernels.cu) each instantiate their own copy.
#pragma once
#include "cbx_device.cuh"
#include "p2p.cuh"

namespace cbx {

// deterministic sums of the per-block / per-record partials into StepState
// (fixed per-thread order, four independent accumulators for load
// parallelism, then a fixed block tree)
// bad_at: the outcome of the step whose sums these are, captured when they
// were deferred (fin_bad); -1 reads the live status words (the sums of the
// step that just ended).  Read once by thread 0 and shared, so the whole
// block takes the same branch.
template <int NT>
__device__ __noinline__ void finalize_body(const KP& P, int stepping, int energies, const double* pe, int n_emb,
                              const double* pp, int n_pairp, int n_ke, int clash_slots = 0,
                              int bad_at = -1) {
  __shared__ double sh[4][32];
  __shared__ int s_bad;
  DevStatus* st = P.st;
  if (threadIdx.x == 0) s_bad = bad_at >= 0 ? bad_at : (st->err | st->n_ovl);
  const int nc = st->n_clash;
  double s_dt = 0.0, s_t = 0.0, s_dtmax = 0.0, s_disp = 0.0;
  long long s_step = 0;
  int s_adapt = 0;
  if (threadIdx.x == 0) {
    s_dt = st->dt_next;
    s_t = st->t;
    s_step = st->step;
    s_adapt = st->adaptive;
    s_dtmax = st->dt_max;
    s_disp = st->max_disp;
  }
  // one pass over every partial array, all loads of a round independent
  double ea[4] = {0, 0, 0, 0}, ep[4] = {0, 0, 0, 0}, ek[4] = {0, 0, 0, 0},
         em[4] = {0, 0, 0, 0};
  const int ne = energies ? n_emb : 0, np = energies ? n_pairp : 0;
  const int nk = stepping >= 0 ? n_ke : 0;
  const int n = max(max(ne, np), nk);
  for (int i0 = threadIdx.x; i0 < n; i0 += 4 * NT) {
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const int i = i0 + u * NT;
      if (i < ne) ea[u] += pe[i];
      if (i < np) ep[u] += pp[i];
      if (i < nk) {  // written by other blocks of a fused k_kick2: L2 loads
        ek[u] += __ldcg(P.part_ke + i);
        em[u] = fmax(em[u], __ldcg(P.part_vmax + i));
      }
    }
  }
  if (clash_slots > 0 && threadIdx.x < clash_slots) {  // the records' block sums
    const int q = P.n_part - clash_slots + threadIdx.x;
    if (energies) {
      ea[1] += __ldcg(pe + q);
      ep[1] += __ldcg(pp + q);
    }
    if (stepping >= 0) {
      ek[1] += __ldcg(P.part_ke + q);
      em[1] = fmax(em[1], __ldcg(P.part_vmax + q));
    }
  }
  for (int i = threadIdx.x; clash_slots == 0 && i < nc; i += NT) {
    if (energies) {
      ea[0] += P.cl.e_emb[i];
      ep[0] += P.cl.e_pair[i];
    }
    if (stepping >= 0) {
      const double v2 = __ldcg(P.cl.v2 + i);
      ek[0] += v2;
      em[0] = fmax(em[0], v2);
    }
  }
  __syncthreads();
  if (s_bad) return;
  double v[4] = {(ea[0] + ea[1]) + (ea[2] + ea[3]), (ep[0] + ep[1]) + (ep[2] + ep[3]),
                 (ek[0] + ek[1]) + (ek[2] + ek[3]), fmax(fmax(em[0], em[1]), fmax(em[2], em[3]))};
  for (int o = 16; o > 0; o >>= 1) {
    v[0] += __shfl_xor_sync(0xffffffffu, v[0], o);
    v[1] += __shfl_xor_sync(0xffffffffu, v[1], o);
    v[2] += __shfl_xor_sync(0xffffffffu, v[2], o);
    v[3] = fmax(v[3], __shfl_xor_sync(0xffffffffu, v[3], o));
  }
  const int w = threadIdx.x >> 5;
  if ((threadIdx.x & 31) == 0)
    for (int q = 0; q < 4; ++q) sh[q][w] = v[q];
  __syncthreads();
  if (threadIdx.x != 0) return;
  double r[4] = {0, 0, 0, 0};
  for (int i = 0; i < NT / 32; ++i) {
    r[0] += sh[0][i];
    r[1] += sh[1][i];
    r[2] += sh[2][i];
    r[3] = fmax(r[3], sh[3][i]);
  }
  if (energies) {
    st->embedding = r[0];
    st->pair = r[1];
  }
  if (stepping >= 0) {  // 1: completed a step, 0: measure only
    st->kinetic = xmul(xmul(xmul(0.5, P.mass), r[2]), P.mv2);  // sim.cpp:269
    st->max_speed = sqrt(r[3]);
    const double vmax = sqrt(r[3]);
    if (stepping == 1) {
      st->step = s_step + 1;
      st->t = xadd(s_t, s_dt);
      st->dt = s_dt;
    }
    if (s_adapt) {  // adaptive_dt, sim.cpp:94-98
      double dt = s_dtmax;
      if (vmax > 0.0) dt = fmin(dt, xdiv(s_disp, vmax));
      st->dt_next = fmax(dt, 1e-7);
    }
  }
}


// the deferred StepState finalize (fin_pending, with its partial counts)
template <int NT>
__device__ void finalize_pending(const KP& P) {
  DevStatus* st = P.st;
  if (!st->fin_pending) return;
  finalize_body<NT>(*P.dself, st->fin_stepping, st->fin_energies, P.part_emb, st->fin_nemb,
                    P.part_pair, st->fin_npp, st->fin_nke, st->fin_clash, st->fin_bad);
  __syncthreads();
  if (threadIdx.x == 0) {
    // slab ranks on the peer-memory transport: the StepState sums over the
    // ranks (every rank's deferred finalize reaches this point in the same
    // kernel of the same step; also after an error, so the ranks stay in step)
    if (st->fin_reduce && P.lk) {
      __threadfence();
      p2p_reduce_thread(*P.dself, *P.lk, st->fin_energies, st->fin_stepping >= 0);
    }
    st->fin_pending = 0;
  }
}

}  // namespace cbx
