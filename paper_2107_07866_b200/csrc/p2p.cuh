// p2p.cuh -- peer-memory primitives of the slab exchange (system-scope
// flags over NVLink) and the deterministic StepState reduction.
#pragma once

#include "cbx_device.cuh"

namespace cbx {

__device__ __forceinline__ unsigned long long ld_acquire_sys(const unsigned long long* p) {
  unsigned long long v;
  asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ unsigned long long global_ns() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
constexpr unsigned long long kWaitNs = 20ull * 1000000000ull;  // a dead peer, not a slow one

__device__ __forceinline__ void st_relaxed_sys(unsigned long long* p, unsigned long long v) {
  asm volatile("st.relaxed.sys.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}

// StepState sums over all ranks, deterministic: every rank stores its
// {pair, embedding, kinetic, max_speed} into slot `rank` of every rank,
// then sums the slots in rank order
__device__ inline void p2p_reduce_thread(const KP& P, const P2PLinks& L, int energies,
                                         int kinetic) {
  DevStatus* st = P.st;
  const unsigned long long e = L.epoch[5] + 1;
  L.epoch[5] = e;
  const double v[4] = {st->pair, st->embedding, st->kinetic, st->max_speed};
  for (int q = 0; q < L.nranks; ++q) {
    double* slot = L.red_dst[q] + 4 * L.rank;
    for (int i = 0; i < 4; ++i) slot[i] = v[i];
  }
  __threadfence_system();
  for (int q = 0; q < L.nranks; ++q) st_relaxed_sys(L.red_flag_dst[q] + L.rank, e);
  const unsigned long long t0 = global_ns();
  for (int q = 0; q < L.nranks; ++q)
    while (ld_acquire_sys(L.red_flag_src + q) < e) {
      if (global_ns() - t0 > kWaitNs) {
        set_error(st, CBX_RUNTIME);
        return;
      }
      __nanosleep(100);
    }
  double a = 0.0, b = 0.0, k = 0.0, m = 0.0;
  for (int q = 0; q < L.nranks; ++q) {
    const double* s = L.red_src + 4 * q;
    a += __ldcg(s + 0);
    b += __ldcg(s + 1);
    k += __ldcg(s + 2);
    m = fmax(m, __ldcg(s + 3));
  }
  if (energies) {
    st->pair = a;
    st->embedding = b;
  }
  if (kinetic) {
    st->kinetic = k;
    st->max_speed = m;
    if (st->adaptive) {  // adaptive_dt on the global max speed, sim.cpp:94-98
      double dt = st->dt_max;
      if (m > 0.0) dt = fmin(dt, xdiv(st->max_disp, m));
      st->dt_next = fmax(dt, 1e-7);
    }
  }
}

}  // namespace cbx
