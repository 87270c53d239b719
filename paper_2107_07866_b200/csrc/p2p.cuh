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

// thread 0 of the block: wait until every flag reaches `epoch` (or time out)
__device__ inline bool wait_flags(const KP& P, const unsigned long long* const* flags, int nflags,
                           unsigned long long epoch) {
  __shared__ int s_ok;
  if (threadIdx.x == 0) {
    int ok = 1;
    const unsigned long long t0 = global_ns();
    for (int f = 0; f < nflags && ok; ++f)
      while (ld_acquire_sys(flags[f]) < epoch) {
        if (global_ns() - t0 > kWaitNs) {
          set_error(P.st, CBX_RUNTIME);
          ok = 0;
          break;
        }
        __nanosleep(200);
      }
    s_ok = ok;
  }
  __syncthreads();
  return s_ok != 0;
}

// all blocks done writing -> the last one bumps the epoch and raises the
// peers' flags.  One system-scope fence per exchange: each block publishes
// its stores at GPU scope (bar.sync + fence + arrival counter, the grid-sync
// pattern); the last block's fence.sc.sys is cumulative over everything it
// has observed, then the flags are plain system-scope stores.
__device__ inline void signal_peers(const P2PLinks& L, int kind) {
  __syncthreads();
  if (threadIdx.x != 0) return;
  __threadfence();
  const unsigned t = atomicAdd(&L.done[kind], 1u);
  if (t != gridDim.x - 1) return;
  __threadfence();
  L.done[kind] = 0;
  const unsigned long long e = L.epoch[kind] + 1;
  L.epoch[kind] = e;
  __threadfence_system();
  st_relaxed_sys(L.flag_dst[kind][0], e);
  st_relaxed_sys(L.flag_dst[kind][1], e);
}

// the consumer of those partials: every block waits for both neighbours'
// flags of exchange `kind` to reach this rank's own epoch (bumped by its own
// pass, earlier in the stream)
__device__ __forceinline__ bool rev_wait(const KP& P, int kind) {
  const P2PLinks& L = *P.lk;
  const unsigned long long* fl[2] = {L.flag_src[kind][0], L.flag_src[kind][1]};
  return wait_flags(P, fl, 2, *(volatile unsigned long long*)&L.epoch[kind]);
}

}  // namespace cbx
