// capi.cu -- the C ABI (include/cascade_b200.h): context lifetime, store
// transfer, and the launch sequences of eval_forces and Simulation::step.
#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <memory>
#include <string>
#include <thread>
#include <tuple>
#include <vector>

#include "cbx_comm.h"
#include "cbx_device.cuh"
#include "cbx_host.h"

using namespace cbx;

// one in-flight snapshot: device pack buffer, page-locked host copy, the
// events of the pack and the D2H, and the thread formatting the file
struct SnapSlot {
  double4* dev = nullptr;
  double4* host = nullptr;
  size_t bytes = 0;
  cudaEvent_t packed = nullptr, copied = nullptr;
  std::thread writer;
  std::string error;
};

struct cbx_ctx {
  std::vector<double> shells;  // distinct lattice distances of the stencil sites within the cutoff
  int device = 0;
  cudaStream_t stream = nullptr;
  cbx_box box{};
  Geo G{};
  long long S = 0;
  Potential pot;
  Offsets offs;
  bool cutoff_ok = true;
  KP P{};
  int mode = CBX_STENCIL_NEWTON3;
  std::string err;
  DevStatus hst{};
  unsigned long long* d_defects = nullptr;
  std::vector<void*> allocs;
  std::vector<cudaTextureObject_t> textures;
  SnapSlot snap[2];  // asynchronous snapshots (double-buffered)
  int snap_next = 0;
  cudaStream_t snap_stream = nullptr;
  cudaGraphExec_t step_graph = nullptr;
  // single-step calls (cbx_step(dt, 1), the Simulation::step loop) use a
  // graph that completes the step itself: no pending kick or sums to flush
  cudaGraphExec_t step_graph1 = nullptr;
  uint64_t graph1_launches = 0;
  bool single = false;
  bool g_defer = false, g_merge = false;  // how step_graph was captured
  bool t_defer = false, t_merge = false;  // how the timed graphs were captured
  uint64_t g_launches = 0, t_launches = 0;  // kernels per launch of each
  cudaGraphExec_t timed_graph = nullptr;
  void* flush_buf = nullptr;
  // deferred StepState finalize (fixed dt, single box): graphs captured with
  // it; a pending finalize may exist on the device; its pair partial count
  bool graph_defer = false, fin_maybe = false;
  // merged kick: the last step's second half kick may be pending on the
  // device (runs in the next step's k_kick_drift, or before the host reads)
  bool graph_merge = false, k2_maybe = false, merge_now = false;
  // the host copy of the status equals the device's and nothing ran since
  // (set by cbx_step on success, cleared on entry to every C-ABI call):
  // a following cbx_step skips its opening status round trip
  bool st_fresh = false, st_was_fresh = false;
  int fin_npp = 0;
  size_t flush_bytes = 0;
  bool use_graph = true;
  bool timing = false;
  bool timing_lite = false;   // capture only the force-kernel events
  bool bench_phases = false;  // cbx_bench_steps: per-phase events inside the graph
  cudaGraphExec_t timed_lite = nullptr;
  cudaEvent_t ev_outer[2]{};
  cudaEvent_t ev[8]{};
  double t_ms[8]{};
  uint64_t launches = 0;
  int n_ghost = 0;
  bool fast_ok = true;
  bool fp32_density = false;  // compressed density records in use (local fp32 guard held)
  bool mask_valid = false;
  bool clash_rho_zero = false;  // the last clash-image pass zeroed the records' rho
  bool clash_f_zero = false;    // the last embed pass zeroed the records' forces
  bool acc_rho_zero = false;    // kick_drift of this step cleared rho (single box)
  bool acc_frc_zero = false;    // ... and the forces
  // z-slab decomposition
  int rank = 0, nranks = 1;
  cbx_box gbox{};       // the global box (slab ranks)
  int rem_base[2] = {0, 0};
  int* d_rem_base = nullptr;  // pmask matches the current positions (density ran last)
  double band = 0.0;
  // this context's stencil tables (device deltas depend on its box), kept
  // to re-bind the device's __constant__ copy when contexts share a GPU
  std::vector<int> c_hd[2], c_fd[2];
  std::vector<long long> c_ff[2];
  int c_hin[2] = {0, 0}, c_fin[2] = {0, 0};
  bool const_ready = false;
  // in-graph NCCL exchange of a slab rank (cbx_slab_comm_init)
  ncclComm_t comm = nullptr;
  unsigned char* sbuf[2] = {nullptr, nullptr};
  unsigned char* rbuf[2] = {nullptr, nullptr};
  double* d_red = nullptr;
  uint64_t graph_launches = 16;  // kernels per captured step
  // host-transfer staging (reference id order), allocated on first use
  double *stage_pos = nullptr, *stage_vel = nullptr, *stage_frc = nullptr,
         *stage_rho = nullptr, *stage_df = nullptr;
  unsigned long long* stage_tag = nullptr;
  unsigned char *stage_valid = nullptr, *stage_ghost = nullptr;
  // peer-memory exchange (cbx_slab_p2p_init): this rank's receive region,
  // the neighbours' regions mapped through CUDA IPC
  unsigned char* p2p_region = nullptr;
  size_t p2p_bytes = 0;
  std::vector<void*> p2p_opened;
  P2PLinks links{};
  P2PLinks* d_links = nullptr;  // device copy (the finalize kernel's reduction)
  // defect series of the last cbx_run (sim.h:54)
  std::vector<double> ser_t;
  std::vector<long> ser_d;
  bool p2p = false;
  bool rev_mapped = false;  // the neighbours' rho / force arrays are mapped (KP::rev)
  // reverse halos as staged exchanges by default; cbx_slab_p2p_set_fused(1)
  // adds the partials straight into the neighbours' memory from the passes
  // (measured at config 5 on one GPU: the fused pass variants cost 0.6 ms per
  // step more than the two staged exchanges, 14.04 vs 13.50 ms)
  bool fused_off = true;

  // device bytes by structure (cbx_memory_report): the category the next
  // allocations are charged to
  int mem_cat = 0;
  size_t mem_bytes[CBX_MEM_CATEGORIES] = {};

  template <class T>
  T* alloc(size_t n) {
    void* p = nullptr;
    if (cudaMalloc(&p, std::max<size_t>(n, 1) * sizeof(T)) != cudaSuccess)
      raise(CBX_CUDA, "cudaMalloc of " + std::to_string(n * sizeof(T)) + " bytes failed");
    mem_bytes[mem_cat] += std::max<size_t>(n, 1) * sizeof(T);
    allocs.push_back(p);
    return static_cast<T*>(p);
  }
};

namespace {

const char* kBuild = "cascade_b200 sm_100a fp64 EAM (abi " "1" ")";

void cuda_check(cudaError_t e, const char* what) {
  if (e != cudaSuccess) raise(CBX_CUDA, std::string(what) + ": " + cudaGetErrorString(e));
}

// The stencil deltas live in __constant__ memory, one copy per device; the
// context whose tables are resident is recorded here and every entry point
// re-binds before it launches (contexts sharing one GPU -- virtual slab
// ranks, several boxes -- are used from one host thread at a time).
cbx_ctx* g_const_owner[64] = {};

void bind_constants(cbx_ctx* c) {
  if (!c->const_ready || c->device < 0 || c->device >= 64) return;
  if (g_const_owner[c->device] == c) return;
  cudaSetDevice(c->device);
  cudaDeviceSynchronize();  // other contexts' work finished with the old tables
  const int* hp[2] = {c->c_hd[0].data(), c->c_hd[1].data()};
  const int* fp[2] = {c->c_fd[0].data(), c->c_fd[1].data()};
  const long long* fl[2] = {c->c_ff[0].data(), c->c_ff[1].data()};
  const int hn[2] = {(int)c->c_hd[0].size(), (int)c->c_hd[1].size()};
  const int fn[2] = {(int)c->c_fd[0].size(), (int)c->c_fd[1].size()};
  upload_offsets(hp, hn, fp, fn, fl, c->c_hin, c->c_fin, c->stream);
  if (cudaStreamSynchronize(c->stream) != cudaSuccess)
    raise(CBX_CUDA, "offset table upload failed");
  g_const_owner[c->device] = c;
}

template <class F>
cbx_status guarded(cbx_ctx* c, F&& f) {
  try {
    if (c) {
      c->st_was_fresh = c->st_fresh;
      c->st_fresh = false;
      bind_constants(c);
    }
    f();
    if (c) c->err.clear();
    return CBX_OK;
  } catch (const Status& s) {
    if (c) c->err = s.what();
    set_thread_error(s.what());
    return s.code;
  } catch (const std::invalid_argument& e) {
    if (c) c->err = e.what();
    set_thread_error(e.what());
    return CBX_INVALID_ARGUMENT;
  } catch (const std::exception& e) {
    if (c) c->err = e.what();
    set_thread_error(e.what());
    return CBX_RUNTIME;
  }
}

void alloc_clash(cbx_ctx* c, Clash& A, int cap) {
  A.key = c->alloc<long long>(cap);
  A.hkey = c->alloc<long long>(cap);
  A.gf = c->alloc<unsigned char>(cap);
  A.src = c->alloc<int>(cap);
  A.px = c->alloc<double>(cap);
  A.py = c->alloc<double>(cap);
  A.pz = c->alloc<double>(cap);
  A.vx = c->alloc<double>(cap);
  A.vy = c->alloc<double>(cap);
  A.vz = c->alloc<double>(cap);
  A.fx = c->alloc<double>(cap);
  A.fy = c->alloc<double>(cap);
  A.fz = c->alloc<double>(cap);
  A.rho = c->alloc<double>(cap);
  A.df = c->alloc<double>(cap);
  A.e_emb = c->alloc<double>(cap);
  A.e_pair = c->alloc<double>(cap);
  A.v2 = c->alloc<double>(cap);
  A.tag = c->alloc<unsigned long long>(cap);
}

Tab upload_tab(cbx_ctx* c, const Spline& s) {
  Tab t{};
  double* d = c->alloc<double>(s.seg.size());
  cuda_check(cudaMemcpy(d, s.seg.data(), s.seg.size() * sizeof(double), cudaMemcpyHostToDevice),
             "table upload");
  t.seg = d;
  t.x0 = s.x0;
  t.h = s.h;
  t.ih = 1.0 / s.h;
  t.xl = s.x_last();
  t.nseg = (int)s.nseg();
  return t;
}

bool has_transport(const cbx_ctx* c);
bool want_merge(const cbx_ctx* c);

void sync_status(cbx_ctx* c) {
  if (c->fin_maybe) {  // the last step's StepState sums before the host reads them
    launch_finalize_pending(c->P, c->stream);
    c->launches += 1;
    c->fin_maybe = false;
  }
  if (c->k2_maybe) {  // the last step's second half kick (+ its StepState sums)
    if (has_transport(c)) {  // slab rank: after the neighbours' force partials,
      KP q = c->P;           // then the sums and the cross-rank reduction
      q.rev_wait = c->P.rev.on ? 4 : 0;
      launch_kick2(q, 1, -2, 0, c->stream);
      launch_finalize(c->P, 1, 1, c->stream, c->d_links);
      c->launches += 2;
    } else {
      launch_kick2(c->P, 1, 1, 1, c->stream, 1, c->fin_npp);
      c->launches += 1;
    }
    c->k2_maybe = false;
  }
  cuda_check(cudaMemcpyAsync(&c->hst, c->P.st, sizeof(DevStatus), cudaMemcpyDeviceToHost,
                             c->stream),
             "status readback");
  cuda_check(cudaStreamSynchronize(c->stream), "stream synchronize");
  cuda_check(cudaGetLastError(), "kernel launch");
}

// turn a device error into the reference's exception text; clears it
void raise_device_error(cbx_ctx* c, bool in_step) {
  DevStatus& h = c->hst;
  if (!h.err && !h.n_ovl) return;
  std::string msg;
  cbx_status code;
  if (h.err) {
    code = (cbx_status)h.err;
    if (h.err == CBX_DOMAIN) {
      msg = "nearest_site: position (" + std::to_string(h.err_pos[0]) + ", " +
            std::to_string(h.err_pos[1]) + ", " + std::to_string(h.err_pos[2]) +
            ") outside the ghost-inclusive box volume";
    } else if (h.err == CBX_LOGIC) {
      msg = "canonicalize_positions: wrap did not converge";
    } else if (h.err == CBX_INVALID_ARGUMENT) {
      msg = "unsupported store state: a clash bucket over a vacant lattice site";
    } else {
      msg = "clash list capacity exceeded";
    }
  } else {
    code = CBX_RUNTIME;
    const int n = std::min(h.n_ovl, kMaxOverlapRecords);
    int best = 0;
    for (int i = 1; i < n; ++i)
      if (h.ovl_key[i] < h.ovl_key[best]) best = i;
    char buf[160];
    std::snprintf(buf, sizeof buf, "atoms %llu and %llu overlap (separation %.3e A)",
                  h.ovl_a[best], h.ovl_b[best], std::sqrt(h.ovl_r2[best]));
    msg = buf;
    if (in_step) {  // sim.cpp:226-231: ++step happened before refresh_forces threw
      h.step += 1;
      msg = "step " + std::to_string(h.step) + ": " + msg;
    }
  }
  h.err = 0;
  h.n_ovl = 0;
  h.n_mov = 0;
  h.halt = 0;
  cudaMemcpyAsync(c->P.st, &h, sizeof(DevStatus), cudaMemcpyHostToDevice, c->stream);
  cudaStreamSynchronize(c->stream);
  raise(code, msg);
}

void write_status(cbx_ctx* c) {
  cuda_check(cudaMemcpyAsync(c->P.st, &c->hst, sizeof(DevStatus), cudaMemcpyHostToDevice,
                             c->stream),
             "status upload");
}

// ---- launch sequences ----------------------------------------------------
bool g_capturing = false;
void ev_mark(cbx_ctx* c, int i) {
  // inside a capture the record must become an external event-record node;
  // the lean timed graph keeps only the force-kernel bracket (6, 7)
  if (c->timing && (!c->timing_lite || i >= 6))
    cudaEventRecordWithFlags(c->ev[i], c->stream, g_capturing ? cudaEventRecordExternal : 0);
}

void seq_fill_ghosts(cbx_ctx* c, bool zero_rho = false) {
  c->mask_valid = false;
  launch_ghost_fill(c->P, c->stream);
  launch_clash_images(c->P, c->stream, zero_rho ? 1 : 0);
  c->clash_rho_zero = zero_rho;
  c->launches += 2;
}
void seq_density(cbx_ctx* c) {
  // on the step path the brick counter was reset by k_clash_images and rho
  // by k_kick_drift; standalone calls clear them here
  if (!c->clash_rho_zero) cudaMemsetAsync(c->P.work, 0, sizeof(int), c->stream);
  if (c->mode != CBX_STENCIL_FULL && !c->acc_rho_zero)
    cudaMemsetAsync(c->P.rho, 0, c->S * sizeof(double), c->stream);
  c->acc_rho_zero = false;
  if (!c->clash_rho_zero) {
    launch_clash_zero(c->P, 0, c->stream);
    c->launches += 1;
  }
  c->clash_rho_zero = false;
  if (!launch_density(c->P, c->mode, c->stream)) {
    launch_clash_density(c->P, c->stream);
    c->launches += 1;
  }
  c->launches += 1;
  c->mask_valid = c->mode != CBX_STENCIL_REFERENCE && c->P.pmask != nullptr;
}
void seq_embed(cbx_ctx* c, int rev_wait = 0) {
  KP q = c->P;
  q.rev_wait = rev_wait;  // the neighbours' density partials arrive first
  launch_embed(q, c->stream, c->mode == CBX_STENCIL_REFERENCE);
  c->clash_f_zero = true;
  c->launches += 1;
}
void seq_force(cbx_ctx* c) {
  // the embedding pass resets the brick counter and the clash records'
  // forces; kick_drift of a step cleared the slot forces
  if (!c->clash_f_zero) cudaMemsetAsync(c->P.work + 1, 0, sizeof(int), c->stream);
  if (c->mode != CBX_STENCIL_FULL && !c->acc_frc_zero)
    cudaMemsetAsync(c->P.frc, 0, 3 * c->S * sizeof(double), c->stream);
  c->acc_frc_zero = false;
  if (!c->clash_f_zero) {
    launch_clash_zero(c->P, 1, c->stream);
    c->launches += 1;
  }
  c->clash_f_zero = false;
  KP q = c->P;
  q.use_mask = c->mask_valid ? 1 : 0;
  q.mark_k2 = c->merge_now && q.use_mask ? 1 : 0;
  ev_mark(c, 6);  // the force kernel alone (roofline of the dominant kernel)
  const bool fused = launch_force(q, c->mode, c->stream);
  ev_mark(c, 7);
  if (!fused) {
    launch_clash_force(c->P, c->stream);
    c->launches += 1;
  }
  c->launches += 1;
}
// ---- z-slab ranks: exchanges and reductions inside the step (NCCL) -------
// Both halves of one exchange go out in one NCCL group: my "down" packet to
// the rank below (it arrives there as "from above") and my "up" packet to the
// rank above.  Messages have a fixed size (slab_msg_bytes), so the sequence
// is capturable; with one rank both peers are this rank (self send/recv).
bool has_transport(const cbx_ctx* c) { return c->comm != nullptr || c->p2p; }
// the RHO / FRC exchanges fused into the passes (peer memory, Newton-3,
// neighbours' accumulators mapped); CBX_P2P_FUSED=0 keeps the staged exchanges
bool rev_fused(const cbx_ctx* c) {
  static const bool on = ab_flag("CBX_P2P_FUSED", 1) != 0;
  return on && c->p2p && c->rev_mapped && !c->fused_off && c->mode == CBX_STENCIL_NEWTON3;
}

void slab_exchange(cbx_ctx* c, int kind) {
  if (c->p2p) {  // fused: pack into the neighbours' memory, wait, unpack
    const long long gs_lo = (kind == 1 && c->rank == 0) ? -1 : 0;
    const long long gs_hi = (kind == 1 && c->rank == c->nranks - 1) ? 1 : 0;
    c->launches += launch_p2p_exchange(c->P, c->links, kind, gs_lo, gs_hi, c->d_rem_base,
                                       c->stream);
    return;
  }
  const NcclApi& N = nccl();
  const long long m = slab_msg_bytes(c->P, kind);
  launch_pack(c->P, kind, -1, c->sbuf[0], m, c->stream);
  launch_pack(c->P, kind, +1, c->sbuf[1], m, c->stream);
  const int lo = (c->rank + c->nranks - 1) % c->nranks, hi = (c->rank + 1) % c->nranks;
  nccl_check(N.group_start(), "ncclGroupStart");
  nccl_check(N.send(c->sbuf[0], (size_t)m, ncclUint8, lo, c->comm, c->stream), "ncclSend");
  nccl_check(N.recv(c->rbuf[1], (size_t)m, ncclUint8, hi, c->comm, c->stream), "ncclRecv");
  nccl_check(N.send(c->sbuf[1], (size_t)m, ncclUint8, hi, c->comm, c->stream), "ncclSend");
  nccl_check(N.recv(c->rbuf[0], (size_t)m, ncclUint8, lo, c->comm, c->stream), "ncclRecv");
  nccl_check(N.group_end(), "ncclGroupEnd");
  // position halos crossing the global z boundary are periodic images
  const long long gs_lo = (kind == 1 && c->rank == 0) ? -1 : 0;
  const long long gs_hi = (kind == 1 && c->rank == c->nranks - 1) ? 1 : 0;
  launch_unpack(c->P, kind, -1, c->rbuf[0], gs_lo, c->d_rem_base + 0, c->stream);
  launch_unpack(c->P, kind, +1, c->rbuf[1], gs_hi, c->d_rem_base + 1, c->stream);
  c->launches += (kind == 1 || kind == 3) ? 8 : 4;
}

// a reverse halo (2 RHO, 4 FRC): with the fused path the pass already
// added into the neighbours' memory -- only raise their flags
void slab_reverse(cbx_ctx* c, int kind) {
  if (c->P.rev.on) {
    launch_rev_signal(c->P, kind, c->stream);
    c->launches += 1;
    return;
  }
  slab_exchange(c, kind);
}

// StepState sums over ranks: energies (pair, embedding) and/or kinetic +
// max speed (sum / max), then adaptive dt from the global max speed
void slab_reduce(cbx_ctx* c, bool energies, bool kinetic) {
  if (c->p2p) {
    launch_p2p_reduce(c->P, c->links, energies, kinetic, c->stream);
    c->launches += 1;
    return;
  }
  const NcclApi& N = nccl();
  launch_slab_red_in(c->P, c->d_red, c->stream);
  double* first = energies ? c->d_red : c->d_red + 2;
  const size_t n = energies ? (kinetic ? 3 : 2) : 1;
  nccl_check(N.all_reduce(first, first, n, ncclFloat64, ncclSum, c->comm, c->stream),
             "ncclAllReduce");
  if (kinetic)
    nccl_check(N.all_reduce(c->d_red + 3, c->d_red + 3, 1, ncclFloat64, ncclMax, c->comm,
                            c->stream),
               "ncclAllReduce");
  launch_slab_red_out(c->P, c->d_red, energies, kinetic, c->stream);
  c->launches += 2;
}

void memset_field(cbx_ctx* c, int* field) { cudaMemsetAsync(field, 0, sizeof(int), c->stream); }

// end of a slab phase: (kick2 when kick >= 0) + finalize + cross-rank
// reduction -- on P2P the reduction is the tail of the finalize kernel
void slab_finish(cbx_ctx* c, int kick, int stepping, int energies) {
  if (c->p2p) {
    if (kick >= 0) {
      KP q = c->P;
      q.rev_wait = c->P.rev.on ? 4 : 0;  // the neighbours' force partials arrive first
      launch_kick2(q, kick, -2, 0, c->stream);
      c->launches += 1;
    } else if (c->P.rev.on) {
      launch_rev_wait(c->P, 4, c->stream);
      c->launches += 1;
    }
    launch_finalize(c->P, stepping, energies, c->stream, c->d_links);
    c->launches += 1;
    return;
  }
  if (kick >= 0) {
    launch_kick2(c->P, kick, stepping, energies, c->stream);
    c->launches += 1;
  } else {
    launch_finalize(c->P, stepping, energies, c->stream);
    c->launches += 1;
  }
  slab_reduce(c, energies != 0, stepping >= 0);
}

// one step of a slab rank: the single-box sequence with the five exchanges
void seq_slab_step(cbx_ctx* c) {
  c->mask_valid = false;
  ev_mark(c, 0);
  memset_field(c, &c->P.st->n_out);
  // merged kick (peer memory, fixed dt): the previous step's second half
  // kick runs in this step's k_kick_drift once the neighbours' force
  // partials are in; its sums + reduction in the density pass's idle block
  const bool merge = want_merge(c);
  c->graph_merge = merge;
  c->graph_defer = false;
  KP qf = c->P;
  qf.use_mask = 1;
  const int npp = force_partials(qf, c->mode);
  c->fin_npp = npp;
  // interior accumulators cleared here, the halo sites' by the POS unpack
  const bool zacc = c->mode != CBX_STENCIL_FULL;
  KP qk = c->P;
  qk.rev_wait = merge && c->P.rev.on ? 4 : 0;
  launch_kick_drift(qk, 1, c->stream, zacc ? 1 : 0, 0, npp);
  slab_exchange(c, 0);  // migrants
  launch_rehash(c->P, c->stream, merge ? 1 : 0, embed_grid(c->P), npp, kick_drift_grid(c->P));
  launch_ghost_fill(c->P, c->stream);
  c->launches += 3;
  memset_field(c, &c->P.st->n_remote);
  slab_exchange(c, 1);  // positions
  ev_mark(c, 1);
  launch_clash_images(c->P, c->stream, 1);
  c->clash_rho_zero = true;
  c->acc_rho_zero = c->acc_frc_zero = zacc;
  c->launches += 1;
  seq_density(c);
  slab_reverse(c, 2);  // density partials (reverse)
  ev_mark(c, 2);
  seq_embed(c, c->P.rev.on ? 2 : 0);
  slab_exchange(c, 3);  // dF
  ev_mark(c, 3);
  launch_remote_df(c->P, c->stream);
  c->launches += 1;
  c->merge_now = merge;
  seq_force(c);
  c->merge_now = false;
  slab_reverse(c, 4);  // force partials (reverse)
  ev_mark(c, 4);
  if (merge) {
    if (!g_capturing) c->k2_maybe = true;
  } else {
    slab_finish(c, 1, 1, 1);
  }
  ev_mark(c, 5);
}

// eval_forces of a slab rank (halos from the current positions)
void seq_slab_eval(cbx_ctx* c) {
  memset_field(c, &c->P.st->n_remote);
  slab_exchange(c, 1);
  ev_mark(c, 1);
  launch_clash_images(c->P, c->stream, 1);
  c->clash_rho_zero = true;
  c->launches += 1;
  seq_density(c);
  slab_reverse(c, 2);
  ev_mark(c, 2);
  seq_embed(c, c->P.rev.on ? 2 : 0);
  slab_exchange(c, 3);
  ev_mark(c, 3);
  launch_remote_df(c->P, c->stream);
  c->launches += 1;
  seq_force(c);
  slab_reverse(c, 4);
  ev_mark(c, 4);
  slab_finish(c, -1, -1, 1);
}

// one velocity-Verlet step, sim.cpp:248-273
// defer the StepState finalize of a step into the next step's first kernel
// (fixed dt only: with adaptive dt the next kick needs the reduced max speed)
bool want_defer(const cbx_ctx* c) {
  static const bool on = ab_flag("CBX_DEFER_FIN", 1) != 0;
  return on && !has_transport(c) && !c->hst.adaptive && !c->single;
}
// merge the second half kick of a step into the next step's kick/drift
// (one pass over v and f less per step): fixed dt, single box, the Newton-3
// mask-replay passes (the density pass's clash blocks run the pending sums)
bool want_merge(const cbx_ctx* c) {
  static const bool on = ab_flag("CBX_MERGE_KICK", 1) && ab_flag("CBX_DENSITY_SMEM", 1);
  // slab ranks on the peer-memory transport merge too: the next k_kick_drift
  // waits for the neighbours' force partials, and the deferred StepState sums
  // carry the cross-rank reduction (finalize_pending); not with NCCL (its
  // all-reduce is a stream operation, not a kernel tail)
  static const bool slab = ab_flag("CBX_SLAB_MERGE", 1) != 0;
  if (has_transport(c))
    return on && slab && c->p2p && !c->hst.adaptive && !c->single &&
           c->mode == CBX_STENCIL_NEWTON3 && c->P.pmask != nullptr;
  return on && want_defer(c) && c->mode == CBX_STENCIL_NEWTON3 && c->P.pmask != nullptr;
}

void seq_step(cbx_ctx* c) {
  if (has_transport(c)) {
    seq_slab_step(c);
    return;
  }
  c->mask_valid = false;
  // timing experiment of the A/B build only (CBX_SKIP bit mask, results
  // invalid): leave a phase out of the step to measure its marginal cost
  static const int skip = ab_flag("CBX_SKIP", 0);
  ev_mark(c, 0);
  const bool zacc = c->mode != CBX_STENCIL_FULL;  // single box: no remote halo sites
  // kick, drift, hash pass 1 and the slot images in one launch; hash pass 2
  // and the clash images in one single-block launch (no k_ghost_fill)
  KP qf = c->P;
  qf.use_mask = 1;  // the force pass below replays the density pass's mask
  const int npp = force_partials(qf, c->mode);
  const bool defer = want_defer(c);
  const bool merge = want_merge(c);
  c->graph_defer = defer;
  c->graph_merge = merge;
  c->fin_npp = npp;
  if (!(skip & 1)) launch_kick_drift(c->P, 1, c->stream, zacc ? 1 : 0, 1, npp);
  c->acc_rho_zero = c->acc_frc_zero = zacc;
  if (!(skip & 2))
    launch_rehash_images(c->P, c->stream, merge ? 1 : 0, embed_grid(c->P), npp,
                         kick_drift_grid(c->P));
  c->clash_rho_zero = true;
  c->launches += 2;
  ev_mark(c, 1);
  if (!(skip & 4)) seq_density(c);
  ev_mark(c, 2);
  if (!(skip & 8)) seq_embed(c);
  ev_mark(c, 3);
  c->merge_now = merge;
  if (!(skip & 16)) seq_force(c);
  c->merge_now = false;
  ev_mark(c, 4);
  if (merge) {
    if (!g_capturing) c->k2_maybe = true;
  } else {
    if (!(skip & 32)) launch_kick2(c->P, 1, (skip & 64) ? -2 : 1, 1, c->stream, defer ? 2 : 1, npp);
    if (defer && !g_capturing) c->fin_maybe = true;
    c->launches += 1;
  }
  ev_mark(c, 5);
}

void accumulate_timing(cbx_ctx* c, bool step) {
  if (!c->timing) return;
  cudaEventSynchronize(c->ev[step ? 5 : 4]);
  float ms = 0;
  if (step) {
    cudaEventElapsedTime(&ms, c->ev[0], c->ev[1]);
    c->t_ms[3] += ms;  // store: kick/drift/hash/rehash/ghosts
    cudaEventElapsedTime(&ms, c->ev[4], c->ev[5]);
    c->t_ms[4] += ms;  // kick2 + finalize
    cudaEventElapsedTime(&ms, c->ev[0], c->ev[5]);
    c->t_ms[5] += ms;
    c->t_ms[6] += 1;
  }
  cudaEventElapsedTime(&ms, c->ev[1], c->ev[2]);
  c->t_ms[0] += ms;
  cudaEventElapsedTime(&ms, c->ev[2], c->ev[3]);
  c->t_ms[1] += ms;
  cudaEventElapsedTime(&ms, c->ev[3], c->ev[4]);
  c->t_ms[2] += ms;
}

cudaGraphExec_t capture_step(cbx_ctx* c, bool with_events) {
  cudaGraph_t g;
  cudaGraphExec_t exec = nullptr;
  const bool t = c->timing;
  c->timing = with_events;
  const uint64_t l0 = c->launches;
  cuda_check(cudaStreamBeginCapture(c->stream, cudaStreamCaptureModeThreadLocal), "capture");
  g_capturing = true;
  seq_step(c);
  g_capturing = false;
  cuda_check(cudaStreamEndCapture(c->stream, &g), "end capture");
  cuda_check(cudaGraphInstantiate(&exec, g, 0), "graph instantiate");
  cudaGraphDestroy(g);
  c->graph_launches = c->launches - l0;
  c->launches = l0;
  c->timing = t;
  return exec;
}

void build_graph(cbx_ctx* c) {
  if (c->single) {
    if (!c->step_graph1) {
      c->step_graph1 = capture_step(c, false);
      c->graph1_launches = c->graph_launches;
    }
    return;
  }
  if (!c->step_graph) {
    c->step_graph = capture_step(c, false);
    c->g_defer = c->graph_defer;
    c->g_merge = c->graph_merge;
    c->g_launches = c->graph_launches;
  }
}

// single-box entry points that a slab rank can only run with its exchanges
void require_box_or_comm(cbx_ctx* c, const char* what) {
  if (c->G.slab && !has_transport(c))
    raise(CBX_LOGIC, std::string(what) +
                         ": slab rank without a communicator (cbx_slab_comm_init, or drive "
                         "cbx_slab_phase with the exchanges)");
}
void require_box(cbx_ctx* c, const char* what) {
  if (c->G.slab) raise(CBX_LOGIC, std::string(what) + ": not available on a slab rank");
}

void drop_graph(cbx_ctx* c) {
  if (c->step_graph) cudaGraphExecDestroy(c->step_graph);
  if (c->step_graph1) cudaGraphExecDestroy(c->step_graph1);
  c->step_graph1 = nullptr;
  if (c->timed_graph) cudaGraphExecDestroy(c->timed_graph);
  if (c->timed_lite) cudaGraphExecDestroy(c->timed_lite);
  c->step_graph = nullptr;
  c->timed_graph = nullptr;
  c->timed_lite = nullptr;
}

// ---- the store view ------------------------------------------------------
// ---- store transfer: raw host arrays move by DMA into / out of device
// staging buffers (reference id order, Vec3 AoS); the layout change to the
// parity-split SoA runs on the device (k_import_store / k_export_store)
struct StoreStage {
  double *pos, *vel, *frc, *rho, *df;
  unsigned long long* tag;
  unsigned char *valid, *ghost;
};

__global__ void k_import_store(KP P, StoreStage H, int has_vel, int has_frc, int has_rho,
                               int has_df, int has_tag, int has_valid, int has_ghost) {
  const long long id = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (id >= P.S) return;
  const Geo& G = P.G;
  const long long S = P.S, d = dev_of_ref(id, G.NC);
  int cx, cy, cz;
  cell_xyz(id >> 1, G, cx, cy, cz);
  bool live = !cell_is_ghost(cx, cy, cz, G);  // ghost cells: regenerated by fill_ghosts
  if (live && has_valid) live = H.valid[id] != 0;
  if (live && has_ghost) live = H.ghost[id] == 0;
  if (!live) {
    P.pdf[d] = make_double4(kVacant, kVacant, kVacant, 0.0);
    for (int a = 0; a < 3; ++a) {
      P.vel[a * S + d] = 0.0;
      P.frc[a * S + d] = 0.0;
    }
    P.rho[d] = 0.0;
    P.tag[d] = 0;
    return;
  }
  P.pdf[d] = make_double4(H.pos[3 * id], H.pos[3 * id + 1], H.pos[3 * id + 2],
                          has_df ? H.df[id] : 0.0);
  for (int a = 0; a < 3; ++a) {
    P.vel[a * S + d] = has_vel ? H.vel[3 * id + a] : 0.0;
    P.frc[a * S + d] = has_frc ? H.frc[3 * id + a] : 0.0;
  }
  P.rho[d] = has_rho ? H.rho[id] : 0.0;
  P.tag[d] = has_tag ? H.tag[id] : 0ull;
}

// download semantics (LatticeStore view): ghosts report their source's
// velocity, rho and tag and zero force
__global__ void k_export_store(KP P, StoreStage H) {
  const long long id = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (id >= P.S) return;
  const long long S = P.S, d = dev_of_ref(id, P.G.NC);
  const long long t = P.tgt[d];
  const double4 p = P.pdf[d];
  const bool valid = p.x < kVacantTest, ghost = t != d;
  H.valid[id] = valid;
  H.ghost[id] = valid && ghost;
  H.pos[3 * id] = p.x;
  H.pos[3 * id + 1] = p.y;
  H.pos[3 * id + 2] = p.z;
  H.df[id] = p.w;
  for (int a = 0; a < 3; ++a) {
    H.vel[3 * id + a] = P.vel[a * S + t];
    H.frc[3 * id + a] = ghost ? 0.0 : P.frc[a * S + d];
  }
  H.rho[id] = P.rho[t];
  H.tag[id] = P.tag[t];
}

StoreStage& stage(cbx_ctx* c) {
  if (!c->stage_pos) {
    const long long S = c->S;
    c->mem_cat = CBX_MEM_STAGING;
    c->stage_pos = c->alloc<double>(3 * S);
    c->stage_vel = c->alloc<double>(3 * S);
    c->stage_frc = c->alloc<double>(3 * S);
    c->stage_rho = c->alloc<double>(S);
    c->stage_df = c->alloc<double>(S);
    c->stage_tag = c->alloc<unsigned long long>(S);
    c->stage_valid = c->alloc<unsigned char>(S);
    c->stage_ghost = c->alloc<unsigned char>(S);
  }
  static thread_local StoreStage H;
  H = StoreStage{c->stage_pos, c->stage_vel, c->stage_frc, c->stage_rho, c->stage_df,
                 c->stage_tag, c->stage_valid, c->stage_ghost};
  return H;
}

void do_upload(cbx_ctx* c, const cbx_store* s) {
  const Geo& G = c->G;
  const long long S = c->S;
  if (s->n_slots != S)
    raise(CBX_INVALID_ARGUMENT, "upload_store: n_slots " + std::to_string(s->n_slots) +
                                    " does not match slot_count " + std::to_string(S));
  if (!s->pos) raise(CBX_INVALID_ARGUMENT, "upload_store: pos is required");
  cudaStream_t st = c->stream;
  const StoreStage& H = stage(c);
  auto h2d = [&](void* dst, const void* src, size_t bytes) {
    if (src) cuda_check(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyHostToDevice, st), "upload");
  };
  h2d(H.pos, s->pos, 3 * S * sizeof(double));
  h2d(H.vel, s->vel, 3 * S * sizeof(double));
  h2d(H.frc, s->force, 3 * S * sizeof(double));
  h2d(H.rho, s->rho, S * sizeof(double));
  h2d(H.df, s->df, S * sizeof(double));
  h2d(H.tag, s->tag, S * sizeof(unsigned long long));
  h2d(H.valid, s->valid, S);
  h2d(H.ghost, s->ghost, S);
  k_import_store<<<(unsigned)((S + 255) / 256), 256, 0, st>>>(
      c->P, H, s->vel != nullptr, s->force != nullptr, s->rho != nullptr, s->df != nullptr,
      s->tag != nullptr, s->valid != nullptr, s->ghost != nullptr);
  c->launches += 1;
  // new positions: no regional displacement bound is valid until the next
  // k_kick_drift + pass 2 publish one
  if (c->P.ustamp) cudaMemsetAsync(c->P.ustamp, 0, sizeof(unsigned long long), st);
  auto site_live = [&](long long id) {
    return (s->valid ? s->valid[id] != 0 : true) && !(s->ghost && s->ghost[id]);
  };
  // interior clash records, in (key, index) order
  std::vector<long long> key;
  std::vector<double> cp, cv, cf, cr, cd;
  std::vector<unsigned long long> ct;
  for (long i = 0; i < s->n_clash; ++i) {
    const long long k = s->clash_key[i];
    if (k < 0 || k >= S) raise(CBX_INVALID_ARGUMENT, "upload_store: clash key out of range");
    int cx, cy, cz;
    cell_xyz(k >> 1, G, cx, cy, cz);
    if (cell_is_ghost(cx, cy, cz, G) || (s->clash_ghost && s->clash_ghost[i])) continue;
    if (!key.empty() && k < key.back())
      raise(CBX_INVALID_ARGUMENT, "upload_store: clash records must be in key order");
    if (!site_live(k))
      raise(CBX_INVALID_ARGUMENT,
            "unsupported store state: a clash bucket over a vacant lattice site");
    key.push_back(k);
    for (int a = 0; a < 3; ++a) {
      cp.push_back(s->clash_pos[3 * i + a]);
      cv.push_back(s->clash_vel ? s->clash_vel[3 * i + a] : 0.0);
      cf.push_back(s->clash_force ? s->clash_force[3 * i + a] : 0.0);
    }
    cr.push_back(s->clash_rho ? s->clash_rho[i] : 0.0);
    cd.push_back(s->clash_df ? s->clash_df[i] : 0.0);
    ct.push_back(s->clash_tag ? s->clash_tag[i] : 0);
  }
  const int nc = (int)key.size();
  if (nc > c->P.cap_clash) raise(CBX_RUNTIME, "clash list capacity exceeded");
  // clash SoA
  std::vector<double> tmp(nc);
  std::vector<unsigned char> zeros(nc, 0);
  std::vector<int> src(nc);
  for (int i = 0; i < nc; ++i) src[i] = i;
  const Clash& A = c->P.cl;
  if (nc) {
    cudaMemcpyAsync(A.key, key.data(), nc * sizeof(long long), cudaMemcpyHostToDevice, st);
    cudaMemcpyAsync(A.gf, zeros.data(), nc, cudaMemcpyHostToDevice, st);
    cudaMemcpyAsync(A.src, src.data(), nc * sizeof(int), cudaMemcpyHostToDevice, st);
    double* dst3[3][3] = {{A.px, A.py, A.pz}, {A.vx, A.vy, A.vz}, {A.fx, A.fy, A.fz}};
    const std::vector<double>* src3[3] = {&cp, &cv, &cf};
    for (int f = 0; f < 3; ++f)
      for (int a = 0; a < 3; ++a) {
        std::vector<double> col(nc);
        for (int i = 0; i < nc; ++i) col[i] = (*src3[f])[3 * i + a];
        cudaMemcpyAsync(dst3[f][a], col.data(), nc * sizeof(double), cudaMemcpyHostToDevice, st);
        cudaStreamSynchronize(st);
      }
    cudaMemcpyAsync(A.rho, cr.data(), nc * sizeof(double), cudaMemcpyHostToDevice, st);
    cudaMemcpyAsync(A.df, cd.data(), nc * sizeof(double), cudaMemcpyHostToDevice, st);
    cudaMemcpyAsync(A.tag, ct.data(), nc * sizeof(unsigned long long), cudaMemcpyHostToDevice, st);
    cudaMemsetAsync(A.e_emb, 0, nc * sizeof(double), st);
    cudaMemsetAsync(A.e_pair, 0, nc * sizeof(double), st);
    cudaMemsetAsync(A.v2, 0, nc * sizeof(double), st);
  }
  // reset the head map and the list counters
  cudaMemsetAsync(c->P.head, 0xff, S * sizeof(int), st);
  sync_status(c);
  c->hst.n_clash = nc;
  c->hst.n_mov = 0;
  c->hst.err = 0;
  c->hst.n_ovl = 0;
  c->hst.halt = 0;
  write_status(c);
  seq_fill_ghosts(c);
  launch_uf_refresh(c->P, c->stream);
  sync_status(c);
  raise_device_error(c, false);
}

template <class T>
std::vector<T> fetch(cbx_ctx* c, const T* d, size_t n) {
  std::vector<T> h(n);
  if (n)
    cuda_check(cudaMemcpyAsync(h.data(), d, n * sizeof(T), cudaMemcpyDeviceToHost, c->stream),
               "download");
  return h;
}

void do_download(cbx_ctx* c, cbx_store* s) {
  const long long S = c->S;
  if (s->n_slots != S) raise(CBX_INVALID_ARGUMENT, "download_store: n_slots mismatch");
  cudaStream_t st = c->stream;
  const StoreStage& H = stage(c);
  k_export_store<<<(unsigned)((S + 255) / 256), 256, 0, st>>>(c->P, H);
  c->launches += 1;
  auto d2h = [&](void* dst, const void* src, size_t bytes) {
    if (dst) cuda_check(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDeviceToHost, st), "download");
  };
  d2h(s->pos, H.pos, 3 * S * sizeof(double));
  d2h(s->vel, H.vel, 3 * S * sizeof(double));
  d2h(s->force, H.frc, 3 * S * sizeof(double));
  d2h(s->rho, H.rho, S * sizeof(double));
  d2h(s->df, H.df, S * sizeof(double));
  d2h(s->tag, H.tag, S * sizeof(unsigned long long));
  d2h(s->valid, H.valid, S);
  d2h(s->ghost, H.ghost, S);
  sync_status(c);
  const int nc = c->hst.n_clash;
  if (s->clash_key == nullptr) {
    s->n_clash = nc;
    return;
  }
  if (s->n_clash < nc) raise(CBX_INVALID_ARGUMENT, "download_store: clash capacity too small");
  s->n_clash = nc;
  const Clash& A = c->P.cl;
  auto key = fetch(c, A.key, nc);
  auto gf = fetch(c, A.gf, nc);
  auto src = fetch(c, A.src, nc);
  auto px = fetch(c, A.px, nc), py = fetch(c, A.py, nc), pz = fetch(c, A.pz, nc);
  auto vx = fetch(c, A.vx, nc), vy = fetch(c, A.vy, nc), vz = fetch(c, A.vz, nc);
  auto fx = fetch(c, A.fx, nc), fy = fetch(c, A.fy, nc), fz = fetch(c, A.fz, nc);
  auto rr = fetch(c, A.rho, nc), dd = fetch(c, A.df, nc);
  auto tt = fetch(c, A.tag, nc);
  cuda_check(cudaStreamSynchronize(c->stream), "download");
  int idx = 0;
  for (int i = 0; i < nc; ++i) {
    idx = (i > 0 && key[i - 1] == key[i]) ? idx + 1 : 0;
    s->clash_key[i] = key[i];
    if (s->clash_idx) s->clash_idx[i] = idx;
    if (s->clash_ghost) s->clash_ghost[i] = gf[i];
    if (s->clash_pos) {
      s->clash_pos[3 * i] = px[i];
      s->clash_pos[3 * i + 1] = py[i];
      s->clash_pos[3 * i + 2] = pz[i];
    }
    if (s->clash_vel) {
      s->clash_vel[3 * i] = vx[i];
      s->clash_vel[3 * i + 1] = vy[i];
      s->clash_vel[3 * i + 2] = vz[i];
    }
    if (s->clash_force) {
      s->clash_force[3 * i] = gf[i] ? 0.0 : fx[i];
      s->clash_force[3 * i + 1] = gf[i] ? 0.0 : fy[i];
      s->clash_force[3 * i + 2] = gf[i] ? 0.0 : fz[i];
    }
    if (s->clash_rho) s->clash_rho[i] = rr[gf[i] ? src[i] : i];
    if (s->clash_df) s->clash_df[i] = dd[i];
    if (s->clash_tag) s->clash_tag[i] = tt[i];
  }
}

// the parameter block's device copy (guard paths take it by pointer)
void sync_kp(cbx_ctx* c) {
  cuda_check(cudaMemcpy(c->P.dself, &c->P, sizeof(KP), cudaMemcpyHostToDevice), "kp upload");
}

// Shared-memory window of the force table (split-3 layout, stencil_fast.cuh).
// shells: the distinct lattice distances of the stencil sites within the
// cutoff, ascending.  The window must hold every record a pair near a shell
// can touch: r in [R - margin, R + margin], and everything from the last
// shell up to the cutoff (the skin shells enter there).  If dropping the
// records below the first shell's margin and a stretch inside the widest gap
// between two shells brings the window down to kLeanTabRecordsGap records,
// the gapped window is used (pairs inside the gap or below the window -- a
// cascade core -- fetch every chunk by texture, as pairs below the window
// always did); otherwise the contiguous top kLeanTabRecords records.
void force_window_setup(cbx_ctx* c, const std::vector<double>& shells) {
  KP& P = c->P;
  const int n1 = P.ff.nseg + 1;  // records 0..nseg
  const int lo0 = n1 - kLeanTabRecords;
  P.fw_lo = ((lo0 > 0 ? lo0 : 0) + 1) & ~1;
  P.fw_gap_lo = 0x7fffffff;
  P.fw_gap_n = 0;
  P.fw_cap = kLeanTabRecords;
  if (shells.empty() || !ab_flag("CBX_FORCE_GAP", 1)) return;
  constexpr double margin = 0.30;  // A: ~3.5 sigma of a bond length at 600 K
  const double x0 = c->pot.zr.x0, h = c->pot.zr.h;
  auto seg_of = [&](double r) { return (int)std::floor((r - x0) / h); };
  int lo = std::max(0, seg_of(shells.front() - margin)) & ~1;
  if (lo < P.fw_lo) lo = P.fw_lo;  // never below the contiguous window's start
  const int need = (n1 - lo) - kLeanTabRecordsGap;
  if (need <= 0) {  // fits without a gap
    P.fw_lo = lo;
    P.fw_cap = kLeanTabRecordsGap;
    return;
  }
  // the widest stretch between two shells' margins
  int best_lo = 0, best_n = 0;
  for (size_t i = 0; i + 1 < shells.size(); ++i) {
    const int a = seg_of(shells[i] + margin) + 1, b = seg_of(shells[i + 1] - margin);
    if (b - a > best_n) {
      best_n = b - a;
      best_lo = a;
    }
  }
  const int gn = (need + 1) & ~1;
  if (best_n < gn + 2) return;  // no stretch wide enough: contiguous window
  const int glo = (best_lo + (best_n - gn) / 2 + 1) & ~1;  // centred, even
  if (glo <= lo || glo + gn >= n1) return;
  P.fw_lo = lo;
  P.fw_gap_lo = glo;
  P.fw_gap_n = gn;
  P.fw_cap = kLeanTabRecordsGap;
}

// fast-path tables and the fp32 filter band (stencil_fast.cuh)
void setup_fast(cbx_ctx* c) {
  KP& P = c->P;
  const Spline& zr = c->pot.zr;
  const Spline& de = c->pot.dens;
  c->fast_ok = zr.x0 == de.x0 && zr.h == de.h && zr.nseg() == de.nseg();
  const int n = (int)de.nseg();
  auto norm = [](const double* g, double h, double out[4]) {  // t = s h
    out[0] = g[0] * h * h * h;
    out[1] = g[1] * h * h;
    out[2] = g[2] * h;
    out[3] = g[3];
  };
  auto pad = [](const double in[4], double out[4]) {  // p(s + 1)
    out[0] = in[0];
    out[1] = 3.0 * in[0] + in[1];
    out[2] = 3.0 * in[0] + 2.0 * in[1] + in[2];
    out[3] = in[0] + in[1] + in[2] + in[3];
  };
  std::vector<double> fd(4 * (n + 1)), ff(8 * (n + 1));
  for (int i = 0; i < n; ++i) {
    norm(&de.seg[7 * i], de.h, &fd[4 * i]);
    norm(&de.seg[7 * i], de.h, &ff[8 * i + 4]);
    if (c->fast_ok) norm(&zr.seg[7 * i], zr.h, &ff[8 * i]);
  }
  pad(&fd[4 * (n - 1)], &fd[4 * n]);
  pad(&ff[8 * (n - 1)], &ff[8 * n]);
  pad(&ff[8 * (n - 1) + 4], &ff[8 * n + 4]);
  double* dfd = c->alloc<double>(fd.size());
  double* dff = c->alloc<double>(ff.size());
  cuda_check(cudaMemcpy(dfd, fd.data(), fd.size() * 8, cudaMemcpyHostToDevice), "fast table");
  cuda_check(cudaMemcpy(dff, ff.data(), ff.size() * 8, cudaMemcpyHostToDevice), "fast table");
  P.fd.rec = dfd;
  {  // fp64 [A B] pairs (shared-memory window) and the [C D] pairs bound to
     // a texture (int4 texels) for the default density pass
    std::vector<double> ab(2 * (n + 1)), cd(2 * (n + 1));
    for (int i = 0; i <= n; ++i) {
      ab[2 * i] = fd[4 * i];
      ab[2 * i + 1] = fd[4 * i + 1];
      cd[2 * i] = fd[4 * i + 2];
      cd[2 * i + 1] = fd[4 * i + 3];
    }
    double* dab = c->alloc<double>(ab.size());
    cuda_check(cudaMemcpy(dab, ab.data(), ab.size() * 8, cudaMemcpyHostToDevice), "fast table");
    P.fdab = dab;
    double* dcd = c->alloc<double>(cd.size());
    cuda_check(cudaMemcpy(dcd, cd.data(), cd.size() * 8, cudaMemcpyHostToDevice), "fast table");
    cudaResourceDesc rd{};
    rd.resType = cudaResourceTypeLinear;
    rd.res.linear.devPtr = dcd;
    rd.res.linear.desc = cudaCreateChannelDesc<int4>();
    rd.res.linear.sizeInBytes = cd.size() * sizeof(double);
    cudaTextureDesc td{};
    td.readMode = cudaReadModeElementType;
    cudaTextureObject_t tex = 0;
    cuda_check(cudaCreateTextureObject(&tex, &rd, &td, nullptr), "density record texture");
    P.tex_fd4 = (unsigned long long)tex;
    c->textures.push_back(tex);
  }
  P.fd.ih = 1.0 / de.h;
  P.fd.c0 = -de.x0 / de.h;
  P.fd.nseg = n;
  P.ff = P.fd;
  P.ff.rec = dff;
  // force-table chunks for the shared-memory window (fp64: a rigorous bound
  // on fp32 cubic terms -- 3 |dA| ih / r per pair with the table's largest
  // |F'| -- exceeds the 1e-10 force tolerance over the window for the
  // BASELINE table, so the force records stay fp64) and the texture view of
  // the full 64-byte records
  {
    std::vector<double> fz(4 * (n + 1)), fzc(2 * (n + 1)), fqc(n + 3, 0.0);
    for (int i = 0; i <= n; ++i) {
      const double* r = &ff[8 * i];
      for (int k = 0; k < 4; ++k) fz[4 * i + k] = r[k];
      fzc[2 * i] = r[2];
      fzc[2 * i + 1] = r[3];
      fqc[i] = r[6];
    }
    auto up = [&](const std::vector<double>& v) {
      double* d = c->alloc<double>(v.size());
      cuda_check(cudaMemcpy(d, v.data(), v.size() * 8, cudaMemcpyHostToDevice), "fast table");
      return d;
    };
    P.ffz = up(fz);
    P.ffzc = up(fzc);
    P.ffqc = up(fqc);
    cudaResourceDesc rd{};
    rd.resType = cudaResourceTypeLinear;
    rd.res.linear.devPtr = const_cast<double*>(P.ff.rec);
    rd.res.linear.desc = cudaCreateChannelDesc<int4>();
    rd.res.linear.sizeInBytes = ff.size() * sizeof(double);
    cudaTextureDesc td{};
    td.readMode = cudaReadModeElementType;
    cudaTextureObject_t tex = 0;
    cuda_check(cudaCreateTextureObject(&tex, &rd, &td, nullptr), "force table texture");
    P.tex_ff = (unsigned long long)tex;
    c->textures.push_back(tex);
    // the two chunks the force pass fetches through TEX, packed: [zA zB qA qB]
    // is one 32-byte sector per segment (in the 64-byte records they sit in
    // two sectors whose other halves -- staged in shared memory -- would
    // occupy L1 beside the partner gathers; thermal displacements spread a
    // warp's pairs over ~2000 segments)
    std::vector<double> fab(4 * (n + 1));
    for (int i = 0; i <= n; ++i) {
      const double* r = &ff[8 * i];
      fab[4 * i] = r[0];
      fab[4 * i + 1] = r[1];
      fab[4 * i + 2] = r[4];
      fab[4 * i + 3] = r[5];
    }
    P.ffab = up(fab);
    rd.res.linear.devPtr = const_cast<double*>(P.ffab);
    rd.res.linear.sizeInBytes = fab.size() * sizeof(double);
    cudaTextureObject_t tex2 = 0;
    cuda_check(cudaCreateTextureObject(&tex2, &rd, &td, nullptr), "force [A B] texture");
    P.tex_fab = (unsigned long long)tex2;
    c->textures.push_back(tex2);
  }
  // compressed density records for the density pass: [D C] in fp64, the
  // cubic and quadratic coefficients A, B (~1e-9 and ~1e-6 of rho at the
  // BASELINE spacing) in fp32.  Local guard over the staged window (the only
  // records the compressed path reads; pairs below it use the fp64 records):
  // for every segment, the fp32 rounding of A and B moves rho(s) by at most
  // kRhoRel of the smallest |rho| the segment can take (|D| - |C| - |B| - |A|,
  // required > 0), so each pair's rho is within kRhoRel relative; rho terms
  // of one sign add up with the same relative bound on every rho-bar (1e-12
  // against the 1e-10 tolerance).  A table failing it anywhere in the window
  // (steep or sign-changing rho) keeps the 32-byte fp64 records.
  P.fdc = nullptr;
  c->fp32_density = false;
  {
    constexpr double kRhoRel = 1e-12;
    const int lo = dens_window_lo_cmp(n);
    bool ok = true;
    int sign = 0;
    for (int i = lo; i <= n && ok; ++i) {
      const double* r = &fd[4 * i];
      const double ea = std::fabs(r[0] - (double)(float)r[0]) + std::fabs(r[1] - (double)(float)r[1]);
      const double m = std::fabs(r[3]) - std::fabs(r[2]) - std::fabs(r[1]) - std::fabs(r[0]);
      const int sg = r[3] > 0.0 ? 1 : -1;
      if (!sign) sign = sg;
      ok = m > 0.0 && sg == sign && ea <= kRhoRel * m;
    }
    if (ok && !ab_flag("CBX_NO_FP32_DENSITY", 0)) {
      std::vector<double> dc(3 * (n + 1) + 2);  // + 16 bytes: the bulk copy rounds up
      for (int i = 0; i <= n; ++i) {
        const double* r = &fd[4 * i];
        dc[2 * i] = r[3];
        dc[2 * i + 1] = r[2];
        const float ab[2] = {(float)r[0], (float)r[1]};
        std::memcpy(&dc[2 * (n + 1) + i], ab, 8);
      }
      double* ddc = c->alloc<double>(dc.size());
      cuda_check(cudaMemcpy(ddc, dc.data(), dc.size() * 8, cudaMemcpyHostToDevice), "fast table");
      P.fdc = ddc;
      c->fp32_density = true;
      cudaResourceDesc rd{};
      rd.resType = cudaResourceTypeLinear;
      rd.res.linear.devPtr = ddc;
      rd.res.linear.desc = cudaCreateChannelDesc<int4>();
      rd.res.linear.sizeInBytes = 16 * (size_t)(n + 1);
      cudaTextureDesc td{};
      td.readMode = cudaReadModeElementType;
      cudaTextureObject_t tex = 0;
      cuda_check(cudaCreateTextureObject(&tex, &rd, &td, nullptr), "density table texture");
      P.tex_fd = (unsigned long long)tex;
      c->textures.push_back(tex);
    }
  }
  // embedding F(rho), same normalisation (its own grid)
  {
    const Spline& em = c->pot.embed;
    const int ne = (int)em.nseg();
    std::vector<double> fe(4 * (ne + 1));
    for (int i = 0; i < ne; ++i) norm(&em.seg[7 * i], em.h, &fe[4 * i]);
    pad(&fe[4 * (ne - 1)], &fe[4 * ne]);
    double* dfe = c->alloc<double>(fe.size());
    cuda_check(cudaMemcpy(dfe, fe.data(), fe.size() * 8, cudaMemcpyHostToDevice), "fast table");
    P.fe.rec = dfe;
    P.fe.ih = 1.0 / em.h;
    P.fe.c0 = -em.x0 / em.h;
    P.fe.nseg = ne;
  }
  // fp32 filter band: |r2_f32 - r2_exact| <= err for coordinates below
  // maxc (two roundings to fp32, exact fp32 difference, three fp32 ops)
  const double maxc = (std::max(std::max(c->G.tx, c->G.ty), c->G.gtz) + 4) * c->G.a0;
  const double ulp = std::ldexp(1.0, std::ilogb(maxc) - 23);
  const double cut2 = P.cut2, dmax = std::sqrt(cut2) + 1.0;
  const double err = 2.0 * dmax * std::sqrt(3.0) * ulp + 3.0 * ulp * ulp +
                     4.0 * std::ldexp(1.0, -23) * (cut2 + 1.0);
  const double band = 8.0 * err + 1e-9;
  P.band_hi = std::nextafter((float)(cut2 + band), 1e30f);
  P.band_lo = std::nextafter((float)(cut2 - band), -1e30f);
  const double x0 = std::max(zr.x0, de.x0);
  P.guard_r2 = x0 * x0 * 1.000001;
  // fp64 r^2 by FMA vs the reference's r^2: a few ulp of r^2 apart
  P.cut2_lo = cut2 * (1.0 - 1e-12);
  P.cut2_hi = cut2 * (1.0 + 1e-12);
  c->band = band;
}

void check_cutoff(cbx_ctx* c) {
  if (!c->cutoff_ok)
    raise(CBX_INVALID_ARGUMENT, "offset index cutoff is smaller than the potential cutoff");
}

}  // namespace

// ===========================================================================
extern "C" {

CBX_API int cbx_abi_version(void) { return CBX_ABI_VERSION; }
CBX_API const char* cbx_build_info(void) { return kBuild; }
CBX_API const char* cbx_last_error(const cbx_ctx* c) {
  return c ? c->err.c_str() : thread_error();
}

CBX_API cbx_status cbx_write_synthetic_table(const char* path, long nrho, long nr) {
  return guarded(nullptr, [&] { write_synthetic_table(path ? path : "", nrho, nr); });
}

CBX_API cbx_status cbx_potential_load(const char* path, cbx_potential** out) {
  return guarded(nullptr, [&] {
    auto* p = new Potential(parse_potential(path));
    auto* o = new cbx_potential{};
    o->atomic_number = p->atomic_number;
    o->mass = p->mass;
    o->lattice_const = p->lattice_const;
    o->cutoff = p->cutoff;
    auto fill = [](cbx_spline& d, const Spline& s) {
      d.x0 = s.x0;
      d.h = s.h;
      d.nseg = s.nseg();
      d.seg = s.seg.data();
    };
    fill(o->embed, p->embed);
    fill(o->zr, p->zr);
    fill(o->dens, p->dens);
    // the owning Potential rides behind the public struct
    struct Owned {
      cbx_potential pub;
      Potential* own;
    };
    auto* w = new Owned{*o, p};
    delete o;
    *out = &w->pub;
  });
}
CBX_API void cbx_potential_free(cbx_potential* pot) {
  if (!pot) return;
  struct Owned {
    cbx_potential pub;
    Potential* own;
  };
  auto* w = reinterpret_cast<Owned*>(pot);
  delete w->own;
  delete w;
}

CBX_API cbx_status cbx_offsets_build(const cbx_box* box, double cutoff, cbx_offsets** out) {
  return guarded(nullptr, [&] {
    Offsets o = build_offsets(*box, cutoff);
    struct Owned {
      cbx_offsets pub;
      std::vector<int64_t> l[4];
    };
    auto* w = new Owned{};
    for (int par = 0; par < 2; ++par) {
      for (const Offset& f : o.full[par]) w->l[par].push_back(f.flat);
      for (const Offset& f : o.half[par]) w->l[2 + par].push_back(f.flat);
    }
    w->pub.cutoff = o.cutoff;
    w->pub.z_reach = o.z_reach;
    w->pub.even_full = w->l[0].data();
    w->pub.odd_full = w->l[1].data();
    w->pub.even_half = w->l[2].data();
    w->pub.odd_half = w->l[3].data();
    w->pub.n_even_full = (long)w->l[0].size();
    w->pub.n_odd_full = (long)w->l[1].size();
    w->pub.n_even_half = (long)w->l[2].size();
    w->pub.n_odd_half = (long)w->l[3].size();
    *out = &w->pub;
  });
}
CBX_API void cbx_offsets_free(cbx_offsets* idx) {
  struct Owned {
    cbx_offsets pub;
    std::vector<int64_t> l[4];
  };
  delete reinterpret_cast<Owned*>(idx);
}

CBX_API cbx_status cbx_make_box(long bx, long by, long bz, double a0_cfg, long gw_cfg,
                                double max_disp, const cbx_potential* pot, cbx_box* out,
                                double* index_cutoff) {
  return guarded(nullptr, [&] {
    if (bx <= 0 || by <= 0 || bz <= 0)
      raise(CBX_INVALID_ARGUMENT, "box: dimensions must be positive");
    const double a0 = a0_cfg > 0.0 ? a0_cfg : pot->lattice_const;
    if (!(a0 > 0.0))
      raise(CBX_INVALID_ARGUMENT,
            "box.a0: the potential file carries no usable lattice constant");
    if (max_disp >= a0 / 2.0)
      raise(CBX_INVALID_ARGUMENT, "max_disp: must stay below half the lattice constant");
    const double ic = pot->cutoff + 0.3 * a0;
    const long gw = gw_cfg > 0 ? gw_cfg : (long)std::ceil(ic / a0);
    *out = cbx_box{bx, by, bz, a0, gw};
    if (index_cutoff) *index_cutoff = pot->cutoff + 0.3 * a0;
  });
}

CBX_API double cbx_pka_speed(double e, double m) {
  return std::sqrt(2.0 * e / m) * speed_factor();
}
CBX_API double cbx_adaptive_dt(double vmax, double dt_max, double max_disp) {
  double dt = dt_max;
  if (vmax > 0.0) dt = std::min(dt, max_disp / vmax);
  return std::max(dt, 1e-7);
}

struct SlabSpec {
  int rank = 0, nranks = 1, zoff = 0, gbz = 0;
};

static cbx_status create_impl(const cbx_box* box, const cbx_potential* pot,
                              const cbx_offsets* idx, int device, const SlabSpec* slab,
                              cbx_ctx** out) {
  auto c = std::make_unique<cbx_ctx>();
  const cbx_status rc = guarded(nullptr, [&] {
    if (box->box_x <= 0 || box->box_y <= 0 || box->box_z <= 0 || !(box->a0 > 0.0) ||
        box->ghost_width < 0)
      raise(CBX_INVALID_ARGUMENT, "LatticeStore: box dimensions must be positive");
    int ndev = 0;
    cuda_check(cudaGetDeviceCount(&ndev), "cudaGetDeviceCount");
    if (device < 0 || device >= ndev) raise(CBX_CUDA, "no such CUDA device");
    c->device = device;
    cuda_check(cudaSetDevice(device), "cudaSetDevice");
    cuda_check(cudaStreamCreateWithFlags(&c->stream, cudaStreamNonBlocking), "stream");
    for (auto& e : c->ev) cudaEventCreate(&e);
    c->box = *box;
    c->G = make_geo(*box);
    if (slab) {
      if (box->box_z < box->ghost_width)
        raise(CBX_INVALID_ARGUMENT, "z slab thinner than the ghost width");
      c->G.zoff = slab->zoff;
      c->G.gbz = slab->gbz;
      c->G.gtz = slab->gbz + 2 * c->G.g;
      c->G.glz = slab->gbz * box->a0;
      c->G.slab = 1;
      c->G.kmz = 0;  // z images come from the neighbouring ranks
      c->rank = slab->rank;
      c->nranks = slab->nranks;
      c->gbox = *box;
      c->gbox.box_z = slab->gbz;
    }
    const Geo& G = c->G;
    c->S = 2 * G.NC;
    if (c->S >= (1ll << 31)) raise(CBX_INVALID_ARGUMENT, "box too large for one device (2^31 sites)");
    // host copy of the potential tables
    c->pot.atomic_number = pot->atomic_number;
    c->pot.mass = pot->mass;
    c->pot.lattice_const = pot->lattice_const;
    c->pot.cutoff = pot->cutoff;
    auto cp = [](Spline& d, const cbx_spline& s) {
      d.x0 = s.x0;
      d.h = s.h;
      d.seg.assign(s.seg, s.seg + 7 * s.nseg);
    };
    cp(c->pot.embed, pot->embed);
    cp(c->pot.zr, pot->zr);
    cp(c->pot.dens, pot->dens);
    // offsets: rebuilt with the reference algorithm, the caller's must agree
    const double ic = idx ? idx->cutoff : pot->cutoff + 0.3 * box->a0;
    c->offs = build_offsets(*box, ic);
    if (idx) {
      auto same = [](const std::vector<Offset>& a, const int64_t* b, long n) {
        if ((long)a.size() != n) return false;
        for (long i = 0; i < n; ++i)
          if (a[i].flat != b[i]) return false;
        return true;
      };
      if (!same(c->offs.full[0], idx->even_full, idx->n_even_full) ||
          !same(c->offs.full[1], idx->odd_full, idx->n_odd_full) ||
          !same(c->offs.half[0], idx->even_half, idx->n_even_half) ||
          !same(c->offs.half[1], idx->odd_half, idx->n_odd_half))
        raise(CBX_INVALID_ARGUMENT, "offset index does not match build_offsets(box, cutoff)");
    }
    c->cutoff_ok = !(c->offs.cutoff < pot->cutoff);
    for (int par = 0; par < 2; ++par)
      if ((int)c->offs.full[par].size() > kMaxOffsets)
        raise(CBX_INVALID_ARGUMENT, "offset index too large for the device tables");
    // device offset deltas, ordered by lattice distance: sites within the
    // potential cutoff first ("inner"), index-skin sites after (stencil_fast.cuh)
    std::vector<int> hd[2], fd[2];
    std::vector<long long> ff[2];
    int hin[2] = {0, 0}, fin[2] = {0, 0};
    SkinGroups skh[2], skf[2];
    int sreach[2] = {0, 0};
    for (int par = 0; par < 2; ++par) {
      auto delta = [&](const Offset& o) {
        const int q = par ^ o.cross;
        return (int)((long long)(q - par) * G.NC + (long long)o.dz * G.txy +
                     (long long)o.dy * G.tx + o.dx);
      };
      auto dist2 = [&](const Offset& o) {
        const double h = o.cross ? (par ? -0.5 : 0.5) : 0.0;
        const double x = o.dx + h, y = o.dy + h, z = o.dz + h;
        return (x * x + y * y + z * z) * box->a0 * box->a0;
      };
      auto order = [&](std::vector<Offset> v, int& nin, SkinGroups& sg, int& reach) {
        std::stable_sort(v.begin(), v.end(),
                         [&](const Offset& a, const Offset& b) { return dist2(a) < dist2(b); });
        nin = 0;
        for (const Offset& o : v)
          if (dist2(o) <= pot->cutoff * pot->cutoff) ++nin;
        // skin shells (equal lattice distance) beyond nin, at most 4 groups:
        // the last one takes every remaining shell at its smallest distance
        sg = SkinGroups{};
        for (int k = nin; k < (int)v.size(); ++k)
          reach = std::max(reach, std::max(std::abs(v[k].dx), std::max(std::abs(v[k].dy),
                                                                      std::abs(v[k].dz))));
        for (int k = nin; k < (int)v.size(); ++k) {
          const bool fresh = k == nin || dist2(v[k]) != dist2(v[k - 1]);
          if (fresh && sg.n < 4) sg.len[sg.n++] = std::sqrt(dist2(v[k]));
          sg.end[sg.n - 1] = k + 1;
        }
        return v;
      };
      for (const Offset& o : order(c->offs.half[par], hin[par], skh[par], sreach[0])) {
        hd[par].push_back(delta(o));
      }
      for (const Offset& o : order(c->offs.full[par], fin[par], skf[par], sreach[1])) {
        fd[par].push_back(delta(o));
        ff[par].push_back(o.flat);
      }
    }
    const int* hp[2] = {hd[0].data(), hd[1].data()};
    const int* fp[2] = {fd[0].data(), fd[1].data()};
    const long long* fl[2] = {ff[0].data(), ff[1].data()};
    const int hn[2] = {(int)hd[0].size(), (int)hd[1].size()};
    const int fn[2] = {(int)fd[0].size(), (int)fd[1].size()};
    (void)hp; (void)fp; (void)fl; (void)hn; (void)fn;
    for (int par = 0; par < 2; ++par) {
      c->c_hd[par] = hd[par];
      c->c_fd[par] = fd[par];
      c->c_ff[par] = ff[par];
      c->c_hin[par] = hin[par];
      c->c_fin[par] = fin[par];
    }
    c->const_ready = true;
    if (c->device < 64 && g_const_owner[c->device] == c.get()) g_const_owner[c->device] = nullptr;
    bind_constants(c.get());
    {  // the force table's shared-memory window, around the stencil's shells
      std::vector<double> shells;
      for (int par = 0; par < 2; ++par)
        for (const Offset& o : c->offs.full[par]) {
          const double hh = o.cross ? (par ? -0.5 : 0.5) : 0.0;
          const double x = o.dx + hh, y = o.dy + hh, z = o.dz + hh;
          const double r = std::sqrt(x * x + y * y + z * z) * box->a0;
          if (r <= pot->cutoff) shells.push_back(r);
        }
      std::sort(shells.begin(), shells.end());
      std::vector<double> uniq;
      for (double r : shells)
        if (uniq.empty() || r - uniq.back() > 1e-6) uniq.push_back(r);
      c->shells = uniq;  // force_window_setup, once the tables exist
    }
    // ghost list and owner map
    const long long S = c->S;
    std::vector<int> tgt(S), gdst, gsrc;
    std::vector<signed char> gk;
    for (long long cell = 0; cell < G.NC; ++cell) {
      int cx, cy, cz;
      cell_xyz(cell, G, cx, cy, cz);
      const bool ghost = cell_is_ghost(cx, cy, cz, G);
      // z-halo planes of a slab rank are remote: filled by the position halo,
      // their partials returned by the reverse halos (tgt = the x/y owner
      // column in the same plane)
      const bool remote = G.slab && (cz < G.g || cz >= G.g + G.bz);
      const long kx = floor_div(cx - G.g, G.bx), ky = floor_div(cy - G.g, G.by),
                 kz = floor_div(cz - G.g, G.bz);
      const long long scell = cell_of((int)(cx - kx * G.bx), (int)(cy - ky * G.by),
                                      (int)(cz - kz * G.bz), G);
      for (int par = 0; par < 2; ++par) {
        const long long d = par * G.NC + cell;
        if (!ghost) {
          tgt[d] = (int)d;
          continue;
        }
        if (remote) {  // in-plane owner column; the plane itself comes by exchange
          tgt[d] = (int)(par * G.NC + cell_of((int)(cx - kx * G.bx), (int)(cy - ky * G.by), cz, G));
          continue;
        }
        const long long s = par * G.NC + scell;
        tgt[d] = (int)s;
        gdst.push_back((int)d);
        gsrc.push_back((int)s);
        gk.push_back((signed char)kx);
        gk.push_back((signed char)ky);
        gk.push_back((signed char)kz);
      }
    }
    KP& P = c->P;
    P.G = G;
    P.S = S;
    for (int par = 0; par < 2; ++par) {
      P.skh[par] = skh[par];
      P.skf[par] = skf[par];
    }
    P.nin64 = std::max(std::max(hin[0], hin[1]), std::max(fin[0], fin[1])) <= 64;
    P.skin_reach[0] = sreach[0];
    P.skin_reach[1] = sreach[1];
    P.accel = accel_factor();
    P.mv2 = mv2_to_ev();
    c->mem_cat = CBX_MEM_SLOTS;
    P.pdf = c->alloc<double4>(S);
    P.rho = c->alloc<double>(S);
    P.vel = c->alloc<double>(3 * S);
    P.frc = c->alloc<double>(3 * S);
    P.tag = c->alloc<unsigned long long>(S);
    P.tgt = c->alloc<int>(S);
    P.head = c->alloc<int>(S);
    P.n_gh = (long long)gdst.size();
    c->n_ghost = (int)gdst.size();
    c->mem_cat = CBX_MEM_GHOSTS;
    P.gh_dst = c->alloc<int>(gdst.size());
    P.gh_src = c->alloc<int>(gsrc.size());
    P.gh_k = c->alloc<signed char>(gk.size());
    cuda_check(cudaMemcpy(P.tgt, tgt.data(), S * sizeof(int), cudaMemcpyHostToDevice), "tgt");
    if (!gdst.empty()) {
      cudaMemcpy(P.gh_dst, gdst.data(), gdst.size() * sizeof(int), cudaMemcpyHostToDevice);
      cudaMemcpy(P.gh_src, gsrc.data(), gsrc.size() * sizeof(int), cudaMemcpyHostToDevice);
      cudaMemcpy(P.gh_k, gk.data(), gk.size(), cudaMemcpyHostToDevice);
    }
    // clash list, movers, sort scratch
    const char* env = std::getenv("CBX_CLASH_CAPACITY");
    int cap = env ? std::atoi(env) : (int)std::max<long long>(1 << 14, S / 64);
    cap = std::min(cap, 1 << 22);
    P.cap_clash = cap;
    P.cap_mov = cap;
    int items = 1;
    while (items < 2 * cap) items <<= 1;
    P.cap_items = items;
    c->mem_cat = CBX_MEM_CLASH;
    alloc_clash(c.get(), P.cl, cap);
    alloc_clash(c.get(), P.cl2, cap);
    c->mem_cat = CBX_MEM_REHASH;
    for (Movers* M : {&P.mv, &P.out}) {
      M->key = c->alloc<long long>(cap);
      M->walk = c->alloc<long long>(cap);
      M->sub = c->alloc<long long>(cap);
      M->cls = c->alloc<int>(cap);
      M->dir = c->alloc<int>(cap);
      M->px = c->alloc<double>(cap);
      M->py = c->alloc<double>(cap);
      M->pz = c->alloc<double>(cap);
      M->vx = c->alloc<double>(cap);
      M->vy = c->alloc<double>(cap);
      M->vz = c->alloc<double>(cap);
      M->tag = c->alloc<unsigned long long>(cap);
    }
    P.cap_rem = std::max(4096, cap / 4);
    c->mem_cat = CBX_MEM_CLASH;
    alloc_clash(c.get(), P.rem, P.cap_rem);
    c->mem_cat = CBX_MEM_REHASH;
    P.sc.k1 = c->alloc<long long>(items);
    P.sc.k2 = c->alloc<long long>(items);
    P.sc.k3 = c->alloc<long long>(items);
    P.sc.pl = c->alloc<int>(items);
    P.sc.flag = c->alloc<int>(items);
    P.sc.pos = c->alloc<int>(items);
    // tables and partials
    c->mem_cat = CBX_MEM_TABLES;
    P.dens = upload_tab(c.get(), c->pot.dens);
    P.zr = upload_tab(c.get(), c->pot.zr);
    P.emb = upload_tab(c.get(), c->pot.embed);
    P.cutoff = pot->cutoff;
    P.cut2 = pot->cutoff * pot->cutoff;
    P.mass = pot->mass;
    const int np = std::max(std::max(eam_blocks(P), embed_blocks(P)), 4 * 148 * 16);
    P.n_part = np;
    c->mem_cat = CBX_MEM_REDUCTION;
    P.part_emb = c->alloc<double>(np);
    P.part_pair = c->alloc<double>(np);
    P.part_ke = c->alloc<double>(np);
    P.part_vmax = c->alloc<double>(np);
    cudaMemset(P.part_emb, 0, np * sizeof(double));
    cudaMemset(P.part_pair, 0, np * sizeof(double));
    cudaMemset(P.part_ke, 0, np * sizeof(double));
    cudaMemset(P.part_vmax, 0, np * sizeof(double));
    c->mem_cat = CBX_MEM_SLOTS;
    P.uf = c->alloc<float4>(S);
    P.offs_const = ab_flag("CBX_OFFS_CONST", 1);
    P.unit_rr = ab_flag("CBX_UNIT_RR", 14);
    {
      // round-robin batches need several per CTA to balance: a small box
      // (config 2: 1027 units, 7 per CTA) would leave half the CTAs without a
      // batch, so it keeps one contiguous unit range per CTA
      int sms = 148, dv = 0;
      cudaGetDevice(&dv);
      cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dv);
      const long long nu = (long long)((G.bx * G.by + 31) / 32) * ((G.bz + 3) / 4);
      if (P.unit_rr > 0 && nu < 2LL * P.unit_rr * sms) P.unit_rr = 0;
    }
    P.idle_pred = ab_flag("CBX_IDLE_PRED", 1);
    P.skin_lane = ab_flag("CBX_SKIN_LANE", 1);
    P.tab_packed = ab_flag("CBX_TAB_PACKED", 1);
    c->mem_cat = CBX_MEM_REDUCTION;
    P.work = c->alloc<int>(4);
    cudaMemset(P.work, 0, 4 * sizeof(int));
    c->mem_cat = CBX_MEM_TABLES;
    setup_fast(c.get());
    force_window_setup(c.get(), c->shells);
    c->mem_cat = CBX_MEM_REDUCTION;
    P.st = c->alloc<DevStatus>(1);
    P.dself = c->alloc<KP>(1);
    c->d_rem_base = c->alloc<int>(2);
    {  // the Wigner-Seitz ball of a BCC site: every other site is >= sqrt(3)/2 a0 away
      const double r = (std::sqrt(3.0) / 4.0 - 1e-6) * G.a0;
      P.hash_r2 = ab_flag("CBX_FAST_HASH", 1) ? r * r : 0.0;
    }
    {
      const int maxn = std::max(std::max(fd[0].size(), fd[1].size()), std::max(hd[0].size(), hd[1].size()));
      c->mem_cat = CBX_MEM_SLOTS;
      P.pmask = maxn <= 126 && !ab_flag("CBX_NOMASK", 0) ? c->alloc<unsigned long long>(2 * S)
                                                         : nullptr;
    }

    // regional displacement bounds (density-pass skin pruning): rows of
    // whole 32-cell chunks only
    P.ub = nullptr;
    P.ustamp = nullptr;
    if (G.bx % 32 == 0 && G.g <= 32 && ab_flag("CBX_SKIN_PRUNE", 1)) {
      c->mem_cat = CBX_MEM_SLOTS;
      P.ub = c->alloc<unsigned long long>(G.NI / 32);
      cudaMemset(P.ub, 0, (G.NI / 32) * sizeof(unsigned long long));
      c->mem_cat = CBX_MEM_REDUCTION;
      P.ustamp = c->alloc<unsigned long long>(2);
      const unsigned long long st0[2] = {0ull, 1ull};
      cudaMemcpy(P.ustamp, st0, sizeof(st0), cudaMemcpyHostToDevice);
    }
    c->mem_cat = CBX_MEM_REDUCTION;
    P.skin_cnt = c->alloc<unsigned long long>(3);
    cudaMemset(P.skin_cnt, 0, 3 * sizeof(unsigned long long));
    c->d_defects = c->alloc<unsigned long long>(4);
    // empty store: every slot vacant
    std::vector<double4> vac(S, make_double4(kVacant, kVacant, kVacant, 0.0));
    cuda_check(cudaMemcpy(P.pdf, vac.data(), S * sizeof(double4), cudaMemcpyHostToDevice), "init");
    cudaMemset(P.rho, 0, S * sizeof(double));
    cudaMemset(P.vel, 0, 3 * S * sizeof(double));
    cudaMemset(P.frc, 0, 3 * S * sizeof(double));
    cudaMemset(P.tag, 0, S * sizeof(unsigned long long));
    cudaMemset(P.head, 0xff, S * sizeof(int));
    launch_uf_refresh(P, c->stream);
    P.n_pair_part = pair_partials(P, 0);
    sync_kp(c.get());
    c->hst = DevStatus{};
    c->hst.dt_next = 1e-3;
    c->hst.dt_max = 1e-3;
    c->hst.max_disp = 0.05;
    cuda_check(cudaMemcpy(P.st, &c->hst, sizeof(DevStatus), cudaMemcpyHostToDevice), "status");
    cuda_check(cudaDeviceSynchronize(), "create");
  });
  if (rc == CBX_OK) *out = c.release();
  else {
    for (void* p : c->allocs) cudaFree(p);
  }
  return rc;
}

CBX_API cbx_status cbx_create(const cbx_box* box, const cbx_potential* pot,
                              const cbx_offsets* idx, int device, cbx_ctx** out) {
  return create_impl(box, pot, idx, device, nullptr, out);
}

CBX_API void cbx_destroy(cbx_ctx* c) {
  if (!c) return;
  cudaSetDevice(c->device);
  if (c->device >= 0 && c->device < 64 && g_const_owner[c->device] == c)
    g_const_owner[c->device] = nullptr;
  drop_graph(c);
  for (SnapSlot& q : c->snap) {
    if (q.writer.joinable()) q.writer.join();
    if (q.dev) cudaFree(q.dev);
    if (q.host) cudaFreeHost(q.host);
    if (q.packed) cudaEventDestroy(q.packed);
    if (q.copied) cudaEventDestroy(q.copied);
  }
  if (c->snap_stream) cudaStreamDestroy(c->snap_stream);
  if (c->comm) {
    if (c->stream) cudaStreamSynchronize(c->stream);
    nccl().comm_destroy(c->comm);
    c->comm = nullptr;
  }
  for (void* p : c->p2p_opened) cudaIpcCloseMemHandle(p);
  if (c->p2p_region) cudaFree(c->p2p_region);
  if (c->stream) cudaStreamSynchronize(c->stream);
  for (cudaTextureObject_t t : c->textures) cudaDestroyTextureObject(t);
  for (void* p : c->allocs) cudaFree(p);
  if (c->flush_buf) cudaFree(c->flush_buf);
  for (auto& e : c->ev)
    if (e) cudaEventDestroy(e);
  for (auto& e : c->ev_outer)
    if (e) cudaEventDestroy(e);
  if (c->stream) cudaStreamDestroy(c->stream);
  delete c;
}

CBX_API cbx_status cbx_set_stencil(cbx_ctx* c, cbx_stencil mode) {
  return guarded(c, [&] {
    if (mode != CBX_STENCIL_NEWTON3 && mode != CBX_STENCIL_FULL &&
        mode != CBX_STENCIL_REFERENCE)
      raise(CBX_INVALID_ARGUMENT, "unknown stencil mode");
    if (mode != CBX_STENCIL_REFERENCE && !c->fast_ok)
      raise(CBX_INVALID_ARGUMENT, "fast stencils need z(r) and rho(r) on one grid");
    if (c->mode != mode) drop_graph(c);
    c->mode = mode;
    c->mask_valid = false;
    c->P.rev.on = rev_fused(c);
    sync_kp(c);
  });
}

CBX_API long cbx_slot_count(const cbx_ctx* c) { return (long)c->S; }

CBX_API cbx_status cbx_upload_store(cbx_ctx* c, const cbx_store* s) {
  return guarded(c, [&] {
    cudaSetDevice(c->device);
    do_upload(c, s);
  });
}
CBX_API cbx_status cbx_download_store(cbx_ctx* c, cbx_store* s) {
  return guarded(c, [&] {
    cudaSetDevice(c->device);
    do_download(c, s);
  });
}
CBX_API long cbx_clash_count(cbx_ctx* c) {
  cudaSetDevice(c->device);
  sync_status(c);
  return c->hst.n_clash;
}

CBX_API cbx_status cbx_init_bcc(cbx_ctx* c, int species, double temperature, uint64_t seed,
                                long* n_atoms) {
  (void)species;
  return guarded(c, [&] {
    cudaSetDevice(c->device);
    // a slab rank keeps its planes of the global lattice (same RNG stream,
    // so the decomposed initial state equals the single-box one)
    HostLattice L = c->G.slab ? init_bcc_slab(c->gbox, c->G, c->pot.mass, temperature, seed)
                              : init_bcc(c->box, c->pot.mass, temperature, seed);
    cbx_store s{};
    s.n_slots = c->S;
    s.pos = L.pos.data();
    s.vel = L.vel.data();
    s.tag = L.tag.data();
    s.valid = L.valid.data();
    do_upload(c, &s);
    if (n_atoms) *n_atoms = L.n_atoms;
  });
}

CBX_API cbx_status cbx_rehash(cbx_ctx* c) {
  return guarded(c, [&] {
    cudaSetDevice(c->device);
    require_box(c, "cbx_rehash");
    launch_kick_drift(c->P, 0, c->stream);
    launch_rehash(c->P, c->stream);
    c->launches += 2;
    seq_fill_ghosts(c);
    sync_status(c);
    raise_device_error(c, false);
  });
}
CBX_API cbx_status cbx_fill_ghosts(cbx_ctx* c) {
  return guarded(c, [&] {
    cudaSetDevice(c->device);
    require_box(c, "cbx_fill_ghosts");
    seq_fill_ghosts(c);
    sync_status(c);
    raise_device_error(c, false);
  });
}

CBX_API cbx_status cbx_eval_forces(cbx_ctx* c, double* e_emb, double* e_pair) {
  return guarded(c, [&] {
    cudaSetDevice(c->device);
    check_cutoff(c);
    require_box_or_comm(c, "cbx_eval_forces");
    if (has_transport(c)) {
      seq_slab_eval(c);
    } else {
      ev_mark(c, 1);
      seq_density(c);
      ev_mark(c, 2);
      seq_embed(c);
      ev_mark(c, 3);
      seq_force(c);
      ev_mark(c, 4);
      launch_finalize(c->P, -1, 1, c->stream);
      c->launches += 1;
    }
    sync_status(c);
    accumulate_timing(c, false);
    raise_device_error(c, false);
    if (e_emb) *e_emb = c->hst.embedding;
    if (e_pair) *e_pair = c->hst.pair;
  });
}
CBX_API cbx_status cbx_compute_density(cbx_ctx* c) {
  return guarded(c, [&] {
    cudaSetDevice(c->device);
    require_box(c, "cbx_compute_density");
    check_cutoff(c);
    seq_density(c);
    sync_status(c);
    raise_device_error(c, false);
  });
}
CBX_API cbx_status cbx_compute_embedding_derivative(cbx_ctx* c, double* e_emb) {
  return guarded(c, [&] {
    cudaSetDevice(c->device);
    require_box(c, "cbx_compute_embedding_derivative");
    seq_embed(c);
    launch_finalize(c->P, -1, 1, c->stream);
    c->launches += 1;
    sync_status(c);
    raise_device_error(c, false);
    if (e_emb) *e_emb = c->hst.embedding;
  });
}
CBX_API cbx_status cbx_compute_pair_forces(cbx_ctx* c, double* e_pair) {
  return guarded(c, [&] {
    cudaSetDevice(c->device);
    require_box(c, "cbx_compute_pair_forces");
    check_cutoff(c);
    seq_force(c);
    launch_finalize(c->P, -1, 1, c->stream);
    c->launches += 1;
    sync_status(c);
    raise_device_error(c, false);
    if (e_pair) *e_pair = c->hst.pair;
  });
}
CBX_API cbx_status cbx_guards(cbx_ctx* c, uint64_t out[2]) {
  return guarded(c, [&] {
    cudaSetDevice(c->device);
    sync_status(c);
    out[0] = c->hst.r_underflow;
    out[1] = c->hst.rho_clamp;
  });
}

CBX_API cbx_status cbx_set_adaptive(cbx_ctx* c, double dt_max, double max_disp) {
  return guarded(c, [&] {
    sync_status(c);
    c->hst.dt_max = dt_max;
    c->hst.max_disp = max_disp;
    write_status(c);
  });
}

CBX_API cbx_status cbx_step(cbx_ctx* c, double dt, long nsteps, cbx_state* out) {
  return guarded(c, [&] {
    cudaSetDevice(c->device);
    check_cutoff(c);
    if (nsteps < 0) raise(CBX_INVALID_ARGUMENT, "nsteps must be >= 0");
    require_box_or_comm(c, "cbx_step");
    const bool fresh = c->st_was_fresh;
    if (!fresh) sync_status(c);
    if (dt > 0.0) {
      if (!fresh || c->hst.adaptive || c->hst.dt_next != dt) {
        c->hst.dt_next = dt;
        c->hst.adaptive = 0;
        write_status(c);
      }
    } else {
      c->hst.adaptive = 1;
      c->hst.dt_next = cbx_adaptive_dt(c->hst.max_speed, c->hst.dt_max, c->hst.max_disp);
      write_status(c);
    }
    struct Single {  // single-step mode for this call only
      cbx_ctx* c;
      ~Single() { c->single = false; }
    } single_guard{c};
    c->single = nsteps == 1;
    if (!c->single && c->step_graph &&
        (c->g_defer != want_defer(c) || c->g_merge != want_merge(c))) {
      cudaGraphExecDestroy(c->step_graph);
      c->step_graph = nullptr;
    }
    if (c->use_graph && !c->timing) build_graph(c);
    for (long i = 0; i < nsteps; ++i) {
      if (c->use_graph && !c->timing) {
        if (c->single) {
          cuda_check(cudaGraphLaunch(c->step_graph1, c->stream), "graph launch");
          c->launches += c->graph1_launches;
          continue;
        }
        cuda_check(cudaGraphLaunch(c->step_graph, c->stream), "graph launch");
        c->launches += c->g_launches;
        if (c->g_merge) c->k2_maybe = true;
        else if (c->g_defer) c->fin_maybe = true;
      } else {
        seq_step(c);
        accumulate_timing(c, true);
      }
    }
    sync_status(c);
    raise_device_error(c, true);
    c->st_fresh = true;
    if (out) {
      out->step = (long)c->hst.step;
      out->t = c->hst.t;
      out->dt = c->hst.dt;
      out->kinetic = c->hst.kinetic;
      out->pair = c->hst.pair;
      out->embedding = c->hst.embedding;
      out->max_speed = c->hst.max_speed;
      out->r_underflow = c->hst.r_underflow;
      out->rho_clamp = c->hst.rho_clamp;
    }
  });
}

CBX_API cbx_status cbx_refresh_forces(cbx_ctx* c) {
  return cbx_eval_forces(c, nullptr, nullptr);
}

CBX_API cbx_status cbx_measure(cbx_ctx* c) {
  return guarded(c, [&] {
    cudaSetDevice(c->device);
    if (has_transport(c)) {
      slab_finish(c, 0, 0, 0);
    } else {
      launch_kick2(c->P, 0, 0, 0, c->stream);
      c->launches += 1;
    }
    sync_status(c);
    raise_device_error(c, false);
  });
}

CBX_API cbx_status cbx_get_state(cbx_ctx* c, cbx_state* out) {
  return guarded(c, [&] {
    cudaSetDevice(c->device);
    sync_status(c);
    out->step = (long)c->hst.step;
    out->t = c->hst.t;
    out->dt = c->hst.dt;
    out->kinetic = c->hst.kinetic;
    out->pair = c->hst.pair;
    out->embedding = c->hst.embedding;
    out->max_speed = c->hst.max_speed;
    out->r_underflow = c->hst.r_underflow;
    out->rho_clamp = c->hst.rho_clamp;
  });
}
CBX_API cbx_status cbx_set_state(cbx_ctx* c, const cbx_state* in) {
  return guarded(c, [&] {
    cudaSetDevice(c->device);
    sync_status(c);
    c->hst.step = in->step;
    c->hst.t = in->t;
    c->hst.dt = in->dt;
    c->hst.kinetic = in->kinetic;
    c->hst.pair = in->pair;
    c->hst.embedding = in->embedding;
    c->hst.max_speed = in->max_speed;
    c->hst.r_underflow = in->r_underflow;
    c->hst.rho_clamp = in->rho_clamp;
    write_status(c);
  });
}

CBX_API cbx_status cbx_inject_pka(cbx_ctx* c, int64_t site, const double v[3]) {
  const cbx_status rc = guarded(c, [&] {
    cudaSetDevice(c->device);
    if (site < 0 || site >= c->S) raise(CBX_INVALID_ARGUMENT, "pka.site: site id out of range");
    const long long d = dev_of_ref(site, c->G.NC);
    double4 p;
    cuda_check(cudaMemcpy(&p, c->P.pdf + d, sizeof p, cudaMemcpyDeviceToHost), "pka");
    if (p.x >= kVacantTest) {
      int cx, cy, cz;
      cell_xyz(site >> 1, c->G, cx, cy, cz);
      raise(CBX_INVALID_ARGUMENT, "pka.site: no atom at cell (" + std::to_string(cx - c->G.g) +
                                      "," + std::to_string(cy - c->G.g) + "," +
                                      std::to_string(cz - c->G.g) + ")");
    }
    for (int a = 0; a < 3; ++a)
      cuda_check(cudaMemcpy(c->P.vel + a * c->S + d, &v[a], sizeof(double),
                            cudaMemcpyHostToDevice),
                 "pka");
  });
  // a slab rank only sets the velocity: cbx_measure is collective there
  return rc == CBX_OK && !c->G.slab ? cbx_measure(c) : rc;
}

// ---- thermostat_rescale (sim.cpp:188-221) ---------------------------------
namespace {
__device__ __forceinline__ bool in_band_dev(long long id, const Geo& G, long band) {
  if (band <= 0) return true;
  const long long tx2 = 2ll * G.tx;
  const long cz = (long)(id / (tx2 * G.ty)), cy = (long)((id / tx2) % G.ty);
  const long cx = (long)((id % tx2) >> 1), g = G.g;
  return cx - g < band || (g + G.bx - 1) - cx < band || cy - g < band ||
         (g + G.by - 1) - cy < band || cz - g < band || (g + G.bz - 1) - cz < band;
}

// blocks [0, nsb): interior slots; [nsb, grid): interior clash records.
// Per-block partial sums of |v|^2 and the in-band atom count.
__global__ void k_thermo_sum(KP P, long band, int nsb, double* psum, double* pcnt) {
  __shared__ double sh[8];
  double v2 = 0.0, n = 0.0;
  if (blockIdx.x < nsb) {
    int par;
    long long d;
    if (map_site(P, par, d) && P.pdf[d].x < kVacantTest &&
        in_band_dev(ref_of_dev(d, P.G.NC), P.G, band)) {
      const long long S = P.S;
      v2 = exact_r2(P.vel[d], P.vel[S + d], P.vel[2 * S + d]);
      n = 1.0;
    }
  } else {
    const int nc = P.st->n_clash;
    for (int i = (blockIdx.x - nsb) * blockDim.x + threadIdx.x; i < nc;
         i += (gridDim.x - nsb) * blockDim.x)
      if (!P.cl.gf[i] && in_band_dev(P.cl.key[i], P.G, band)) {
        v2 += exact_r2(P.cl.vx[i], P.cl.vy[i], P.cl.vz[i]);
        n += 1.0;
      }
  }
  const double a = block_sum<256>(v2, sh);
  const double b = block_sum<256>(n, sh);
  if (threadIdx.x == 0) {
    psum[blockIdx.x] = a;
    pcnt[blockIdx.x] = b;
  }
}

__global__ void k_thermo_scale(KP P, long band, int nsb, double f) {
  if (blockIdx.x < nsb) {
    int par;
    long long d;
    if (map_site(P, par, d) && P.pdf[d].x < kVacantTest &&
        in_band_dev(ref_of_dev(d, P.G.NC), P.G, band)) {
      const long long S = P.S;
      P.vel[d] *= f;
      P.vel[S + d] *= f;
      P.vel[2 * S + d] *= f;
    }
  } else {
    const int nc = P.st->n_clash;
    for (int i = (blockIdx.x - nsb) * blockDim.x + threadIdx.x; i < nc;
         i += (gridDim.x - nsb) * blockDim.x)
      if (!P.cl.gf[i] && in_band_dev(P.cl.key[i], P.G, band)) {
        P.cl.vx[i] *= f;
        P.cl.vy[i] *= f;
        P.cl.vz[i] *= f;
      }
  }
}

const char* const kSymbols[] = {  // analysis.cpp:11-19
    "X",  "H",  "He", "Li", "Be", "B",  "C",  "N",  "O",  "F",  "Ne", "Na", "Mg", "Al", "Si",
    "P",  "S",  "Cl", "Ar", "K",  "Ca", "Sc", "Ti", "V",  "Cr", "Mn", "Fe", "Co", "Ni", "Cu",
    "Zn", "Ga", "Ge", "As", "Se", "Br", "Kr", "Rb", "Sr", "Y",  "Zr", "Nb", "Mo", "Tc", "Ru",
    "Rh", "Pd", "Ag", "Cd", "In", "Sn", "Sb", "Te", "I",  "Xe", "Cs", "Ba", "La", "Ce", "Pr",
    "Nd", "Pm", "Sm", "Eu", "Gd", "Tb", "Dy", "Ho", "Er", "Tm", "Yb", "Lu", "Hf", "Ta", "W",
    "Re", "Os", "Ir", "Pt", "Au", "Hg", "Tl", "Pb", "Bi", "Po", "At", "Rn", "Fr", "Ra", "Ac",
    "Th", "Pa", "U"};
}  // namespace

CBX_API cbx_status cbx_thermostat_rescale(cbx_ctx* c, double temperature, long boundary_cells) {
  const cbx_status rc = guarded(c, [&] {
    cudaSetDevice(c->device);
    require_box(c, "cbx_thermostat_rescale");
    // a pending merged second half kick / deferred StepState sum first: the
    // sums below read the velocities and reuse the KE partials as scratch
    sync_status(c);
    raise_device_error(c, false);
    const int nsb = eam_blocks(c->P), grid = nsb + 8;
    double* psum = c->P.part_ke;  // scratch: the next measure rewrites them
    double* pcnt = c->P.part_vmax;
    if (grid > c->P.n_part) raise(CBX_RUNTIME, "thermostat: partial buffer too small");
    k_thermo_sum<<<grid, 256, 0, c->stream>>>(c->P, boundary_cells, nsb, psum, pcnt);
    std::vector<double> hs(grid), hc(grid);
    cuda_check(cudaMemcpyAsync(hs.data(), psum, grid * sizeof(double), cudaMemcpyDeviceToHost,
                               c->stream), "thermostat");
    cuda_check(cudaMemcpyAsync(hc.data(), pcnt, grid * sizeof(double), cudaMemcpyDeviceToHost,
                               c->stream), "thermostat");
    sync_status(c);
    raise_device_error(c, false);
    double sum_v2 = 0.0, n = 0.0;
    for (int i = 0; i < grid; ++i) {
      sum_v2 += hs[i];
      n += hc[i];
    }
    const double measured =
        n > 0.0 ? c->pot.mass * sum_v2 * mv2_to_ev() / (3.0 * n * boltzmann_ev()) : 0.0;
    if (!(measured > 0.0)) {
      std::fprintf(stderr, "thermostat: measured temperature is zero, skipping\n");
      c->launches += 1;
      return;
    }
    const double f = std::sqrt(temperature / measured);
    k_thermo_scale<<<grid, 256, 0, c->stream>>>(c->P, boundary_cells, nsb, f);
    c->launches += 2;
    c->mask_valid = false;
  });
  return rc == CBX_OK ? cbx_measure(c) : rc;
}

// ---- write_snapshot (analysis.cpp:90-116) with an asynchronous D2H --------
// The interior slots in reference-id order (for_each_interior_id,
// store.h:82-93) and the clash records in (key, bucket) order are packed on
// the step stream into a device buffer (one 32-byte entry per site / record:
// x, y, z, tag bits; vacant sites and ghost records flagged by x = 1e30),
// copied to page-locked host memory on a side stream, and formatted by a host
// thread -- while the following steps run.  Two slots: a third snapshot waits
// for the oldest.  The file text equals the reference's byte for byte.
namespace {
__global__ void k_snapshot_pack(KP P, double4* out, long long ni, int n_clash) {
  const Geo& G = P.G;
  const long long row = 2ll * G.bx;
  for (long long e = (long long)blockIdx.x * blockDim.x + threadIdx.x; e < ni + n_clash;
       e += (long long)gridDim.x * blockDim.x) {
    if (e < ni) {
      const long long r = e / row, x2 = e - r * row;
      const int y = (int)(r % G.by), z = (int)(r / G.by);
      const int par = (int)(x2 & 1);
      const long long d =
          par * G.NC + cell_of((int)(x2 >> 1) + G.g, y + G.g, z + G.g, G);
      const double4 p = P.pdf[d];
      out[e] = make_double4(p.x, p.y, p.z, __longlong_as_double((long long)P.tag[d]));
    } else {
      const int i = (int)(e - ni);
      out[e] = make_double4(P.cl.gf[i] ? kVacant : P.cl.px[i], P.cl.py[i], P.cl.pz[i],
                            __longlong_as_double((long long)P.cl.tag[i]));
    }
  }
}

// the reference's text from a packed snapshot (host side, any thread)
bool format_snapshot(const char* path, const double4* e, long long ni, long nc, double t_ps,
                     const cbx_box& box, const char* sym) {
  long n_atoms = 0;
  for (long long i = 0; i < ni + nc; ++i) n_atoms += e[i].x < kVacantTest;
  std::FILE* f = std::fopen(path, "w");
  if (!f) return false;
  const double a0 = box.a0, shift = box.ghost_width * a0;
  char tb[48];
  std::snprintf(tb, sizeof tb, "%.9g", t_ps);  // csv_time (analysis.cpp:66-75)
  if (!std::strpbrk(tb, ".eE") && std::strspn(tb, "-0123456789") == std::strlen(tb))
    std::strcat(tb, ".0");
  std::fprintf(f, "%ld\n", n_atoms);
  std::fprintf(f,
               "Lattice=\"%.10g 0 0 0 %.10g 0 0 0 %.10g\" "
               "Properties=species:S:1:pos:R:3:tag:I:1 Time=%s\n",
               box.box_x * a0, box.box_y * a0, box.box_z * a0, tb);
  for (long long i = 0; i < ni + nc; ++i) {
    if (!(e[i].x < kVacantTest)) continue;
    unsigned long long tag;
    std::memcpy(&tag, &e[i].w, sizeof tag);
    std::fprintf(f, "%s %.10g %.10g %.10g %llu\n", sym, e[i].x - shift, e[i].y - shift,
                 e[i].z - shift, tag);
  }
  const bool bad = std::ferror(f) != 0;
  std::fclose(f);
  return !bad;
}

// wait for snapshot slot k's writer; its error text, if any
std::string snapshot_join(cbx_ctx* c, int k) {
  SnapSlot& q = c->snap[k];
  if (q.writer.joinable()) q.writer.join();
  std::string e;
  e.swap(q.error);
  return e;
}
}  // namespace

// pack + async D2H + background formatting of one snapshot
void snapshot_async(cbx_ctx* c, const std::string& path, double t_ps) {
  const Geo& G = c->G;
  const long long ni = 2ll * G.bx * G.by * G.bz;
  const int k = c->snap_next;
  const std::string prev = snapshot_join(c, k);
  if (!prev.empty()) raise(CBX_RUNTIME, prev);
  SnapSlot& q = c->snap[k];
  sync_status(c);  // n_clash, pending kicks
  raise_device_error(c, false);
  const int nc = c->hst.n_clash;
  const size_t need = (size_t)(ni + nc) * sizeof(double4);
  if (need > q.bytes) {
    if (q.dev) cudaFree(q.dev);
    if (q.host) cudaFreeHost(q.host);
    q.dev = nullptr;
    q.host = nullptr;
    const size_t cap = (size_t)(ni + c->P.cap_clash) * sizeof(double4);
    cuda_check(cudaMalloc(&q.dev, cap), "snapshot buffer");
    cuda_check(cudaHostAlloc(&q.host, cap, cudaHostAllocDefault), "snapshot host buffer");
    q.bytes = cap;
  }
  if (!c->snap_stream)
    cuda_check(cudaStreamCreateWithFlags(&c->snap_stream, cudaStreamNonBlocking), "stream");
  if (!q.packed) cuda_check(cudaEventCreateWithFlags(&q.packed, cudaEventDisableTiming), "event");
  if (!q.copied) cuda_check(cudaEventCreateWithFlags(&q.copied, cudaEventDisableTiming), "event");
  const long long n = ni + nc;
  const int grid = (int)std::min<long long>((n + 255) / 256, 8 * 148);
  k_snapshot_pack<<<grid, 256, 0, c->stream>>>(c->P, q.dev, ni, nc);
  c->launches += 1;
  cuda_check(cudaEventRecord(q.packed, c->stream), "event");
  cuda_check(cudaStreamWaitEvent(c->snap_stream, q.packed, 0), "event");
  cuda_check(cudaMemcpyAsync(q.host, q.dev, (size_t)n * sizeof(double4), cudaMemcpyDeviceToHost,
                             c->snap_stream),
             "snapshot D2H");
  cuda_check(cudaEventRecord(q.copied, c->snap_stream), "event");
  const unsigned z = (unsigned)c->pot.atomic_number;
  const char* sym = z < sizeof(kSymbols) / sizeof(kSymbols[0]) ? kSymbols[z] : "X";
  const int dev = c->device;
  const cbx_box box = c->box;
  q.writer = std::thread([&q, path, t_ps, ni, nc, box, sym, dev] {
    cudaSetDevice(dev);
    if (cudaEventSynchronize(q.copied) != cudaSuccess) {
      q.error = "snapshot copy failed: " + path;
      return;
    }
    if (!format_snapshot(path.c_str(), q.host, ni, nc, t_ps, box, sym))
      q.error = "cannot write " + path;
  });
  c->snap_next ^= 1;
}

// every pending snapshot written (the first error raised)
void snapshot_wait(cbx_ctx* c) {
  std::string err;
  for (int k = 0; k < 2; ++k) {
    const std::string e = snapshot_join(c, k);
    if (err.empty()) err = e;
  }
  if (!err.empty()) raise(CBX_RUNTIME, err);
}

CBX_API cbx_status cbx_write_snapshot_async(cbx_ctx* c, const char* path, double t_ps) {
  return guarded(c, [&] {
    cudaSetDevice(c->device);
    require_box(c, "cbx_write_snapshot");
    snapshot_async(c, path, t_ps);
  });
}

CBX_API cbx_status cbx_snapshot_wait(cbx_ctx* c) {
  return guarded(c, [&] { snapshot_wait(c); });
}

// write_snapshot (analysis.cpp:90-116): interior slots in id order, then the
// interior clash records in (key, bucket) order, at time t_ps; returns once
// the file is written
CBX_API cbx_status cbx_write_snapshot(cbx_ctx* c, const char* path, double t_ps) {
  return guarded(c, [&] {
    cudaSetDevice(c->device);
    require_box(c, "cbx_write_snapshot");
    snapshot_async(c, path, t_ps);
    snapshot_wait(c);
  });
}

// ---- Simulation::run (sim.cpp:289-360) over the public entry points ------
namespace {
void csv_time(double t, char out[48]) {  // analysis.cpp:66-75
  std::snprintf(out, 48, "%.9g", t);
  if (!std::strpbrk(out, ".eE") && std::strspn(out, "-0123456789") == std::strlen(out))
    std::strcat(out, ".0");
}
bool nonempty(const char* s) { return s && s[0]; }
}  // namespace

CBX_API cbx_status cbx_write_timeseries(const char* path, long n, const double* t,
                                        const long* d) {
  return guarded(nullptr, [&] {
    std::FILE* f = std::fopen(path, "w");
    if (!f) raise(CBX_RUNTIME, std::string("cannot open ") + path + " for writing");
    std::fputs("t_ps,vacancies,interstitials,frenkel_pairs\n", f);
    char tb[48];
    for (long i = 0; i < n; ++i) {
      csv_time(t[i], tb);
      std::fprintf(f, "%s,%ld,%ld,%ld\n", tb, d[3 * i], d[3 * i + 1], d[3 * i + 2]);
    }
    const bool bad = std::ferror(f) != 0;
    std::fclose(f);
    if (bad) raise(CBX_RUNTIME, std::string("write failed: ") + path);
  });
}

CBX_API long cbx_run_series(cbx_ctx* c, double* t, long* d) {
  const long n = (long)c->ser_t.size();
  if (t) std::memcpy(t, c->ser_t.data(), n * sizeof(double));
  if (d) std::memcpy(d, c->ser_d.data(), 3 * n * sizeof(long));
  return n;
}

CBX_API cbx_status cbx_run(cbx_ctx* c, const cbx_run_spec* r, const char* log_path) {
  if (c->G.slab) {
    set_thread_error("cbx_run: single-box contexts only");
    c->err = "cbx_run: single-box contexts only";
    return CBX_LOGIC;
  }
  std::FILE* log = nullptr;
  if (nonempty(log_path))
    log = std::strcmp(log_path, "-") == 0 ? stdout : std::fopen(log_path, "w");
  c->ser_t.clear();
  c->ser_d.clear();
  cbx_state st{};
  cbx_status rc = CBX_OK;
  auto sample = [&]() -> cbx_status {  // sim.cpp:275-277
    long d[3];
    const cbx_status e = cbx_count_defects(c, d);
    if (e) return e;
    const cbx_status g = cbx_get_state(c, &st);
    if (g) return g;
    c->ser_t.push_back(st.t);
    c->ser_d.insert(c->ser_d.end(), d, d + 3);
    return CBX_OK;
  };
  auto snapshot = [&](const char* suffix) -> cbx_status {  // sim.cpp:279-282
    if (!nonempty(r->snapshot_prefix)) return CBX_OK;
    cbx_get_state(c, &st);
    // written in the background while the next steps run (cbx_snapshot_wait
    // before cbx_run returns)
    return cbx_write_snapshot_async(c, (std::string(r->snapshot_prefix) + suffix).c_str(), st.t);
  };
  auto log_line = [&]() {
    if (!log) return;
    cbx_get_state(c, &st);
    long n_atoms = 0;
    {
      // atom count: interior slots + interior clash records (store.h:73)
      long d[3];
      cbx_count_defects(c, d);  // vacancies of the interior (cheap, keeps the count exact)
      const long sites = 2 * c->box.box_x * c->box.box_y * c->box.box_z;
      n_atoms = sites - d[0] + d[1];
    }
    const double T = n_atoms == 0 ? 0.0
                                  : 2.0 * st.kinetic / (3.0 * (double)n_atoms * boltzmann_ev());
    char tb[48];
    csv_time(st.t, tb);
    std::fprintf(log, "step %ld  t=%s ps  dt=%.4g  E=%.6f eV  T=%.1f K  FP=%ld\n", st.step, tb,
                 st.dt, st.kinetic + st.pair + st.embedding, T, c->ser_d.back());
  };
  // one step with the post-mortem outputs on failure (sim.cpp:303-315)
  auto guarded_steps = [&](long n) -> cbx_status {
    const cbx_status e = cbx_step(c, -1.0, n, &st);
    if (e) {
      const std::string err = c->err;
      cbx_snapshot_wait(c);
      if (nonempty(r->snapshot_prefix)) {
        cbx_get_state(c, &st);
        cbx_write_snapshot(c, (std::string(r->snapshot_prefix) + "_postmortem.xyz").c_str(),
                           st.t);
      }
      if (nonempty(r->timeseries))
        cbx_write_timeseries(r->timeseries, (long)c->ser_t.size(), c->ser_t.data(),
                             c->ser_d.data());
      c->err = err;
    }
    return e;
  };
  auto thermostat = [&]() { return cbx_thermostat_rescale(c, r->temperature, r->thermostat_boundary_cells); };
  do {
    if ((rc = sample())) break;
    if (r->snapshot_interval > 0 && (rc = snapshot("_000000.xyz"))) break;
    for (long i = 0; i < r->equilibration_steps && !rc; ++i) {
      if ((rc = guarded_steps(1))) break;
      if (r->thermostat_enabled && (i + 1) % r->thermostat_interval == 0) rc = thermostat();
    }
    if (rc) break;
    if (r->pka_energy_kev > 0.0) {  // Simulation::inject_pka (sim.cpp:163-186)
      const long cx = r->pka_site[0] >= 0 ? r->pka_site[0] : c->box.box_x / 2;
      const long cy = r->pka_site[1] >= 0 ? r->pka_site[1] : c->box.box_y / 2;
      const long cz = r->pka_site[2] >= 0 ? r->pka_site[2] : c->box.box_z / 2;
      const long g = c->box.ghost_width;
      const long long tx = c->box.box_x + 2 * g, ty = c->box.box_y + 2 * g;
      const long long site = ((g + cz) * ty + (g + cy)) * 2 * tx + 2 * (g + cx);
      const double dx = (double)r->pka_dir[0], dy = (double)r->pka_dir[1],
                   dz = (double)r->pka_dir[2];
      const double len = std::sqrt(dx * dx + dy * dy + dz * dz);
      if (!(len > 0.0)) {
        c->err = "pka.direction: must not be the zero vector";
        rc = CBX_INVALID_ARGUMENT;
        break;
      }
      const double v = std::sqrt(2.0 * (r->pka_energy_kev * 1000.0) / c->pot.mass) *
                       speed_factor();
      const double sc = v / len;
      const double vel[3] = {sc * dx, sc * dy, sc * dz};
      if ((rc = cbx_inject_pka(c, site, vel))) break;
    }
    long done = 0;
    bool sampled_last = true;
    const bool per_step = r->max_time > 0.0;  // the time cap is checked after every step
    while (!rc) {
      const bool step_cap = r->steps > 0 && done >= r->steps;
      cbx_get_state(c, &st);
      const bool time_cap = r->max_time > 0.0 && st.t >= r->max_time;
      const bool no_budget = r->steps == 0 && r->max_time == 0.0;
      if (step_cap || time_cap || no_budget) break;
      // steps until the next event (sample, snapshot, thermostat, cap)
      long n = 1;
      if (!per_step) {
        n = r->steps > 0 ? r->steps - done : 1;
        auto upto = [&](long iv) {
          if (iv > 0) n = std::min(n, iv - done % iv);
        };
        upto(r->defect_interval);
        upto(r->snapshot_interval);
        if (r->thermostat_enabled) upto(r->thermostat_interval);
      }
      if ((rc = guarded_steps(n))) break;
      done += n;
      if (r->thermostat_enabled && done % r->thermostat_interval == 0 && (rc = thermostat()))
        break;
      sampled_last = false;
      if (r->defect_interval > 0 && done % r->defect_interval == 0) {
        if ((rc = sample())) break;
        sampled_last = true;
        log_line();
      }
      if (r->snapshot_interval > 0 && done % r->snapshot_interval == 0) {
        char suffix[32];
        std::snprintf(suffix, sizeof suffix, "_%06ld.xyz", done);
        if ((rc = snapshot(suffix))) break;
      }
    }
    if (rc) break;
    if (!sampled_last) {
      if ((rc = sample())) break;
      log_line();
    }
    if (nonempty(r->timeseries) &&
        (rc = cbx_write_timeseries(r->timeseries, (long)c->ser_t.size(), c->ser_t.data(),
                                   c->ser_d.data())))
      break;
    rc = snapshot("_final.xyz");
  } while (false);
  {  // the background snapshot writers finish before the run returns
    const cbx_status w = cbx_snapshot_wait(c);
    if (!rc) rc = w;
  }
  if (log && log != stdout) std::fclose(log);
  if (log == stdout) std::fflush(stdout);
  return rc;
}

CBX_API cbx_status cbx_count_defects(cbx_ctx* c, long out[3]) {
  return guarded(c, [&] {
    cudaSetDevice(c->device);
    cudaMemsetAsync(c->d_defects, 0, 4 * sizeof(unsigned long long), c->stream);
    launch_count_defects(c->P, c->d_defects, c->stream);
    unsigned long long h[4];
    cuda_check(cudaMemcpyAsync(h, c->d_defects, sizeof h, cudaMemcpyDeviceToHost, c->stream),
               "defects");
    cuda_check(cudaStreamSynchronize(c->stream), "defects");
    out[0] = (long)(h[0] - h[2]);
    out[1] = (long)h[1];
    out[2] = std::max(out[0], out[1]);
  });
}

CBX_API cbx_status cbx_enable_timing(cbx_ctx* c, int on) {
  return guarded(c, [&] {
    c->timing = on != 0;
    for (double& t : c->t_ms) t = 0.0;
  });
}
CBX_API cbx_status cbx_last_timings(cbx_ctx* c, double out_ms[8]) {
  return guarded(c, [&] {
    for (int i = 0; i < 8; ++i) out_ms[i] = c->t_ms[i];
  });
}
CBX_API cbx_status cbx_skin_stats(cbx_ctx* c, int enable, uint64_t out[2]) {
  return guarded(c, [&] {
    cudaSetDevice(c->device);
    unsigned long long h[3];
    cuda_check(cudaMemcpyAsync(h, c->P.skin_cnt, sizeof h, cudaMemcpyDeviceToHost, c->stream),
               "skin stats");
    cuda_check(cudaStreamSynchronize(c->stream), "skin stats");
    out[0] = h[0];
    out[1] = h[1];
    const unsigned long long z[3] = {0ull, 0ull, enable ? 1ull : 0ull};
    if (enable) cudaMemcpyAsync(c->P.skin_cnt, z, sizeof z, cudaMemcpyHostToDevice, c->stream);
    else cudaMemcpyAsync(c->P.skin_cnt + 2, z + 2, sizeof z[2], cudaMemcpyHostToDevice, c->stream);
    cuda_check(cudaStreamSynchronize(c->stream), "skin stats");
  });
}

CBX_API cbx_status cbx_count_pairs(cbx_ctx* c, uint64_t out[2]) {
  return guarded(c, [&] {
    cudaSetDevice(c->device);
    sync_status(c);
    c->hst.cnt_cand = 0;
    c->hst.cnt_pair = 0;
    write_status(c);
    // one counting pass of the reference-literal half-list kernel (same
    // candidate / in-cutoff pair sets as every stencil), then a clean density
    KP saved = c->P;
    c->P.count_pairs = 1;
    cudaMemsetAsync(c->P.rho, 0, c->S * sizeof(double), c->stream);
    launch_density(c->P, CBX_STENCIL_REFERENCE, c->stream);
    c->P = saved;
    sync_status(c);
    out[0] = c->hst.cnt_cand;
    out[1] = c->hst.cnt_pair;
    seq_density(c);
    sync_status(c);
    raise_device_error(c, false);
  });
}

// streams a buffer through L2 (the result lands in an unused work word)
__global__ void k_l2_read(const double4* __restrict__ b, size_t n, int* sink) {
  double acc = 0.0;
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n;
       i += (size_t)gridDim.x * blockDim.x) {
    const double4 v = b[i];
    acc += v.x + v.w;
  }
  if (acc == 1.2345e300) *sink = 1;  // keeps the loads
}

CBX_API cbx_status cbx_bench_steps(cbx_ctx* c, double dt, long nsteps, double flush_mb,
                                   double out_ms[8]) {
  return guarded(c, [&] {
    cudaSetDevice(c->device);
    check_cutoff(c);
    sync_status(c);
    require_box_or_comm(c, "cbx_bench_steps");
    c->hst.dt_next = dt;
    c->hst.adaptive = 0;
    write_status(c);
    const bool phases = c->bench_phases;
    if ((c->timed_graph || c->timed_lite) &&
        (c->t_defer != want_defer(c) || c->t_merge != want_merge(c)))
      drop_graph(c);
    cudaGraphExec_t* gp = phases ? &c->timed_graph : &c->timed_lite;
    if (!*gp) {
      c->timing_lite = !phases;
      *gp = capture_step(c, true);
      c->timing_lite = false;
      c->t_defer = c->graph_defer;
      c->t_merge = c->graph_merge;
      c->t_launches = c->graph_launches;
    }
    if (!c->ev_outer[0])
      for (auto& e : c->ev_outer) cuda_check(cudaEventCreate(&e), "event");
    const size_t fb = (size_t)(flush_mb * 1048576.0);
    if (fb > c->flush_bytes) {
      if (c->flush_buf) cudaFree(c->flush_buf);
      cuda_check(cudaMalloc(&c->flush_buf, fb), "flush buffer");
      c->flush_bytes = fb;
    }
    double acc[8] = {0};
    for (long i = 0; i < nsteps; ++i) {
      if (fb) {  // evict L2: write a buffer larger than L2, then read it back so the
                 // step starts on clean lines (no write-back of the flush data in it)
        cudaMemsetAsync(c->flush_buf, (int)(i & 0xff), fb, c->stream);
        k_l2_read<<<4 * 148, 512, 0, c->stream>>>(static_cast<const double4*>(c->flush_buf),
                                                  fb / sizeof(double4), c->P.work + 3);
      }
      // the step: events on the stream around the graph launch
      cudaEventRecord(c->ev_outer[0], c->stream);
      cuda_check(cudaGraphLaunch(*gp, c->stream), "graph launch");
      cudaEventRecord(c->ev_outer[1], c->stream);
      c->launches += c->t_launches;
      if (c->t_merge) c->k2_maybe = true;
      else if (c->t_defer) c->fin_maybe = true;
      cuda_check(cudaEventSynchronize(c->ev_outer[1]), "event sync");
      float ms;
      cudaEventElapsedTime(&ms, c->ev_outer[0], c->ev_outer[1]);
      acc[5] += ms;
      cudaEventElapsedTime(&ms, c->ev[6], c->ev[7]);
      acc[7] += ms;
      if (phases) {
        const int seg[5][2] = {{1, 2}, {2, 3}, {3, 4}, {0, 1}, {4, 5}};
        for (int k = 0; k < 5; ++k) {
          cudaEventElapsedTime(&ms, c->ev[seg[k][0]], c->ev[seg[k][1]]);
          acc[k] += ms;
        }
      }
    }
    acc[6] = (double)nsteps;
    sync_status(c);
    raise_device_error(c, true);
    for (int k = 0; k < 8; ++k) out_ms[k] = acc[k];
  });
}

CBX_API cbx_status cbx_bench_phases(cbx_ctx* c, int on) {
  return guarded(c, [&] { c->bench_phases = on != 0; });
}

CBX_API cbx_status cbx_describe(cbx_ctx* c, char* buf, long n) {
  return guarded(c, [&] {
    std::snprintf(buf, n,
                  "{\"stencil\": %d, \"fast_ok\": %d, \"fp32_density\": %d, "
                  "\"force_table\": %d, "
                  "\"pair_mask\": %d, \"slots\": %lld, \"ghost_sites\": %d, "
                  "\"clash_capacity\": %d, \"band_A2\": %.3e, \"skin_prune\": %d, "
                  "\"kick_drift_bulk\": %d, \"force_window\": [%d, %d, %d, %d], "
                  "\"unit_rr\": %d, \"sm_count\": %d}",
                  c->mode, (int)c->fast_ok, (int)c->fp32_density, force_table_mode(),
                  (int)(c->P.pmask != nullptr), c->S, c->n_ghost, c->P.cap_clash, c->band,
                  (int)(c->P.ub != nullptr), (int)kd_bulk(c->P), c->P.fw_lo,
                  c->P.fw_gap_n ? c->P.fw_gap_lo : -1, c->P.fw_gap_n, c->P.fw_cap, c->P.unit_rr,
                  [] {
                    int d = 0, n = 0;
                    cudaGetDevice(&d);
                    cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, d);
                    return n;
                  }());
  });
}

CBX_API cbx_status cbx_memory_report(cbx_ctx* c, long long out[CBX_MEM_CATEGORIES + 4]) {
  return guarded(c, [&] {
    for (int k = 0; k < CBX_MEM_CATEGORIES; ++k) out[k] = (long long)c->mem_bytes[k];
    out[CBX_MEM_CATEGORIES] = c->S;                       // slots (ghost-inclusive)
    out[CBX_MEM_CATEGORIES + 1] = c->P.cap_clash;         // clash capacity (records)
    out[CBX_MEM_CATEGORIES + 2] = c->n_ghost;             // ghost links
    out[CBX_MEM_CATEGORIES + 3] = (long long)(           // offset lists (__constant__)
        sizeof(int) * (c->c_fd[0].size() + c->c_fd[1].size() + c->c_hd[0].size() +
                       c->c_hd[1].size()));
  });
}

CBX_API cbx_status cbx_kernel_launches(cbx_ctx* c, uint64_t* n) {
  *n = c->launches;
  return CBX_OK;
}

// ===========================================================================
// z-slab decomposition (multi-GPU), driven phase by phase by the host
// (paper_2107_07866_b200/slab.py) with the exchanges in between.

CBX_API cbx_status cbx_create_slab(const cbx_box* global_box, const cbx_potential* pot,
                                   const cbx_offsets* idx, int rank, int nranks, int device,
                                   cbx_ctx** out) {
  if (nranks < 1 || rank < 0 || rank >= nranks) {
    set_thread_error("cbx_create_slab: bad rank / nranks");
    return CBX_INVALID_ARGUMENT;
  }
  const long gbz = global_box->box_z;
  const long z0 = rank * gbz / nranks, z1 = (rank + 1) * gbz / nranks;
  cbx_box local = *global_box;
  local.box_z = z1 - z0;
  SlabSpec sp;
  sp.rank = rank;
  sp.nranks = nranks;
  sp.zoff = (int)z0;
  sp.gbz = (int)gbz;
  return create_impl(&local, pot, idx, device, &sp, out);
}

CBX_API cbx_status cbx_slab_info(cbx_ctx* c, long out[8]) {
  return guarded(c, [&] {
    out[0] = c->rank;
    out[1] = c->nranks;
    out[2] = c->G.zoff;
    out[3] = c->G.bz;
    out[4] = c->G.g;
    out[5] = c->G.tx;
    out[6] = c->G.ty;
    out[7] = c->G.gbz;
  });
}

CBX_API long cbx_slab_buffer_bytes(cbx_ctx* c, int kind) {
  return (long)slab_buffer_bytes(c->P, kind);
}

// phases: 0 begin step (kick, drift, wrap, hash, outbound migrants),
// 1 rehash + x/y ghosts, 2 clash images + density, 3 embedding,
// 4 force, 5 end step (second kick, local sums), 6 local energy sums only
// Lockstep driving of the peer-memory transport: the host runs the step's
// phases (cbx_slab_phase) and each exchange as a send (pack into the
// neighbours' mapped buffers, raise their flags, wait for completion) and a
// receive (flags already raised: unpack), with a barrier of all ranks in
// between -- so no kernel ever waits on another rank's kernel, which is what
// ranks sharing one GPU need (several processes on one device).  Reverse
// halos go as staged exchanges (no fused peer atomics in this mode).
CBX_API cbx_status cbx_slab_p2p_send(cbx_ctx* c, int kind) {
  return guarded(c, [&] {
    cudaSetDevice(c->device);
    if (!c->p2p) raise(CBX_LOGIC, "cbx_slab_p2p_send: no peer-memory transport");
    if (kind < 0 || kind > 4) raise(CBX_INVALID_ARGUMENT, "cbx_slab_p2p_send: unknown kind");
    if (c->P.rev.on) raise(CBX_LOGIC, "cbx_slab_p2p_send: reverse halos are fused");
    if (kind == 1) {  // the receive's remote-record count starts from zero
      sync_status(c);
      c->hst.n_remote = 0;
      write_status(c);
    }
    launch_p2p_send(c->P, c->links, kind, c->stream);
    c->launches += 1;
    sync_status(c);
    raise_device_error(c, false);
  });
}
CBX_API cbx_status cbx_slab_p2p_recv(cbx_ctx* c, int kind) {
  return guarded(c, [&] {
    cudaSetDevice(c->device);
    if (!c->p2p) raise(CBX_LOGIC, "cbx_slab_p2p_recv: no peer-memory transport");
    if (kind < 0 || kind > 4) raise(CBX_INVALID_ARGUMENT, "cbx_slab_p2p_recv: unknown kind");
    const long long gs_lo = (kind == 1 && c->rank == 0) ? -1 : 0;
    const long long gs_hi = (kind == 1 && c->rank == c->nranks - 1) ? 1 : 0;
    launch_p2p_recv(c->P, c->links, kind, gs_lo, gs_hi, c->d_rem_base, c->stream);
    c->launches += 1;
    sync_status(c);
    raise_device_error(c, false);
  });
}

CBX_API cbx_status cbx_slab_phase(cbx_ctx* c, int phase, double dt) {
  return guarded(c, [&] {
    cudaSetDevice(c->device);
    if (c->p2p && c->P.rev.on)
      raise(CBX_LOGIC, "cbx_slab_phase: this rank's reverse halos are fused into the passes");
    check_cutoff(c);
    switch (phase) {
      case 0:
        sync_status(c);
        if (dt > 0.0) {
          c->hst.dt_next = dt;
          c->hst.adaptive = 0;
        } else {
          c->hst.adaptive = 1;
          c->hst.dt_next = cbx_adaptive_dt(c->hst.max_speed, c->hst.dt_max, c->hst.max_disp);
        }
        c->hst.n_out = 0;
        write_status(c);
        c->mask_valid = false;
        launch_kick_drift(c->P, 1, c->stream);
        c->launches += 1;
        break;
      case 1:
        launch_rehash(c->P, c->stream);
        launch_ghost_fill(c->P, c->stream);
        c->launches += 2;
        sync_status(c);
        c->hst.n_remote = 0;
        write_status(c);
        break;
      case 2:
        launch_clash_images(c->P, c->stream, 1);
        c->clash_rho_zero = true;
        c->launches += 1;
        seq_density(c);
        break;
      case 3:
        seq_embed(c);
        break;
      case 4:
        launch_remote_df(c->P, c->stream);
        c->launches += 1;
        seq_force(c);
        break;
      case 5:
        launch_kick2(c->P, 1, 1, 1, c->stream);
        c->launches += 1;
        break;
      case 6:
        launch_finalize(c->P, -1, 1, c->stream);
        c->launches += 1;
        break;
      case 7:  // measure only (kinetic energy, max speed)
        launch_kick2(c->P, 0, 0, 0, c->stream);
        c->launches += 1;
        break;
      default:
        raise(CBX_INVALID_ARGUMENT, "cbx_slab_phase: unknown phase");
    }
    sync_status(c);
    raise_device_error(c, phase >= 2 && phase <= 5);
  });
}

// dir -1: toward the rank below, +1: toward the rank above
CBX_API cbx_status cbx_slab_pack(cbx_ctx* c, int kind, int dir, void* buf, long cap,
                                 long* bytes) {
  return guarded(c, [&] {
    cudaSetDevice(c->device);
    if (kind < 0 || kind > 4 || (dir != -1 && dir != 1))
      raise(CBX_INVALID_ARGUMENT, "cbx_slab_pack: bad kind / direction");
    launch_pack(c->P, kind, dir, static_cast<unsigned char*>(buf), cap, c->stream);
    const long long pb = kind == 0 ? 0 : slab_buffer_bytes(c->P, kind) -
                                             ((kind == 1 || kind == 3)
                                                  ? 16 + (long long)c->P.cap_rem * 72
                                                  : 0);
    long long n = 0;
    long long used = 0;
    if (kind == 0 || kind == 1 || kind == 3) {
      // record count sits at the start of the record section
      const long long plane = kind == 0 ? 0 : 2ll * c->G.g * c->G.txy * (kind == 1 ? 40 : 8);
      cuda_check(cudaMemcpyAsync(&n, static_cast<unsigned char*>(buf) + plane, 8,
                                 cudaMemcpyDeviceToHost, c->stream),
                 "pack count");
      cuda_check(cudaStreamSynchronize(c->stream), "pack");
      used = plane + 16 + n * (kind == 0 ? 88 : 72);
    } else {
      used = 2ll * c->G.g * c->G.txy * (kind == 2 ? 8 : 24);
      cuda_check(cudaStreamSynchronize(c->stream), "pack");
    }
    (void)pb;
    sync_status(c);
    raise_device_error(c, false);
    *bytes = (long)used;
  });
}

// from -1: data sent by the rank below, +1: by the rank above
CBX_API cbx_status cbx_slab_unpack(cbx_ctx* c, int kind, int from, const void* buf, long bytes) {
  return guarded(c, [&] {
    cudaSetDevice(c->device);
    if (kind < 0 || kind > 4 || (from != -1 && from != 1))
      raise(CBX_INVALID_ARGUMENT, "cbx_slab_unpack: bad kind / direction");
    (void)bytes;
    // position halos crossing the global z boundary are periodic images
    long long gshift = 0;
    if (kind == 1 && from < 0 && c->rank == 0) gshift = -1;
    if (kind == 1 && from > 0 && c->rank == c->nranks - 1) gshift = 1;
    launch_unpack(c->P, kind, from, static_cast<const unsigned char*>(buf), gshift,
                  c->d_rem_base + (from < 0 ? 0 : 1), c->stream);
    sync_status(c);
    raise_device_error(c, false);
  });
}

CBX_API cbx_status cbx_slab_local_state(cbx_ctx* c, double out[8]) {
  return guarded(c, [&] {
    cudaSetDevice(c->device);
    sync_status(c);
    out[0] = c->hst.kinetic;
    out[1] = c->hst.pair;
    out[2] = c->hst.embedding;
    out[3] = c->hst.max_speed;
    out[4] = (double)c->hst.r_underflow;
    out[5] = (double)c->hst.rho_clamp;
    out[6] = (double)c->hst.step;
    out[7] = c->hst.t;
  });
}

// the all-reduced sums / max become this rank's StepState
CBX_API cbx_status cbx_slab_commit(cbx_ctx* c, const double in[4]) {
  return guarded(c, [&] {
    cudaSetDevice(c->device);
    sync_status(c);
    c->hst.kinetic = in[0];
    c->hst.pair = in[1];
    c->hst.embedding = in[2];
    c->hst.max_speed = in[3];
    if (c->hst.adaptive)
      c->hst.dt_next = cbx_adaptive_dt(in[3], c->hst.dt_max, c->hst.max_disp);
    write_status(c);
  });
}

CBX_API cbx_status cbx_nccl_unique_id(void* out, long nbytes) {
  return guarded(nullptr, [&] {
    if (nbytes < (long)sizeof(ncclUniqueId))
      raise(CBX_INVALID_ARGUMENT, "cbx_nccl_unique_id: buffer smaller than 128 bytes");
    ncclUniqueId id;
    nccl_check(nccl().get_unique_id(&id), "ncclGetUniqueId");
    std::memcpy(out, &id, sizeof id);
  });
}

// collective over the slab ranks: every rank passes the same id
CBX_API cbx_status cbx_slab_comm_init(cbx_ctx* c, const void* id, long nbytes) {
  return guarded(c, [&] {
    cudaSetDevice(c->device);
    if (!c->G.slab) raise(CBX_LOGIC, "cbx_slab_comm_init: not a slab rank");
    if (c->comm) raise(CBX_LOGIC, "cbx_slab_comm_init: communicator already set");
    if (nbytes < (long)sizeof(ncclUniqueId))
      raise(CBX_INVALID_ARGUMENT, "cbx_slab_comm_init: id smaller than 128 bytes");
    ncclUniqueId u;
    std::memcpy(&u, id, sizeof u);
    long long mx = 0;
    for (int k = 0; k < 5; ++k) mx = std::max(mx, slab_msg_bytes(c->P, k));
    c->mem_cat = CBX_MEM_EXCHANGE;
    for (int i = 0; i < 2; ++i) {
      c->sbuf[i] = c->alloc<unsigned char>(mx);
      c->rbuf[i] = c->alloc<unsigned char>(mx);
      cudaMemset(c->rbuf[i], 0, mx);
    }
    c->d_red = c->alloc<double>(8);
    ncclComm_t comm = nullptr;
    nccl_check(nccl().comm_init_rank(&comm, c->nranks, u, c->rank), "ncclCommInitRank");
    c->comm = comm;
    drop_graph(c);
  });
}

// ---- P2P transport: receive regions exchanged as CUDA IPC handles --------
// region layout (identical on every rank: message sizes depend only on the
// shared x/y extent and ghost width): flags [5][2] u64 @0, reduction flags
// [8] u64 @256, reduction slots [8][4] f64 @512, receive buffers from @1024
namespace {
constexpr size_t kFlagOff = 0, kRedFlagOff = 256, kRedOff = 512, kBufOff = 1024;
size_t p2p_buf_off(const KP& P, int kind, int from) {
  size_t o = kBufOff;
  for (int k = 0; k < 5; ++k)
    for (int f = 0; f < 2; ++f) {
      if (k == kind && f == from) return o;
      o += (size_t)slab_msg_bytes(P, k);
    }
  return o;
}
}  // namespace

CBX_API cbx_status cbx_slab_p2p_handle(cbx_ctx* c, void* out, long nbytes) {
  return guarded(c, [&] {
    cudaSetDevice(c->device);
    if (!c->G.slab) raise(CBX_LOGIC, "cbx_slab_p2p_handle: not a slab rank");
    if (nbytes < CBX_P2P_HANDLE_BYTES)
      raise(CBX_INVALID_ARGUMENT, "cbx_slab_p2p_handle: buffer smaller than CBX_P2P_HANDLE_BYTES");
    if (!c->p2p_region) {
      c->p2p_bytes = p2p_buf_off(c->P, 5, 0);
      cuda_check(cudaMalloc(&c->p2p_region, c->p2p_bytes), "p2p region");
      c->mem_bytes[CBX_MEM_EXCHANGE] += c->p2p_bytes;
      cuda_check(cudaMemset(c->p2p_region, 0, c->p2p_bytes), "p2p region");
    }
    // [receive region][rho][force] IPC handles, then NC, S, bz of this rank
    unsigned char* o = static_cast<unsigned char*>(out);
    std::memset(o, 0, CBX_P2P_HANDLE_BYTES);
    const void* bases[3] = {c->p2p_region, c->P.rho, c->P.frc};
    for (int k = 0; k < 3; ++k) {
      cudaIpcMemHandle_t h;
      cuda_check(cudaIpcGetMemHandle(&h, const_cast<void*>(bases[k])), "cudaIpcGetMemHandle");
      std::memcpy(o + 64 * k, &h, sizeof h);
    }
    // PCI bus id of this rank's GPU: the neighbours check native peer atomics
    int bus = 0, dev_id = 0, dom = 0;
    cudaDeviceGetAttribute(&bus, cudaDevAttrPciBusId, c->device);
    cudaDeviceGetAttribute(&dev_id, cudaDevAttrPciDeviceId, c->device);
    cudaDeviceGetAttribute(&dom, cudaDevAttrPciDomainId, c->device);
    const long long geo[4] = {c->G.NC, c->S, (long long)c->G.bz,
                              ((long long)dom << 32) | ((long long)bus << 16) | dev_id};
    std::memcpy(o + 192, geo, sizeof geo);
  });
}

// collective in the sense that every rank must call it before any step;
// handles[q] is rank q's cbx_slab_p2p_handle
CBX_API cbx_status cbx_slab_p2p_init(cbx_ctx* c, const void* handles, long nbytes) {
  return guarded(c, [&] {
    cudaSetDevice(c->device);
    if (!c->p2p_region) raise(CBX_LOGIC, "cbx_slab_p2p_init: call cbx_slab_p2p_handle first");
    if (c->p2p) raise(CBX_LOGIC, "cbx_slab_p2p_init: already initialised");
    const int n = c->nranks;
    if (n > kMaxP2PRanks) raise(CBX_INVALID_ARGUMENT, "cbx_slab_p2p_init: more than 8 ranks");
    if (nbytes < (long)n * CBX_P2P_HANDLE_BYTES)
      raise(CBX_INVALID_ARGUMENT,
            "cbx_slab_p2p_init: need one CBX_P2P_HANDLE_BYTES handle per rank");
    const unsigned char* hb = static_cast<const unsigned char*>(handles);
    auto open = [&](int q, int k) -> void* {  // rank q's k-th exported allocation
      if (q == c->rank) return k == 0 ? (void*)c->p2p_region : k == 1 ? (void*)c->P.rho
                                                                      : (void*)c->P.frc;
      cudaIpcMemHandle_t h;
      std::memcpy(&h, hb + (size_t)q * CBX_P2P_HANDLE_BYTES + 64 * k, sizeof h);
      void* p = nullptr;
      cuda_check(cudaIpcOpenMemHandle(&p, h, cudaIpcMemLazyEnablePeerAccess),
                 "cudaIpcOpenMemHandle (ranks must share a node with peer access)");
      c->p2p_opened.push_back(p);
      return p;
    };
    std::vector<unsigned char*> base(n);
    for (int q = 0; q < n; ++q) base[q] = static_cast<unsigned char*>(open(q, 0));
    P2PLinks& L = c->links;
    L = P2PLinks{};
    const int lo = (c->rank + n - 1) % n, hi = (c->rank + 1) % n;
    // fused reverse halo: the neighbours' accumulators (KP::rev)
    {
      RevHalo& R = c->P.rev;
      R = RevHalo{};
      const Geo& G = c->G;
      long long plane0[2] = {0, 0};
      const int nb[2] = {lo, hi};
      void* rho_nb[2] = {nullptr, nullptr};
      void* frc_nb[2] = {nullptr, nullptr};
      // the fused reverse halo adds into the neighbours' memory with fp64
      // atomics: only where the links support them natively (NVLink).  Every
      // rank checks every pair, so all ranks take the same path.
      bool atomics = true;
      std::vector<int> devs(n, -1);
      int ndev = 0;
      cudaGetDeviceCount(&ndev);
      for (int q = 0; q < n; ++q) {
        long long pci = 0;
        std::memcpy(&pci, hb + (size_t)q * CBX_P2P_HANDLE_BYTES + 216, sizeof pci);
        for (int d = 0; d < ndev && devs[q] < 0; ++d) {
          int b = 0, i = 0, m = 0;
          cudaDeviceGetAttribute(&b, cudaDevAttrPciBusId, d);
          cudaDeviceGetAttribute(&i, cudaDevAttrPciDeviceId, d);
          cudaDeviceGetAttribute(&m, cudaDevAttrPciDomainId, d);
          if ((((long long)m << 32) | ((long long)b << 16) | i) == pci) devs[q] = d;
        }
        if (devs[q] < 0) atomics = false;
      }
      for (int a = 0; a < n && atomics; ++a)
        for (int b = 0; b < n && atomics; ++b) {
          if (a == b) continue;
          int v = 0;
          if (devs[a] == devs[b] ||
              cudaDeviceGetP2PAttribute(&v, cudaDevP2PAttrNativeAtomicSupported, devs[a],
                                        devs[b]) != cudaSuccess || !v)
            atomics = false;
        }
      cudaGetLastError();
      for (int side = 0; side < 2 && atomics; ++side) {
        const int q = nb[side];
        if (side == 1 && hi == lo) {  // two ranks: one neighbour on both sides
          rho_nb[1] = rho_nb[0];
          frc_nb[1] = frc_nb[0];
        } else {
          rho_nb[side] = open(q, 1);
          frc_nb[side] = open(q, 2);
        }
        long long geo[3];
        std::memcpy(geo, hb + (size_t)q * CBX_P2P_HANDLE_BYTES + 192, sizeof geo);
        R.rho[side] = static_cast<double*>(rho_nb[side]);
        R.frc[side] = static_cast<double*>(frc_nb[side]);
        R.NC[side] = geo[0];
        R.S[side] = geo[1];
        // my lower halo lands on the top boundary planes of the rank below,
        // my upper halo on the bottom boundary planes of the rank above
        plane0[side] = side == 0 ? geo[2] : G.g;
      }
      R.lo = (long long)G.g * G.txy;
      R.hi = (long long)(G.g + G.bz) * G.txy;
      R.delta[0] = plane0[0] * G.txy;  // c in [0, g txy) -> the planes [bz_lo, bz_lo + g)
      R.delta[1] = (long long)G.g * G.txy - R.hi;  // [hi, hi + g txy) -> [g, 2 g)
      c->rev_mapped = atomics;
    }
    auto flag = [&](unsigned char* b, int kind, int from) {
      return reinterpret_cast<unsigned long long*>(b + kFlagOff) + 2 * kind + from;
    };
    for (int k = 0; k < 5; ++k) {
      L.msg[k] = slab_msg_bytes(c->P, k);
      L.plane_bytes[k] = k == 0 ? 0 : slab_plane_bytes(c->P, k);
      L.dst[k][0] = base[lo] + p2p_buf_off(c->P, k, 1);  // arrives "from above" below me
      L.dst[k][1] = base[hi] + p2p_buf_off(c->P, k, 0);  // arrives "from below" above me
      L.flag_dst[k][0] = flag(base[lo], k, 1);
      L.flag_dst[k][1] = flag(base[hi], k, 0);
      for (int f = 0; f < 2; ++f) {
        L.src[k][f] = c->p2p_region + p2p_buf_off(c->P, k, f);
        L.flag_src[k][f] = flag(c->p2p_region, k, f);
      }
    }
    for (int q = 0; q < n; ++q) {
      L.red_dst[q] = reinterpret_cast<double*>(base[q] + kRedOff);
      L.red_flag_dst[q] = reinterpret_cast<unsigned long long*>(base[q] + kRedFlagOff);
    }
    L.red_src = reinterpret_cast<const double*>(c->p2p_region + kRedOff);
    L.red_flag_src = reinterpret_cast<const unsigned long long*>(c->p2p_region + kRedFlagOff);
    c->mem_cat = CBX_MEM_EXCHANGE;
    L.epoch = c->alloc<unsigned long long>(6);
    L.done = c->alloc<unsigned>(6);
    cudaMemset(L.epoch, 0, 6 * sizeof(unsigned long long));
    cudaMemset(L.done, 0, 6 * sizeof(unsigned));
    L.rank = c->rank;
    L.nranks = n;
    c->d_links = c->alloc<P2PLinks>(1);
    cuda_check(cudaMemcpy(c->d_links, &L, sizeof L, cudaMemcpyHostToDevice), "p2p links");
    c->p2p = true;
    c->P.lk = c->d_links;
    c->P.rev.on = rev_fused(c);
    sync_kp(c);
    cuda_check(cudaDeviceSynchronize(), "p2p init");
    drop_graph(c);
  });
}

// the reverse halos fused into the passes (1) or staged exchanges (0); every
// rank must use the same: the Python connect() agrees on it and sets it
CBX_API int cbx_slab_p2p_fused(cbx_ctx* c) { return c->P.rev.on ? 1 : 0; }
// back to no device transport (a rank whose peers could not all map peer
// memory; the caller then connects NCCL)
CBX_API cbx_status cbx_slab_p2p_close(cbx_ctx* c) {
  return guarded(c, [&] {
    c->p2p = false;
    c->P.rev.on = 0;
    sync_kp(c);
    drop_graph(c);
  });
}
CBX_API cbx_status cbx_slab_p2p_set_fused(cbx_ctx* c, int on) {
  return guarded(c, [&] {
    if (!c->p2p) raise(CBX_LOGIC, "cbx_slab_p2p_set_fused: no peer-memory transport");
    if (on && !c->rev_mapped)
      raise(CBX_INVALID_ARGUMENT, "cbx_slab_p2p_set_fused: no native peer atomics");
    c->fused_off = !on;
    c->P.rev.on = rev_fused(c);
    sync_kp(c);
    drop_graph(c);
  });
}

// global store <-> this slab (tests, setup)
CBX_API cbx_status cbx_upload_store_global(cbx_ctx* c, const cbx_store* g) {
  return guarded(c, [&] {
    cudaSetDevice(c->device);
    const Geo& G = c->G;
    const long long pid = 2ll * G.tx * G.ty, S = c->S, off = (long long)G.zoff * pid;
    std::vector<double> pos(3 * S, 0.0), vel(3 * S, 0.0), frc(3 * S, 0.0), rho(S, 0.0), df(S, 0.0);
    std::vector<uint64_t> tag(S, 0);
    std::vector<uint8_t> valid(S, 0);
    // local interior planes cz in [g, g + bz) <- global ids + off
    for (long long id = (long long)G.g * pid; id < (long long)(G.g + G.bz) * pid; ++id) {
      const long long gid = id + off;
      if (gid < 0 || gid >= g->n_slots) continue;
      valid[id] = g->valid ? g->valid[gid] && !(g->ghost && g->ghost[gid]) : 1;
      for (int a = 0; a < 3; ++a) {
        pos[3 * id + a] = g->pos[3 * gid + a];
        if (g->vel) vel[3 * id + a] = g->vel[3 * gid + a];
        if (g->force) frc[3 * id + a] = g->force[3 * gid + a];
      }
      if (g->rho) rho[id] = g->rho[gid];
      if (g->df) df[id] = g->df[gid];
      if (g->tag) tag[id] = g->tag[gid];
    }
    std::vector<int64_t> ck;
    std::vector<double> cp, cv, cf, cr, cd;
    std::vector<uint64_t> ct;
    for (long i = 0; i < g->n_clash; ++i) {
      if (g->clash_ghost && g->clash_ghost[i]) continue;
      const long long k = g->clash_key[i] - off;
      const long cz = site_cz(k, G);
      if (cz < G.g || cz >= G.g + G.bz) continue;
      ck.push_back(k);
      for (int a = 0; a < 3; ++a) {
        cp.push_back(g->clash_pos[3 * i + a]);
        cv.push_back(g->clash_vel ? g->clash_vel[3 * i + a] : 0.0);
        cf.push_back(g->clash_force ? g->clash_force[3 * i + a] : 0.0);
      }
      cr.push_back(g->clash_rho ? g->clash_rho[i] : 0.0);
      cd.push_back(g->clash_df ? g->clash_df[i] : 0.0);
      ct.push_back(g->clash_tag ? g->clash_tag[i] : 0);
    }
    cbx_store l{};
    l.n_slots = S;
    l.pos = pos.data();
    l.vel = vel.data();
    l.force = frc.data();
    l.rho = rho.data();
    l.df = df.data();
    l.tag = tag.data();
    l.valid = valid.data();
    l.n_clash = (long)ck.size();
    l.clash_key = ck.data();
    l.clash_pos = cp.data();
    l.clash_vel = cv.data();
    l.clash_force = cf.data();
    l.clash_rho = cr.data();
    l.clash_df = cd.data();
    l.clash_tag = ct.data();
    do_upload(c, &l);
  });
}

// writes this slab's interior sites into the global arrays (by global id)
// and appends its interior clash records (global keys) at g->clash_* from
// index *n_clash_inout
CBX_API cbx_status cbx_download_store_global(cbx_ctx* c, cbx_store* g, long* n_clash_inout) {
  return guarded(c, [&] {
    cudaSetDevice(c->device);
    const Geo& G = c->G;
    const long long pid = 2ll * G.tx * G.ty, S = c->S, off = (long long)G.zoff * pid;
    std::vector<double> pos(3 * S), vel(3 * S), frc(3 * S), rho(S), df(S);
    std::vector<uint64_t> tag(S);
    std::vector<uint8_t> valid(S), ghost(S);
    cbx_store l{};
    l.n_slots = S;
    l.pos = pos.data();
    l.vel = vel.data();
    l.force = frc.data();
    l.rho = rho.data();
    l.df = df.data();
    l.tag = tag.data();
    l.valid = valid.data();
    l.ghost = ghost.data();
    do_download(c, &l);  // counts only (clash_key null)
    const long nc = l.n_clash;
    std::vector<int64_t> ck(nc);
    std::vector<int32_t> ci(nc);
    std::vector<double> cp(3 * nc), cv(3 * nc), cf(3 * nc), cr(nc), cd(nc);
    std::vector<uint64_t> ct(nc);
    std::vector<uint8_t> cg(nc);
    l.clash_key = ck.data();
    l.clash_idx = ci.data();
    l.clash_pos = cp.data();
    l.clash_vel = cv.data();
    l.clash_force = cf.data();
    l.clash_rho = cr.data();
    l.clash_df = cd.data();
    l.clash_tag = ct.data();
    l.clash_ghost = cg.data();
    do_download(c, &l);
    for (long long id = (long long)G.g * pid; id < (long long)(G.g + G.bz) * pid; ++id) {
      const long long gid = id + off;
      if (gid < 0 || gid >= g->n_slots) continue;
      if (g->valid) g->valid[gid] = valid[id];
      if (g->ghost) g->ghost[gid] = ghost[id];
      for (int a = 0; a < 3; ++a) {
        if (g->pos) g->pos[3 * gid + a] = pos[3 * id + a];
        if (g->vel) g->vel[3 * gid + a] = vel[3 * id + a];
        if (g->force) g->force[3 * gid + a] = frc[3 * id + a];
      }
      if (g->rho) g->rho[gid] = rho[id];
      if (g->df) g->df[gid] = df[id];
      if (g->tag) g->tag[gid] = tag[id];
    }
    long k = *n_clash_inout;
    for (long i = 0; i < nc; ++i) {
      if (cg[i]) continue;
      if (k >= g->n_clash) raise(CBX_INVALID_ARGUMENT, "download_store_global: clash capacity");
      if (g->clash_key) g->clash_key[k] = ck[i] + off;
      if (g->clash_idx) g->clash_idx[k] = ci[i];
      for (int a = 0; a < 3; ++a) {
        if (g->clash_pos) g->clash_pos[3 * k + a] = cp[3 * i + a];
        if (g->clash_vel) g->clash_vel[3 * k + a] = cv[3 * i + a];
        if (g->clash_force) g->clash_force[3 * k + a] = cf[3 * i + a];
      }
      if (g->clash_rho) g->clash_rho[k] = cr[i];
      if (g->clash_df) g->clash_df[k] = cd[i];
      if (g->clash_tag) g->clash_tag[k] = ct[i];
      if (g->clash_ghost) g->clash_ghost[k] = 0;
      ++k;
    }
    *n_clash_inout = k;
  });
}

}  // extern "C"
