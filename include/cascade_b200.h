/*
 * cascade_b200.h -- C ABI of the B200-native EAM hot path (libcascade_b200.so).
 *
 * The drop-in boundary for the reference's force engine and step loop
 * (cascademd, /root/reference/proj).  Plain pointers and sizes only; no
 * torch or CUDA types.  Each entry point names the reference interface it
 * replaces (paths relative to /root/reference/proj/core).
 *
 * Model: a context owns device-resident state (slot arrays over the
 * ghost-inclusive lattice, the clash list, potential tables, offsets).  Host
 * buffers are borrowed per call.  A context is not thread-safe (the
 * reference's WorkerPool is not reentrant either, src/parallel.cpp:26-59).
 * Errors: every call returns a cbx_status; the message (same text as the
 * reference's exception) is read with cbx_last_error().  The C++ header
 * cascade_b200.hpp rethrows them as the reference's exception types.
 */
#ifndef CASCADE_B200_H
#define CASCADE_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define CBX_API __attribute__((visibility("default")))
#define CBX_ABI_VERSION 1

typedef struct cbx_ctx cbx_ctx;

/* status codes, mirroring the reference's exception classes */
typedef enum {
  CBX_OK = 0,
  CBX_INVALID_ARGUMENT = 1, /* std::invalid_argument */
  CBX_RUNTIME = 2,          /* std::runtime_error: overlap, parse, capacity */
  CBX_DOMAIN = 3,           /* std::domain_error: hash outside the box */
  CBX_LOGIC = 4,            /* std::logic_error: wrap did not converge */
  CBX_CUDA = 5,             /* device / driver failure */
  CBX_NCCL = 6              /* collective failure (multi-GPU) */
} cbx_status;

/* BoxSpec, include/cascademd/lattice.h:21-42 */
typedef struct {
  long box_x, box_y, box_z;
  double a0;
  long ghost_width;
} cbx_box;

/* SplineTable, include/cascademd/spline.h:16-27: nseg segments of 7 doubles
 * {a,b,c,d,e,f,g} -- byte-compatible with std::vector<SplineTable::Seg> */
typedef struct {
  double x0, h;
  long nseg;
  const double* seg;
} cbx_spline;

/* EamPotential, include/cascademd/potential.h:33-60 */
typedef struct {
  int atomic_number;
  double mass, lattice_const, cutoff;
  cbx_spline embed, zr, dens;
} cbx_potential;

/* OffsetIndex, include/cascademd/neighbors.h:17-29 (flat signed site-id
 * offsets, ascending).  The library rebuilds the lists from (box, cutoff)
 * with the reference algorithm (src/neighbors.cpp:11-87) and rejects a
 * caller index that differs. */
typedef struct {
  double cutoff;
  long z_reach;
  const int64_t *even_full, *odd_full, *even_half, *odd_half;
  long n_even_full, n_odd_full, n_even_half, n_odd_half;
} cbx_offsets;

/* a LatticeStore view (include/cascademd/store.h:16-78): slot arrays by
 * site id (n_slots = BoxSpec::slot_count()), xyz interleaved like Vec3; the
 * clash map flattened in (key, bucket index) order.  NULL fields are skipped
 * (upload: zero) . */
typedef struct {
  long n_slots;
  double *pos, *vel, *force; /* [3*n_slots] */
  double *rho, *df;          /* [n_slots] */
  uint64_t* tag;
  uint8_t *valid, *ghost;
  long n_clash; /* upload: records given; download: capacity in, records out */
  int64_t* clash_key;
  int32_t* clash_idx;
  double *clash_pos, *clash_vel, *clash_force, *clash_rho, *clash_df;
  uint64_t* clash_tag;
  uint8_t* clash_ghost;
} cbx_store;

/* StepState, include/cascademd/sim.h:11-21 */
typedef struct {
  long step;
  double t, dt, kinetic, pair, embedding, max_speed;
  uint64_t r_underflow, rho_clamp;
} cbx_state;

/* kernel selection for the two EAM stencil passes */
typedef enum {
  CBX_STENCIL_NEWTON3 = 0, /* half list, ordered reduction into owners (default) */
  CBX_STENCIL_FULL = 1,     /* full list, owner computes (no atomics, deterministic) */
  CBX_STENCIL_REFERENCE = 2 /* half list with the reference's literal arithmetic (checker) */
} cbx_stencil;

/* ---- version / build ---------------------------------------------------- */
CBX_API int cbx_abi_version(void);
CBX_API const char* cbx_build_info(void);
CBX_API const char* cbx_last_error(const cbx_ctx* ctx); /* ctx may be NULL */

/* ---- host-side setup (no GPU needed) ------------------------------------- */
/* parse_potential_file, src/potential.cpp:134-185 (+ build_spline,
 * src/spline.cpp:14-77).  Returns an owned potential; free with
 * cbx_potential_free. */
CBX_API cbx_status cbx_potential_load(const char* path, cbx_potential** out);
CBX_API void cbx_potential_free(cbx_potential* pot);
/* build_offsets, src/neighbors.cpp:11-87.  Owned; free with cbx_offsets_free. */
CBX_API cbx_status cbx_offsets_build(const cbx_box* box, double cutoff, cbx_offsets** out);
CBX_API void cbx_offsets_free(cbx_offsets* idx);
/* make_box + index cutoff, src/sim.cpp:62-84 */
CBX_API cbx_status cbx_make_box(long box_x, long box_y, long box_z, double a0_cfg,
                                long ghost_width_cfg, double max_disp,
                                const cbx_potential* pot, cbx_box* out, double* index_cutoff);
CBX_API double cbx_pka_speed(double energy_ev, double mass_amu); /* src/sim.cpp:88-92 */
/* synthetic::write_table, src/synthetic.cpp:49-98: the reference's own
 * single-element test table (the CLI's gen-potential).  Same bytes. */
CBX_API cbx_status cbx_write_synthetic_table(const char* path, long nrho, long nr);
CBX_API double cbx_adaptive_dt(double max_speed, double dt_max, double max_disp); /* 94-98 */

/* ---- context -------------------------------------------------------------- */
/* Simulation's owned members (include/cascademd/sim.h:82-90) moved to the
 * device.  idx may be NULL (built internally). */
CBX_API cbx_status cbx_create(const cbx_box* box, const cbx_potential* pot,
                              const cbx_offsets* idx, int device, cbx_ctx** out);
CBX_API void cbx_destroy(cbx_ctx* ctx);
CBX_API cbx_status cbx_set_stencil(cbx_ctx* ctx, cbx_stencil mode);
CBX_API long cbx_slot_count(const cbx_ctx* ctx);

/* ---- store transfer ------------------------------------------------------- */
/* upload a LatticeStore; ghost slots/records are regenerated on the device
 * exactly as LatticeStore::fill_ghosts (src/store.cpp:120-195) */
CBX_API cbx_status cbx_upload_store(cbx_ctx* ctx, const cbx_store* s);
CBX_API cbx_status cbx_download_store(cbx_ctx* ctx, cbx_store* s);
CBX_API long cbx_clash_count(cbx_ctx* ctx);
/* init_bcc (src/sim.cpp:100-130) on the host with the reference RNG, then
 * upload + fill_ghosts; returns the atom count in *n_atoms */
CBX_API cbx_status cbx_init_bcc(cbx_ctx* ctx, int species, double temperature, uint64_t seed,
                                long* n_atoms);

/* ---- LatticeStore operations on device state (src/store.cpp) -------------- */
CBX_API cbx_status cbx_rehash(cbx_ctx* ctx); /* canonicalize_positions + update_hash + fill_ghosts */
CBX_API cbx_status cbx_fill_ghosts(cbx_ctx* ctx);

/* ---- force engine (include/cascademd/forces.h:42-67) ---------------------- */
CBX_API cbx_status cbx_eval_forces(cbx_ctx* ctx, double* e_emb, double* e_pair); /* forces.cpp:414-447 */
CBX_API cbx_status cbx_compute_density(cbx_ctx* ctx);                            /* 368-379 */
CBX_API cbx_status cbx_compute_embedding_derivative(cbx_ctx* ctx, double* e_emb); /* 381-388 */
CBX_API cbx_status cbx_compute_pair_forces(cbx_ctx* ctx, double* e_pair);         /* 390-402 */
CBX_API cbx_status cbx_guards(cbx_ctx* ctx, uint64_t out[2]); /* GuardCounters, potential.h:13-28 */

/* ---- Simulation (include/cascademd/sim.h:38-91) --------------------------- */
/* velocity-Verlet steps with device-resident state (sim.cpp:248-273).
 * dt > 0: fixed; dt <= 0: adaptive_dt per step from the previous max speed
 * with (dt_max, max_disp) from cbx_set_adaptive.  One host sync per call. */
CBX_API cbx_status cbx_step(cbx_ctx* ctx, double dt, long nsteps, cbx_state* out);
CBX_API cbx_status cbx_set_adaptive(cbx_ctx* ctx, double dt_max, double max_disp);
CBX_API cbx_status cbx_refresh_forces(cbx_ctx* ctx); /* sim.cpp:223-235 */
CBX_API cbx_status cbx_measure(cbx_ctx* ctx);        /* sim.cpp:237-246 */
CBX_API cbx_status cbx_get_state(cbx_ctx* ctx, cbx_state* out);
CBX_API cbx_status cbx_set_state(cbx_ctx* ctx, const cbx_state* in);
/* inject_pka (sim.cpp:163-186): overwrite the velocity of the slot atom at
 * reference site id `site`, then measure */
CBX_API cbx_status cbx_inject_pka(cbx_ctx* ctx, int64_t site, const double v[3]);
CBX_API cbx_status cbx_count_defects(cbx_ctx* ctx, long out[3]); /* analysis.cpp:40-56 */

/* ---- instrumentation ------------------------------------------------------ */
/* per-launch device time (CUDA events on the context stream) of the last
 * eval/step: {density, embed, force, clash, store} ms; and candidate / pair
 * counters of the last density pass {candidates, pairs} */
CBX_API cbx_status cbx_last_timings(cbx_ctx* ctx, double out_ms[8]);
CBX_API cbx_status cbx_enable_timing(cbx_ctx* ctx, int on);
CBX_API cbx_status cbx_count_pairs(cbx_ctx* ctx, uint64_t out[2]);
CBX_API cbx_status cbx_kernel_launches(cbx_ctx* ctx, uint64_t* n); /* cumulative */
/* skin-candidate counters of the density passes run while counting is on:
 * enable = 1 zeroes them and starts counting, 0 stops; out = {skin candidates
 * examined, skin candidates listed} (the regional displacement bound prunes
 * the difference; site slots of live lanes, vacant ones included) */
CBX_API cbx_status cbx_skin_stats(cbx_ctx* ctx, int enable, uint64_t out[2]);
/* JSON description of the context's kernel configuration */
/* Device bytes by structure (the CLI's bench-mem, tools/src/main.cpp:72-115):
 * out[k] for k < CBX_MEM_CATEGORIES, then slots, clash capacity, ghost
 * links and the offset-list bytes. */
enum {
  CBX_MEM_SLOTS = 0,     /* per-slot SoA: pos+dF, shadow, vel, force, rho, tag, owner, mask */
  CBX_MEM_CLASH = 1,     /* clash records (double-buffered) + the halo clash arena */
  CBX_MEM_GHOSTS = 2,    /* ghost-image links */
  CBX_MEM_REHASH = 3,    /* movers and sort scratch of update_hash */
  CBX_MEM_TABLES = 4,    /* spline segments (reference and fast layouts) */
  CBX_MEM_REDUCTION = 5, /* partial sums, status, counters */
  CBX_MEM_STAGING = 6,   /* reference-layout upload/download staging */
  CBX_MEM_EXCHANGE = 7,  /* slab exchange buffers (NCCL / peer memory) */
  CBX_MEM_CATEGORIES = 8
};
CBX_API cbx_status cbx_memory_report(cbx_ctx* ctx, long long out[CBX_MEM_CATEGORIES + 4]);
CBX_API cbx_status cbx_describe(cbx_ctx* ctx, char* buf, long n);
/* benchmark loop: nsteps fixed-dt steps, each preceded (outside the timed
 * region) by a write of flush_mb MB to evict L2; per-step CUDA events on the
 * context stream.  out_ms = {density, embed, force, store, integrate, step,
 * steps, force kernel alone} summed over the steps.  The step time comes
 * from events around each graph launch and the force kernel from an event
 * pair inside the graph; the per-phase entries (which include their
 * memsets) are measured only after cbx_bench_phases(ctx, 1) -- their event
 * nodes add latency to the step -- and are 0 otherwise. */
CBX_API cbx_status cbx_bench_steps(cbx_ctx* ctx, double dt, long nsteps, double flush_mb,
                                   double out_ms[8]);
/* measured fp64 peak of this device: a dependent-free DFMA stream over all
 * SMs, timed with CUDA events (TFLOP/s, DFMA = 2 flops) */
CBX_API cbx_status cbx_fp64_peak(int device, double* tflops, double* sm_mhz);
CBX_API cbx_status cbx_bench_phases(cbx_ctx* ctx, int on);

/* ---- the run loop and its outputs ------------------------
 * Simulation::run (sim.cpp:289-360): equilibrate (with the thermostat), inject
 * the PKA, step with the adaptive dt until the step or time cap, sampling
 * Wigner-Seitz defects and writing snapshots at the configured intervals;
 * then the defect time series and the final snapshot.  On a failed step the
 * post-mortem snapshot and the series so far are written and the error is
 * returned.  Files are byte-compatible with the reference's writers
 * (analysis.cpp:66-116).  Single-box contexts. */
typedef struct {
  long steps;                      /* step cap, 0 = none */
  double max_time;                 /* ps cap, 0 = none */
  long equilibration_steps;        /* thermal steps before the PKA */
  int thermostat_enabled;          /* ThermostatSpec (config.h:16-20) */
  long thermostat_interval;
  long thermostat_boundary_cells;  /* 0 = whole box */
  double temperature;              /* thermostat target, K */
  const char* timeseries;          /* defect CSV path; NULL / "" = skip */
  const char* snapshot_prefix;     /* XYZ prefix; NULL / "" = skip */
  long snapshot_interval;          /* 0 = only the final snapshot */
  long defect_interval;            /* 0 = ends only */
  long pka_site[3];                /* corner-sublattice cell, -1 = box centre */
  double pka_energy_kev;           /* 0 = no PKA */
  long pka_dir[3];
} cbx_run_spec;

/* log_path: NULL / "" = no log, "-" = stdout (sim.cpp:294-300 line format) */
CBX_API cbx_status cbx_run(cbx_ctx* ctx, const cbx_run_spec* spec, const char* log_path);
/* the defect series of the last run (sim.h:54): returns its length; t and
 * defects (3 per sample: vacancies, interstitials, Frenkel pairs) may be NULL */
CBX_API long cbx_run_series(cbx_ctx* ctx, double* t, long* defects);
/* thermostat_rescale (sim.cpp:188-221) toward `temperature` in the band of
 * `boundary_cells` cells at the faces (0 = whole box); then measure */
CBX_API cbx_status cbx_thermostat_rescale(cbx_ctx* ctx, double temperature, long boundary_cells);
/* write_snapshot / write_timeseries (analysis.cpp:77-116).  cbx_write_snapshot
 * returns once the file is written; cbx_write_snapshot_async packs the store on
 * the device, copies it to page-locked memory on a side stream and writes the
 * file from a host thread while later calls (steps) proceed -- two in flight,
 * a third waits for the oldest; cbx_snapshot_wait joins them (the first write
 * error is returned).  cbx_run uses the asynchronous form. */
CBX_API cbx_status cbx_write_snapshot(cbx_ctx* ctx, const char* path, double t_ps);
CBX_API cbx_status cbx_write_snapshot_async(cbx_ctx* ctx, const char* path, double t_ps);
CBX_API cbx_status cbx_snapshot_wait(cbx_ctx* ctx);
CBX_API cbx_status cbx_write_timeseries(const char* path, long n, const double* t,
                                        const long* defects);

/* ---- z-slab domain decomposition (multi-GPU) ------------- */
/* rank r of n owns global interior z planes [r*bz/n, (r+1)*bz/n) of the
 * global box; positions, hashes and keys stay in the global frame.  A step
 * is driven phase by phase by the host with the exchanges in between
 * (paper_2107_07866_b200/slab.py):
 *   phase 0 -> pack/unpack MIGRANTS(0) -> phase 1 -> POS(1) -> phase 2 ->
 *   RHO(2) -> phase 3 -> DF(3) -> phase 4 -> FRC(4) -> phase 5 -> all-reduce
 *   of cbx_slab_local_state -> cbx_slab_commit.
 * pack: dir -1 toward the rank below, +1 above; unpack: from -1 / +1.
 * Buffers are device memory of cbx_slab_buffer_bytes(kind) bytes. */
CBX_API cbx_status cbx_create_slab(const cbx_box* global_box, const cbx_potential* pot,
                                   const cbx_offsets* idx, int rank, int nranks, int device,
                                   cbx_ctx** out);
CBX_API cbx_status cbx_slab_info(cbx_ctx* ctx, long out[8]);
CBX_API long cbx_slab_buffer_bytes(cbx_ctx* ctx, int kind);
CBX_API cbx_status cbx_slab_phase(cbx_ctx* ctx, int phase, double dt);
/* Lockstep peer-memory exchange (ranks sharing a GPU, or host-driven runs of
 * the P2P transport): cbx_slab_p2p_send packs an exchange into the
 * neighbours' mapped buffers and raises their flags (returns when done);
 * after a barrier of all ranks, cbx_slab_p2p_recv unpacks what arrived.  Only
 * with the staged reverse halos (cbx_slab_p2p_set_fused(ctx, 0)). */
CBX_API cbx_status cbx_slab_p2p_send(cbx_ctx* ctx, int kind);
CBX_API cbx_status cbx_slab_p2p_recv(cbx_ctx* ctx, int kind);
CBX_API cbx_status cbx_slab_pack(cbx_ctx* ctx, int kind, int dir, void* dev_buf, long cap,
                                 long* bytes);
CBX_API cbx_status cbx_slab_unpack(cbx_ctx* ctx, int kind, int from, const void* dev_buf,
                                   long bytes);
CBX_API cbx_status cbx_slab_local_state(cbx_ctx* ctx, double out[8]);
CBX_API cbx_status cbx_slab_commit(cbx_ctx* ctx, const double in[4]);
/* In-graph exchange (one process per GPU): rank 0 makes an NCCL id, every
 * rank passes it to cbx_slab_comm_init (collective).  cbx_step,
 * cbx_eval_forces / cbx_refresh_forces, cbx_measure and cbx_bench_steps then
 * run the whole decomposed step -- exchanges and the StepState all-reduce --
 * as one CUDA graph per rank; with nranks == 1 the exchange is a self
 * send/recv (the periodic z images of a one-slab box). */
CBX_API cbx_status cbx_nccl_unique_id(void* out, long nbytes);
CBX_API cbx_status cbx_slab_comm_init(cbx_ctx* ctx, const void* id, long nbytes);
/* Peer-memory exchange (ranks on one node, NVLink / NVSwitch): each rank
 * exports a CBX_P2P_HANDLE_BYTES handle (CUDA IPC handles of its receive
 * region and of its rho / force accumulators, plus its slab geometry); every
 * rank passes the handles of all ranks (in rank order) to cbx_slab_p2p_init.
 * The forward exchanges (migrants, positions, dF) are one kernel each -- the
 * sender stores its boundary data straight into the neighbour's memory and
 * raises a flag, the receiver waits on it and unpacks.  The reverse ones
 * (density and force partials of the halo planes) are fused into the passes:
 * with the Newton-3 stencil a partial for a halo site is added straight into
 * the neighbour's boundary site over NVLink, and the consumer (embedding,
 * second half kick) waits on the neighbours' flags.  The StepState reduction
 * is the tail of the finalize kernel.  Takes precedence over an NCCL
 * communicator.  nranks == 1 maps the rank onto itself. */
#define CBX_P2P_HANDLE_BYTES 256
CBX_API cbx_status cbx_slab_p2p_handle(cbx_ctx* ctx, void* out, long nbytes);
CBX_API cbx_status cbx_slab_p2p_init(cbx_ctx* ctx, const void* handles, long nbytes);
/* 1 when this rank adds its halo partials straight into the neighbours'
 * memory (needs native fp64 peer atomics between every pair of the ranks'
 * GPUs), 0 for the staged reverse exchanges.  All ranks must agree: a caller
 * that cannot guarantee identical device visibility on every rank sets the
 * minimum over ranks with cbx_slab_p2p_set_fused. */
CBX_API int cbx_slab_p2p_fused(cbx_ctx* ctx);
CBX_API cbx_status cbx_slab_p2p_set_fused(cbx_ctx* ctx, int on);
/* drop the peer-memory transport again (before any step), e.g. when another
 * rank could not map its neighbours; connect NCCL afterwards */
CBX_API cbx_status cbx_slab_p2p_close(cbx_ctx* ctx);
CBX_API cbx_status cbx_upload_store_global(cbx_ctx* ctx, const cbx_store* global_store);
CBX_API cbx_status cbx_download_store_global(cbx_ctx* ctx, cbx_store* global_store,
                                             long* n_clash_inout);

#ifdef __cplusplus
}
#endif
#endif
