/*
 * cascade_oracle.h -- CPU restatement of the reference EAM hot path.
 *
 * TEST INFRASTRUCTURE ONLY.  This header and cascade_oracle.c are the
 * checker the CUDA path is compared against (tests/, __graft_entry__.smoke()
 * and bench.py's cpu_baseline leg).  Nothing in paper_2107_07866_b200/
 * links, loads or calls it.
 *
 * The same C API is implemented twice:
 *   oracle/cascade_oracle.c  -- plain-C restatement (this header), serial,
 *                               W = 1 semantics, each function citing the
 *                               reference file:line it restates;
 *   oracle/ref_harness.cpp   -- thin adapter over the *real* reference core
 *                               (compiled from /root/reference by
 *                               oracle/Makefile into oracle/_ref/), used to
 *                               pin the restatement bit-for-bit.
 * Python loads either through oracle/oracle.py.
 *
 * Reference paths are relative to /root/reference/proj.
 */
#ifndef CASCADE_ORACLE_H
#define CASCADE_ORACLE_H

#ifdef __cplusplus
extern "C" {
#endif

typedef struct orc_ctx orc_ctx;

/* the SimConfig fields the hot path consumes (core/include/cascademd/config.h:36-53) */
typedef struct {
  long box_x, box_y, box_z;
  double a0;          /* 0 = lattice constant from the potential file */
  long ghost_width;   /* 0 = ceil(index_cutoff / a0) (sim.cpp:74-76) */
  double temperature; /* K */
  unsigned long long seed;
  int workers;        /* ref harness: WorkerPool size; restatement: ignored (W = 1) */
  long pka_site[3];   /* corner-sublattice cell, -1 = box centre */
  double pka_energy_kev;
  long pka_dir[3];
  double dt_max, max_disp;
  long thermostat_boundary_cells; /* ThermostatSpec::boundary_cells (config.h:16-20) */
} orc_config;

/* StepState (sim.h:11-21) */
typedef struct {
  long step;
  double t, dt, kinetic, pair, embedding, max_speed;
  unsigned long long r_underflow, rho_clamp;
} orc_state;

/* status codes: 0 ok, 1 invalid_argument, 2 runtime_error (overlap, parse),
 * 3 domain_error, 4 logic_error */
enum { ORC_OK = 0, ORC_INVALID = 1, ORC_RUNTIME = 2, ORC_DOMAIN = 3, ORC_LOGIC = 4 };

/* create: init_lattice != 0 runs the full Simulation constructor
 * (sim.cpp:135-148: init_bcc, fill_ghosts, refresh_forces, measure);
 * init_lattice == 0 leaves an empty store for insert()-built scenarios.
 * Returns NULL on failure; the message is then in orc_create_error(). */
orc_ctx* orc_create(const char* potential_path, const orc_config* cfg, int init_lattice);
const char* orc_create_error(void);
void orc_destroy(orc_ctx* c);
const char* orc_error(const orc_ctx* c);

void orc_box(const orc_ctx* c, long out_dims[4], double* a0);
double orc_index_cutoff(const orc_ctx* c);
double orc_potential_cutoff(const orc_ctx* c);
double orc_mass(const orc_ctx* c);

/* LatticeStore ops (store.h:52-77) */
int orc_insert(orc_ctx* c, const double pos[3], const double vel[3], unsigned long long tag);
/* add disp[3i..3i+2] to the i-th valid interior slot atom (interior-id order);
 * returns the number of atoms displaced (a harness feature: BASELINE config 2) */
long orc_displace_interior(orc_ctx* c, const double* disp, long n);
int orc_set_atom(orc_ctx* c, long long site, int clash_idx, const double pos[3], const double vel[3]);
int orc_canonicalize(orc_ctx* c);
int orc_update_hash(orc_ctx* c);
int orc_fill_ghosts(orc_ctx* c);
int orc_rehash(orc_ctx* c); /* canonicalize + update_hash + fill_ghosts (helpers.h:196-200) */
long orc_atom_count(const orc_ctx* c);
long long orc_nearest_site(orc_ctx* c, const double p[3]); /* -1 on domain error */

/* force engine (forces.h:42-67) */
int orc_eval_forces(orc_ctx* c, double* e_emb, double* e_pair);
int orc_compute_density(orc_ctx* c);
int orc_compute_embedding(orc_ctx* c, double* e_emb);
int orc_compute_pair(orc_ctx* c, double* e_pair);
void orc_guards(const orc_ctx* c, unsigned long long out[2]);

/* Simulation (sim.h:38-91) */
int orc_refresh_forces(orc_ctx* c);
int orc_measure(orc_ctx* c);
int orc_step(orc_ctx* c, double dt, long nsteps); /* dt <= 0: adaptive_dt per step */
int orc_inject_pka(orc_ctx* c);
void orc_get_state(const orc_ctx* c, orc_state* st);
int orc_count_defects(const orc_ctx* c, long out[3]);

/* store dumps; any output pointer may be NULL.  Slots: slot_count records by
 * site id.  Clash: every record in (key, bucket index) order, ghosts included. */
long orc_slot_count(const orc_ctx* c);
void orc_get_slots(const orc_ctx* c, double* pos, double* vel, double* force, double* rho,
                   double* df, unsigned long long* tag, unsigned char* valid,
                   unsigned char* ghost);
long orc_clash_count(const orc_ctx* c);
void orc_get_clash(const orc_ctx* c, long long* key, int* idx, double* pos, double* vel,
                   double* force, double* rho, double* df, unsigned long long* tag,
                   unsigned char* ghost);

/* offsets (neighbors.h:17-36): counts = {even_full, odd_full, even_half, odd_half} */
void orc_offsets(const orc_ctx* c, long counts[4], long long* even_full, long long* odd_full,
                 long long* even_half, long long* odd_half, long* z_reach);

/* potential evaluation (potential.h:50-59): which 0 density, 1 pair, 2 embedding */
int orc_potential_eval(orc_ctx* c, int which, double x, double out[2]);
/* spline coefficient table dump (spline.h:16-27): which 0 embed, 1 zr, 2 dens.
 * seg may be NULL (query nseg); returns nseg, fills x0/h. */
long orc_spline(const orc_ctx* c, int which, double* x0, double* h, double* seg);

/* ---- the run loop and its outputs ---------------
 * the SimConfig fields Simulation::run consumes (config.h:16-53); strings may
 * be NULL or "" (skip) */
typedef struct {
  long steps;               /* step cap, 0 = none */
  double max_time;          /* ps cap, 0 = none */
  long equilibration_steps; /* thermal steps before the PKA */
  int thermostat_enabled;
  long thermostat_interval;
  long thermostat_boundary_cells; /* 0 = whole box */
  const char* timeseries;      /* defect CSV path */
  const char* snapshot_prefix; /* XYZ prefix */
  long snapshot_interval;      /* 0 = only the final snapshot */
  long defect_interval;        /* 0 = ends only */
} orc_run_spec;

/* thermostat_rescale (sim.cpp:188-221): rescale toward cfg.temperature in
 * the band cfg.thermostat_boundary_cells (0 = whole box) */
int orc_thermostat_rescale(orc_ctx* c);
/* write_snapshot (analysis.cpp:90-116) */
int orc_write_snapshot(const orc_ctx* c, const char* path);
/* write_timeseries (analysis.cpp:77-88): n samples, defects as 3n longs */
int orc_write_timeseries(const char* path, long n, const double* t, const long* defects);
/* Simulation::run (sim.cpp:289-360); log_path NULL/"" = no log, "-" = stdout.
 * The ref harness runs a fresh Simulation built from the creation config. */
int orc_run(orc_ctx* c, const orc_run_spec* spec, const char* log_path);
/* the defect series of the last run: returns its length; t / defects (3n) may be NULL */
long orc_series(const orc_ctx* c, double* t, long* defects);

double orc_pka_speed(double energy_ev, double mass_amu);
double orc_adaptive_dt(double max_speed, double dt_max, double max_disp);
/* write the reference's synthetic Fe-like table (synthetic.cpp:50-98) */
int orc_write_synthetic_table(const char* path, long nrho, long nr);

#ifdef __cplusplus
}
#endif
#endif
