// ref_harness.cpp -- the cascade_oracle.h C API implemented over the REAL
// reference core library (compiled unchanged from /root/reference/proj/core
// by oracle/Makefile into oracle/_ref/).
//
// TEST INFRASTRUCTURE ONLY.  Used (a) to pin the plain-C restatement in
// cascade_oracle.c bit-for-bit against the reference and (b) as bench.py's
// `--impl reference` / cpu_baseline arm (Simulation::step with a WorkerPool
// of all host cores).  No product code links it.
#include <cmath>
#include <cstdio>
#include <cstring>
#include <memory>
#include <stdexcept>
#include <string>
#include <vector>

#include "cascade_oracle.h"
#include "cascademd/analysis.h"
#include "cascademd/forces.h"
#include "cascademd/potential.h"
#include "cascademd/sim.h"
#include "cascademd/synthetic.h"

using namespace cascademd;

struct orc_ctx {
  orc_config cfg{};
  std::string pot_path;
  std::unique_ptr<Simulation> sim;  // init_lattice != 0
  // standalone store (init_lattice == 0)
  std::unique_ptr<EamPotential> pot_own;
  BoxSpec box_own{};
  std::unique_ptr<LatticeStore> store_own;
  OffsetIndex idx_own;
  ColorPartition part_own;
  std::unique_ptr<WorkerPool> pool;
  StepState st_own{};
  std::string err;

  LatticeStore& store() { return sim ? sim->store() : *store_own; }
  const LatticeStore& store() const { return sim ? sim->store() : *store_own; }
  const EamPotential& pot() const { return sim ? sim->potential() : *pot_own; }
  const BoxSpec& box() const { return sim ? sim->box() : box_own; }
  const OffsetIndex& idx() const { return sim ? sim->offsets() : idx_own; }
  const ColorPartition& part() const { return sim ? sim->partition() : part_own; }
};

namespace {

std::string g_err;

int code_of(const std::exception& e) {
  if (dynamic_cast<const std::invalid_argument*>(&e)) return ORC_INVALID;
  if (dynamic_cast<const std::domain_error*>(&e)) return ORC_DOMAIN;
  if (dynamic_cast<const std::logic_error*>(&e)) return ORC_LOGIC;
  return ORC_RUNTIME;
}

template <class F>
int guard(orc_ctx* c, F&& f) {
  try {
    f();
    return ORC_OK;
  } catch (const std::exception& e) {
    c->err = e.what();
    return code_of(e);
  }
}

SimConfig to_sim_config(const orc_config* cfg) {
  SimConfig s;
  s.box_x = cfg->box_x;
  s.box_y = cfg->box_y;
  s.box_z = cfg->box_z;
  s.a0 = cfg->a0;
  s.ghost_width = cfg->ghost_width;
  s.temperature = cfg->temperature;
  s.seed = cfg->seed;
  s.workers = cfg->workers > 0 ? cfg->workers : 1;
  s.pka.site_x = cfg->pka_site[0];
  s.pka.site_y = cfg->pka_site[1];
  s.pka.site_z = cfg->pka_site[2];
  s.pka.energy_kev = cfg->pka_energy_kev;
  s.pka.dir_x = cfg->pka_dir[0];
  s.pka.dir_y = cfg->pka_dir[1];
  s.pka.dir_z = cfg->pka_dir[2];
  if (cfg->dt_max > 0.0) s.dt_max = cfg->dt_max;
  if (cfg->max_disp > 0.0) s.max_disp = cfg->max_disp;
  s.thermostat.boundary_cells = cfg->thermostat_boundary_cells;
  return s;
}

void copy_state(const StepState& s, orc_state* o) {
  o->step = s.step;
  o->t = s.t;
  o->dt = s.dt;
  o->kinetic = s.kinetic;
  o->pair = s.pair;
  o->embedding = s.embedding;
  o->max_speed = s.max_speed;
  o->r_underflow = s.r_underflow;
  o->rho_clamp = s.rho_clamp;
}

}  // namespace

extern "C" {

const char* orc_create_error(void) { return g_err.c_str(); }

orc_ctx* orc_create(const char* path, const orc_config* cfg, int init_lattice) {
  auto c = std::make_unique<orc_ctx>();
  c->cfg = *cfg;
  c->pot_path = path;
  try {
    EamPotential pot = parse_potential_file(path);
    const SimConfig sc = to_sim_config(cfg);
    if (init_lattice) {
      c->sim = std::make_unique<Simulation>(sc, std::move(pot));
      c->pool = std::make_unique<WorkerPool>(c->sim->partition().workers);
    } else {
      // the same derivation as make_box / index_cutoff_of (sim.cpp:62-84)
      validate_config(sc);
      const double a0 = sc.a0 > 0.0 ? sc.a0 : pot.lattice_const;
      const double ic = pot.cutoff + 0.3 * a0;
      const long gw = sc.ghost_width > 0 ? sc.ghost_width
                                         : static_cast<long>(std::ceil(ic / a0));
      c->box_own = BoxSpec{sc.box_x, sc.box_y, sc.box_z, a0, gw};
      c->pot_own = std::make_unique<EamPotential>(std::move(pot));
      c->store_own = std::make_unique<LatticeStore>(c->box_own);
      c->idx_own = build_offsets(c->box_own, ic);
      c->part_own = build_color_partition(c->box_own, sc.workers, ic);
      c->pool = std::make_unique<WorkerPool>(c->part_own.workers);
    }
  } catch (const std::exception& e) {
    g_err = e.what();
    return nullptr;
  }
  return c.release();
}

void orc_destroy(orc_ctx* c) { delete c; }
const char* orc_error(const orc_ctx* c) { return c->err.c_str(); }

void orc_box(const orc_ctx* c, long d[4], double* a0) {
  const BoxSpec& b = c->box();
  d[0] = b.box_x;
  d[1] = b.box_y;
  d[2] = b.box_z;
  d[3] = b.ghost_width;
  *a0 = b.a0;
}
double orc_index_cutoff(const orc_ctx* c) { return c->idx().cutoff; }
double orc_potential_cutoff(const orc_ctx* c) { return c->pot().cutoff; }
double orc_mass(const orc_ctx* c) { return c->pot().mass; }

int orc_insert(orc_ctx* c, const double p[3], const double v[3], unsigned long long tag) {
  return guard(c, [&] {
    AtomRecord r;
    r.position = Vec3{p[0], p[1], p[2]};
    if (v) r.velocity = Vec3{v[0], v[1], v[2]};
    r.tag = tag;
    r.species = static_cast<std::uint16_t>(c->pot().atomic_number);
    c->store().insert(r);
  });
}

int orc_set_atom(orc_ctx* c, long long site, int idx, const double p[3], const double v[3]) {
  return guard(c, [&] {
    AtomRecord& r = c->store().at(AtomRef{site, idx});
    if (p) r.position = Vec3{p[0], p[1], p[2]};
    if (v) r.velocity = Vec3{v[0], v[1], v[2]};
  });
}

long orc_displace_interior(orc_ctx* c, const double* disp, long n) {
  long i = 0;
  LatticeStore& s = c->store();
  for_each_interior_id(s.box, [&](LatticeId id) {
    AtomRecord& r = s.slots[static_cast<std::size_t>(id)];
    if (!r.valid || i >= n) return;
    r.position += Vec3{disp[3 * i], disp[3 * i + 1], disp[3 * i + 2]};
    ++i;
  });
  return i;
}
int orc_canonicalize(orc_ctx* c) { return guard(c, [&] { c->store().canonicalize_positions(); }); }
int orc_update_hash(orc_ctx* c) { return guard(c, [&] { c->store().update_hash(); }); }
int orc_fill_ghosts(orc_ctx* c) { return guard(c, [&] { c->store().fill_ghosts(); }); }
int orc_rehash(orc_ctx* c) {
  return guard(c, [&] {
    c->store().canonicalize_positions();
    c->store().update_hash();
    c->store().fill_ghosts();
  });
}
long orc_atom_count(const orc_ctx* c) { return c->store().atom_count(); }
long long orc_nearest_site(orc_ctx* c, const double p[3]) {
  long long id = -1;
  guard(c, [&] { id = nearest_site(Vec3{p[0], p[1], p[2]}, c->box()); });
  return id;
}

int orc_eval_forces(orc_ctx* c, double* e_emb, double* e_pair) {
  return guard(c, [&] {
    const ForceEnergies en = eval_forces(c->store(), c->idx(), c->pot(), c->part(), *c->pool);
    if (e_emb) *e_emb = en.embedding;
    if (e_pair) *e_pair = en.pair;
  });
}
int orc_compute_density(orc_ctx* c) {
  return guard(c, [&] { compute_density(c->store(), c->idx(), c->pot()); });
}
int orc_compute_embedding(orc_ctx* c, double* e) {
  return guard(c, [&] {
    const double v = compute_embedding_derivative(c->store(), c->pot());
    if (e) *e = v;
  });
}
int orc_compute_pair(orc_ctx* c, double* e) {
  return guard(c, [&] {
    const double v = compute_pair_forces(c->store(), c->idx(), c->pot());
    if (e) *e = v;
  });
}
void orc_guards(const orc_ctx* c, unsigned long long out[2]) {
  out[0] = c->pot().guards.r_underflow.load();
  out[1] = c->pot().guards.rho_clamp.load();
}

int orc_refresh_forces(orc_ctx* c) { return orc_eval_forces(c, nullptr, nullptr); }
int orc_measure(orc_ctx* c) {
  c->err = "measure: private in the reference Simulation";
  return ORC_LOGIC;
}
int orc_step(orc_ctx* c, double dt, long nsteps) {
  if (!c->sim) {
    c->err = "step: needs a Simulation-backed context";
    return ORC_LOGIC;
  }
  return guard(c, [&] {
    for (long i = 0; i < nsteps; ++i) {
      if (dt > 0.0) c->sim->step(dt);
      else c->sim->step();
    }
  });
}
int orc_inject_pka(orc_ctx* c) {
  if (!c->sim) {
    c->err = "inject_pka: needs a Simulation-backed context";
    return ORC_LOGIC;
  }
  return guard(c, [&] { c->sim->inject_pka(); });
}
void orc_get_state(const orc_ctx* c, orc_state* st) {
  copy_state(c->sim ? c->sim->state() : c->st_own, st);
}
int orc_count_defects(const orc_ctx* c, long out[3]) {
  const DefectReport r = count_defects(c->store());
  out[0] = r.vacancies;
  out[1] = r.interstitials;
  out[2] = r.frenkel_pairs;
  return ORC_OK;
}

long orc_slot_count(const orc_ctx* c) { return static_cast<long>(c->store().slots.size()); }
void orc_get_slots(const orc_ctx* c, double* pos, double* vel, double* force, double* rho,
                   double* df, unsigned long long* tag, unsigned char* valid,
                   unsigned char* ghost) {
  const auto& s = c->store().slots;
  for (std::size_t i = 0; i < s.size(); ++i) {
    const AtomRecord& r = s[i];
    if (pos) { pos[3 * i] = r.position.x; pos[3 * i + 1] = r.position.y; pos[3 * i + 2] = r.position.z; }
    if (vel) { vel[3 * i] = r.velocity.x; vel[3 * i + 1] = r.velocity.y; vel[3 * i + 2] = r.velocity.z; }
    if (force) { force[3 * i] = r.force.x; force[3 * i + 1] = r.force.y; force[3 * i + 2] = r.force.z; }
    if (rho) rho[i] = r.rho_bar;
    if (df) df[i] = r.df;
    if (tag) tag[i] = r.tag;
    if (valid) valid[i] = r.valid;
    if (ghost) ghost[i] = r.ghost;
  }
}
long orc_clash_count(const orc_ctx* c) {
  long n = 0;
  for (const auto& kv : c->store().clash) n += static_cast<long>(kv.second.size());
  return n;
}
void orc_get_clash(const orc_ctx* c, long long* key, int* idx, double* pos, double* vel,
                   double* force, double* rho, double* df, unsigned long long* tag,
                   unsigned char* ghost) {
  long n = 0;
  for (const auto& kv : c->store().clash) {
    for (std::size_t j = 0; j < kv.second.size(); ++j, ++n) {
      const AtomRecord& r = kv.second[j];
      if (key) key[n] = kv.first;
      if (idx) idx[n] = static_cast<int>(j);
      if (pos) { pos[3 * n] = r.position.x; pos[3 * n + 1] = r.position.y; pos[3 * n + 2] = r.position.z; }
      if (vel) { vel[3 * n] = r.velocity.x; vel[3 * n + 1] = r.velocity.y; vel[3 * n + 2] = r.velocity.z; }
      if (force) { force[3 * n] = r.force.x; force[3 * n + 1] = r.force.y; force[3 * n + 2] = r.force.z; }
      if (rho) rho[n] = r.rho_bar;
      if (df) df[n] = r.df;
      if (tag) tag[n] = r.tag;
      if (ghost) ghost[n] = r.ghost;
    }
  }
}

void orc_offsets(const orc_ctx* c, long counts[4], long long* ef, long long* of, long long* eh,
                 long long* oh, long* z_reach) {
  const OffsetIndex& ix = c->idx();
  counts[0] = static_cast<long>(ix.even_full.size());
  counts[1] = static_cast<long>(ix.odd_full.size());
  counts[2] = static_cast<long>(ix.even_half.size());
  counts[3] = static_cast<long>(ix.odd_half.size());
  if (ef) std::memcpy(ef, ix.even_full.data(), sizeof(long long) * ix.even_full.size());
  if (of) std::memcpy(of, ix.odd_full.data(), sizeof(long long) * ix.odd_full.size());
  if (eh) std::memcpy(eh, ix.even_half.data(), sizeof(long long) * ix.even_half.size());
  if (oh) std::memcpy(oh, ix.odd_half.data(), sizeof(long long) * ix.odd_half.size());
  if (z_reach) *z_reach = ix.z_reach;
}

int orc_potential_eval(orc_ctx* c, int which, double x, double out[2]) {
  return guard(c, [&] {
    SplineEval e{};
    if (which == 0) e = c->pot().density(x);
    else if (which == 1) e = c->pot().pair(x);
    else e = c->pot().embedding(x);
    out[0] = e.value;
    out[1] = e.deriv;
  });
}

long orc_spline(const orc_ctx* c, int which, double* x0, double* h, double* seg) {
  const EamPotential& p = c->pot();
  const SplineTable& s = which == 0 ? p.embed : (which == 1 ? p.zr : p.dens);
  if (x0) *x0 = s.x0;
  if (h) *h = s.h;
  if (seg) {
    for (std::size_t i = 0; i < s.seg.size(); ++i) {
      const auto& g = s.seg[i];
      double* o = seg + 7 * i;
      o[0] = g.a; o[1] = g.b; o[2] = g.c; o[3] = g.d; o[4] = g.e; o[5] = g.f; o[6] = g.g;
    }
  }
  return static_cast<long>(s.seg.size());
}

double orc_pka_speed(double e, double m) { return pka_speed(e, m); }
double orc_adaptive_dt(double vmax, double dt_max, double max_disp) {
  SimConfig cfg;
  cfg.dt_max = dt_max;
  cfg.max_disp = max_disp;
  return adaptive_dt(vmax, cfg);
}
int orc_write_synthetic_table(const char* path, long nrho, long nr) {
  try {
    synthetic::write_table(path, nrho, nr);
  } catch (const std::exception& e) {
    g_err = e.what();
    return ORC_RUNTIME;
  }
  return ORC_OK;
}

}  // extern "C"

// ------------------------------------------------------------- run loop
extern "C" {

int orc_thermostat_rescale(orc_ctx* c) {
  if (!c->sim) {
    c->err = "thermostat: needs a Simulation-backed context";
    return ORC_LOGIC;
  }
  return guard(c, [&] { c->sim->thermostat_rescale(); });
}

int orc_write_snapshot(const orc_ctx* c, const char* path) {
  return guard(const_cast<orc_ctx*>(c), [&] {
    write_snapshot(path, c->store(), c->sim ? c->sim->state().t : c->st_own.t);
  });
}

int orc_write_timeseries(const char* path, long n, const double* t, const long* d) {
  std::vector<DefectSample> v;
  for (long i = 0; i < n; ++i) {
    DefectReport r;
    r.vacancies = d[3 * i];
    r.interstitials = d[3 * i + 1];
    r.frenkel_pairs = d[3 * i + 2];
    v.push_back(DefectSample{t[i], r});
  }
  try {
    write_timeseries(path, v);
  } catch (const std::exception&) {
    return ORC_RUNTIME;
  }
  return ORC_OK;
}

// a fresh Simulation from the creation config plus the run spec (the
// reference fixes cfg_ at construction), which then replaces the context's
int orc_run(orc_ctx* c, const orc_run_spec* r, const char* log_path) {
  return guard(c, [&] {
    SimConfig sc = to_sim_config(&c->cfg);
    sc.steps = r->steps;
    sc.max_time = r->max_time;
    sc.equilibration_steps = r->equilibration_steps;
    sc.thermostat.enabled = r->thermostat_enabled != 0;
    sc.thermostat.interval = r->thermostat_interval;
    sc.thermostat.boundary_cells = r->thermostat_boundary_cells;
    sc.output.timeseries = r->timeseries ? r->timeseries : "";
    sc.output.snapshot_prefix = r->snapshot_prefix ? r->snapshot_prefix : "";
    sc.output.snapshot_interval = r->snapshot_interval;
    sc.output.defect_interval = r->defect_interval;
    c->cfg.thermostat_boundary_cells = r->thermostat_boundary_cells;
    c->sim = std::make_unique<Simulation>(sc, parse_potential_file(c->pot_path));
    std::FILE* log = nullptr;
    if (log_path && log_path[0]) log = std::strcmp(log_path, "-") == 0 ? stdout : std::fopen(log_path, "w");
    try {
      c->sim->run(log);
    } catch (...) {
      if (log && log != stdout) std::fclose(log);
      throw;
    }
    if (log && log != stdout) std::fclose(log);
    if (log == stdout) std::fflush(stdout);
  });
}

long orc_series(const orc_ctx* c, double* t, long* d) {
  if (!c->sim) return 0;
  const auto& s = c->sim->series();
  for (size_t i = 0; i < s.size(); ++i) {
    if (t) t[i] = s[i].t_ps;
    if (d) {
      d[3 * i] = s[i].defects.vacancies;
      d[3 * i + 1] = s[i].defects.interstitials;
      d[3 * i + 2] = s[i].defects.frenkel_pairs;
    }
  }
  return static_cast<long>(s.size());
}

}  // extern "C"

// ------------------------------------------------------- config front end
// config.cpp:162-188 through the real reference: the parsed SimConfig as
// key=value lines (the layout of paper_2107_07866_b200.config.dump_config),
// or the exception message.  Returns ORC_OK, ORC_INVALID (invalid_argument)
// or ORC_RUNTIME (runtime_error).
#include "cascademd/config.h"
extern "C" {

int ref_load_config(const char* path, const char* const* overrides, int n, char* out, long cap) {
  std::string text;
  int rc = ORC_OK;
  try {
    std::vector<std::string> ov(overrides, overrides + n);
    const SimConfig c = load_config(path, ov);
    char b[256];
    auto add = [&](const char* k, const std::string& v) { text += std::string(k) + "=" + v + "\n"; };
    auto L = [&](long x) { return std::to_string(x); };
    auto D = [&](double x) {
      std::snprintf(b, sizeof b, "%.17g", x);
      return std::string(b);
    };
    auto T = [&](long x, long y, long z) { return L(x) + "," + L(y) + "," + L(z); };
    add("box.x", L(c.box_x));
    add("box.y", L(c.box_y));
    add("box.z", L(c.box_z));
    add("box.a0", D(c.a0));
    add("box.ghost_width", L(c.ghost_width));
    add("temperature", D(c.temperature));
    add("potential", c.potential_path);
    add("pka.site", T(c.pka.site_x, c.pka.site_y, c.pka.site_z));
    add("pka.energy", D(c.pka.energy_kev));
    add("pka.direction", T(c.pka.dir_x, c.pka.dir_y, c.pka.dir_z));
    add("steps", L(c.steps));
    add("max_time", D(c.max_time));
    add("dt_max", D(c.dt_max));
    add("max_disp", D(c.max_disp));
    add("thermostat.enabled", L(c.thermostat.enabled ? 1 : 0));
    add("thermostat.interval", L(c.thermostat.interval));
    add("thermostat.boundary_cells", L(c.thermostat.boundary_cells));
    add("output.timeseries", c.output.timeseries);
    add("output.snapshot_prefix", c.output.snapshot_prefix);
    add("output.snapshot_interval", L(c.output.snapshot_interval));
    add("output.defect_interval", L(c.output.defect_interval));
    add("workers", L(c.workers));
    add("seed", std::to_string(c.seed));
    add("equilibration_steps", L(c.equilibration_steps));
    add("displacement_energy", D(c.displacement_energy));
  } catch (const std::invalid_argument& e) {
    text = e.what();
    rc = ORC_INVALID;
  } catch (const std::exception& e) {
    text = e.what();
    rc = ORC_RUNTIME;
  }
  std::snprintf(out, cap, "%s", text.c_str());
  return rc;
}

int ref_nrt_displacements(double e, double ed, double* out) {
  try {
    *out = nrt_displacements(e, ed);
  } catch (const std::invalid_argument& x) {
    g_err = x.what();
    return ORC_INVALID;
  }
  return ORC_OK;
}

}  // extern "C"
