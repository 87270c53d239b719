// cascade_b200.hpp -- C++ host mirror of the reference's force engine and
// step loop over the C ABI (cascade_b200.h).  Header only.
//
// Names, arguments and exception types follow the reference
// (/root/reference/proj/core/include/cascademd): status codes are rethrown
// as std::invalid_argument / std::runtime_error / std::domain_error /
// std::logic_error with the reference's message text, so a caller that
// swaps `cascademd::eval_forces(store, idx, pot, part, pool)` for
// `cascade_b200::Engine::eval_forces()` keeps its error handling.
#pragma once

#include <cstdint>
#include <stdexcept>
#include <string>
#include <vector>

#include "cascade_b200.h"

namespace cascade_b200 {

[[noreturn]] inline void throw_status(cbx_status s, const char* msg) {
  const std::string m = msg ? msg : "";
  switch (s) {
    case CBX_INVALID_ARGUMENT: throw std::invalid_argument(m);
    case CBX_DOMAIN: throw std::domain_error(m);
    case CBX_LOGIC: throw std::logic_error(m);
    default: throw std::runtime_error(m);
  }
}

inline void check(cbx_status s, const cbx_ctx* c = nullptr) {
  if (s != CBX_OK) throw_status(s, cbx_last_error(c));
}

// EamPotential + parse_potential_file (potential.h:33-69)
class Potential {
 public:
  explicit Potential(const std::string& path) { check(cbx_potential_load(path.c_str(), &p_)); }
  ~Potential() { cbx_potential_free(p_); }
  Potential(const Potential&) = delete;
  Potential& operator=(const Potential&) = delete;
  const cbx_potential* get() const { return p_; }
  double cutoff() const { return p_->cutoff; }
  double mass() const { return p_->mass; }
  double lattice_const() const { return p_->lattice_const; }

 private:
  cbx_potential* p_ = nullptr;
};

// OffsetIndex + build_offsets (neighbors.h:17-36)
class Offsets {
 public:
  Offsets(const cbx_box& b, double cutoff) { check(cbx_offsets_build(&b, cutoff, &o_)); }
  ~Offsets() { cbx_offsets_free(o_); }
  Offsets(const Offsets&) = delete;
  Offsets& operator=(const Offsets&) = delete;
  const cbx_offsets* get() const { return o_; }
  long full_count(bool odd) const { return odd ? o_->n_odd_full : o_->n_even_full; }
  long half_count(bool odd) const { return odd ? o_->n_odd_half : o_->n_even_half; }
  long z_reach() const { return o_->z_reach; }

 private:
  cbx_offsets* o_ = nullptr;
};

// make_box (sim.cpp:62-84)
inline cbx_box make_box(long bx, long by, long bz, const Potential& pot, double a0 = 0.0,
                        long ghost_width = 0, double max_disp = 0.05,
                        double* index_cutoff = nullptr) {
  cbx_box b{};
  check(cbx_make_box(bx, by, bz, a0, ghost_width, max_disp, pot.get(), &b, index_cutoff));
  return b;
}

// A LatticeStore resident on one GPU with the force engine and the step loop.
class Engine {
 public:
  Engine(const cbx_box& box, const Potential& pot, const Offsets* idx = nullptr, int device = 0) {
    check(cbx_create(&box, pot.get(), idx ? idx->get() : nullptr, device, &c_));
  }
  explicit Engine(cbx_ctx* adopt) : c_(adopt) {}
  ~Engine() { cbx_destroy(c_); }
  Engine(const Engine&) = delete;
  Engine& operator=(const Engine&) = delete;

  long slot_count() const { return cbx_slot_count(c_); }
  void set_stencil(cbx_stencil m) { check(cbx_set_stencil(c_, m), c_); }

  // store transfer (LatticeStore views, store.h:16-78)
  void upload(const cbx_store& s) { check(cbx_upload_store(c_, &s), c_); }
  void download(cbx_store& s) { check(cbx_download_store(c_, &s), c_); }
  long init_bcc(double temperature, uint64_t seed, int species = 26) {
    long n = 0;
    check(cbx_init_bcc(c_, species, temperature, seed, &n), c_);
    return n;
  }

  // LatticeStore operations (store.cpp)
  void rehash() { check(cbx_rehash(c_), c_); }
  void fill_ghosts() { check(cbx_fill_ghosts(c_), c_); }

  // forces.h:42-67
  struct ForceEnergies {
    double embedding = 0.0, pair = 0.0;
  };
  ForceEnergies eval_forces() {
    ForceEnergies e;
    check(cbx_eval_forces(c_, &e.embedding, &e.pair), c_);
    return e;
  }
  void compute_density() { check(cbx_compute_density(c_), c_); }
  double compute_embedding_derivative() {
    double e = 0;
    check(cbx_compute_embedding_derivative(c_, &e), c_);
    return e;
  }
  double compute_pair_forces() {
    double e = 0;
    check(cbx_compute_pair_forces(c_, &e), c_);
    return e;
  }

  // Simulation (sim.h:38-91) with device-resident state
  cbx_state step(double dt, long n = 1) {
    cbx_state s{};
    check(cbx_step(c_, dt, n, &s), c_);
    return s;
  }
  void set_adaptive(double dt_max, double max_disp) {
    check(cbx_set_adaptive(c_, dt_max, max_disp), c_);
  }
  cbx_state state() {
    cbx_state s{};
    check(cbx_get_state(c_, &s), c_);
    return s;
  }
  void measure() { check(cbx_measure(c_), c_); }
  void inject_pka(int64_t site, const double v[3]) { check(cbx_inject_pka(c_, site, v), c_); }
  void count_defects(long& vac, long& inter, long& fp) {
    long o[3];
    check(cbx_count_defects(c_, o), c_);
    vac = o[0];
    inter = o[1];
    fp = o[2];
  }
  // Simulation::run and its outputs (sim.cpp:188-360, analysis.cpp:66-116)
  void thermostat_rescale(double temperature, long boundary_cells = 0) {
    check(cbx_thermostat_rescale(c_, temperature, boundary_cells), c_);
  }
  void write_snapshot(const std::string& path, double t_ps) {
    check(cbx_write_snapshot(c_, path.c_str(), t_ps), c_);
  }
  void run(const cbx_run_spec& spec, const std::string& log_path = "") {
    check(cbx_run(c_, &spec, log_path.c_str()), c_);
  }
  struct DefectSample {
    double t_ps;
    long vacancies, interstitials, frenkel_pairs;
  };
  std::vector<DefectSample> series() const {
    const long n = cbx_run_series(c_, nullptr, nullptr);
    std::vector<double> t(n);
    std::vector<long> d(3 * n);
    cbx_run_series(c_, t.data(), d.data());
    std::vector<DefectSample> out(n);
    for (long i = 0; i < n; ++i) out[i] = {t[i], d[3 * i], d[3 * i + 1], d[3 * i + 2]};
    return out;
  }
  cbx_ctx* raw() const { return c_; }

 private:
  cbx_ctx* c_ = nullptr;
};

// One z slab of a box decomposed over `nranks` GPUs: the same
// Engine operations (step, eval_forces, measure, count_defects) run the
// decomposed step once the ranks are connected.  Peer memory (ranks of one
// node): every rank exports p2p_handle(), every rank passes all handles in
// rank order to connect_p2p().  NCCL: rank 0 makes nccl_unique_id(), every
// rank passes it to connect_nccl().
class SlabEngine : public Engine {
 public:
  SlabEngine(const cbx_box& global_box, const Potential& pot, int rank, int nranks,
             int device = 0)
      : Engine(create(global_box, pot, rank, nranks, device)) {}

  std::vector<unsigned char> p2p_handle() {
    std::vector<unsigned char> h(CBX_P2P_HANDLE_BYTES);
    check(cbx_slab_p2p_handle(raw(), h.data(), (long)h.size()), raw());
    return h;
  }
  void connect_p2p(const std::vector<unsigned char>& all_handles) {
    check(cbx_slab_p2p_init(raw(), all_handles.data(), (long)all_handles.size()), raw());
  }
  static std::vector<unsigned char> nccl_unique_id() {
    std::vector<unsigned char> id(128);
    check(cbx_nccl_unique_id(id.data(), (long)id.size()));
    return id;
  }
  void connect_nccl(const std::vector<unsigned char>& id) {
    check(cbx_slab_comm_init(raw(), id.data(), (long)id.size()), raw());
  }
  // global store <-> this slab (reference-layout arrays of the whole box)
  void upload_global(const cbx_store& s) { check(cbx_upload_store_global(raw(), &s), raw()); }
  long download_global(cbx_store& s, long n_clash_in = 0) {
    long n = n_clash_in;
    check(cbx_download_store_global(raw(), &s, &n), raw());
    return n;
  }

 private:
  static cbx_ctx* create(const cbx_box& b, const Potential& pot, int rank, int nranks,
                         int device) {
    cbx_ctx* c = nullptr;
    check(cbx_create_slab(&b, pot.get(), nullptr, rank, nranks, device, &c));
    return c;
  }
};

}  // namespace cascade_b200
