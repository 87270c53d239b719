// cbx_host.h -- host-side runtime of the B200 EAM library: potential file
// parsing and spline construction, offset tables, box derivation and the
// initial lattice.  These restate the reference's host setup so a context
// built from a potential file is bit-identical to the reference's in-memory
// tables; they run once per context, never per step.
#pragma once

#include <cstdint>
#include <stdexcept>
#include <string>
#include <vector>

#include "../../include/cascade_b200.h"
#include "cbx_internal.h"

namespace cbx {

struct Status : std::runtime_error {
  cbx_status code;
  Status(cbx_status c, const std::string& m) : std::runtime_error(m), code(c) {}
};
[[noreturn]] inline void raise(cbx_status c, const std::string& m) { throw Status(c, m); }

void set_thread_error(const std::string& msg);
const char* thread_error();

struct Spline {
  double x0 = 0, h = 0;
  std::vector<double> seg;  // 7 per segment: a b c d e f g
  long nseg() const { return (long)(seg.size() / 7); }
  double x_last() const { return x0 + h * (double)nseg(); }
};

// src/spline.cpp:14-77
Spline build_spline(double x0, double h, const std::vector<double>& y);

struct Potential {
  std::string comment, lattice_name;
  int atomic_number = 0;
  double mass = 0, lattice_const = 0, cutoff = 0;
  Spline embed, zr, dens;
};
// src/potential.cpp:134-185
Potential parse_potential(const std::string& path);
// synthetic::write_table (synthetic.cpp:49-98): the reference's test table
void write_synthetic_table(const std::string& path, long nrho, long nr);

// one neighbour offset in cell units: partner cell = cell + (dx, dy, dz),
// partner sublattice = par ^ cross
struct Offset {
  int64_t flat;  // reference site-id offset (neighbors.h:22-23)
  int dx, dy, dz, cross;
};
struct Offsets {
  double cutoff = 0;
  long z_reach = 0;
  std::vector<Offset> full[2], half[2];  // [parity]
};
// src/neighbors.cpp:11-87
Offsets build_offsets(const cbx_box& b, double cutoff);

// src/sim.cpp:100-130: perfect BCC lattice with Maxwell-Boltzmann velocities
// from std::mt19937_64 + Box-Muller, momentum removed; arrays by reference
// site id over the whole ghost-inclusive box (ghost entries left invalid)
struct HostLattice {
  std::vector<double> pos, vel;
  std::vector<uint64_t> tag;
  std::vector<uint8_t> valid;
  long n_atoms = 0;
};
HostLattice init_bcc(const cbx_box& b, double mass, double temperature, uint64_t seed);
HostLattice init_bcc_slab(const cbx_box& global, const Geo& local, double mass,
                          double temperature, uint64_t seed);

Geo make_geo(const cbx_box& b);

// units.h:17-24, evaluated by the host compiler exactly as the reference does
double accel_factor();
double mv2_to_ev();
double speed_factor();
double boltzmann_ev();  // units.h:31

}  // namespace cbx
