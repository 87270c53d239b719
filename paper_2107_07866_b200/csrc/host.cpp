// host.cpp -- host-side setup for the B200 EAM library (see cbx_host.h).
// Compiled with -ffp-contract=off so every expression rounds like the
// reference's (the reference never contracts to FMA).
#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <fstream>
#include <random>
#include <sstream>

#include "cbx_host.h"

namespace cbx {

namespace {
thread_local std::string t_err;

// units.h:11-27 (the same constant expressions)
constexpr double ev_si = 1.602176634e-19;
constexpr double amu_si = 1.66053906660e-27;
constexpr double boltzmann_si = 1.380649e-23;
constexpr double angstrom_si = 1e-10;
constexpr double picosecond_si = 1e-12;
constexpr double accel_factor_c =
    (ev_si / angstrom_si / amu_si) * (picosecond_si * picosecond_si) / angstrom_si;
constexpr double boltzmann_ev_c = boltzmann_si / ev_si;
}  // namespace

void set_thread_error(const std::string& msg) { t_err = msg; }
const char* thread_error() { return t_err.c_str(); }

Spline build_spline(double x0, double h, const std::vector<double>& y) {
  const std::size_t n = y.size();
  if (n < 4)
    raise(CBX_INVALID_ARGUMENT, "build_spline: need at least 4 knots, got " + std::to_string(n));
  if (!(h > 0.0) || !std::isfinite(h) || !std::isfinite(x0))
    raise(CBX_INVALID_ARGUMENT, "build_spline: non-finite or non-positive grid");
  for (double v : y)
    if (!std::isfinite(v)) raise(CBX_INVALID_ARGUMENT, "build_spline: non-finite knot value");
  // second derivatives from the not-a-knot tridiagonal system
  std::vector<double> rhs2(n, 0.0), M(n, 0.0);
  const double inv_h2 = 1.0 / (h * h);
  for (std::size_t i = 1; i + 1 < n; ++i)
    rhs2[i] = 6.0 * (y[i + 1] - 2.0 * y[i] + y[i - 1]) * inv_h2;
  M[1] = rhs2[1] / 6.0;
  M[n - 2] = rhs2[n - 2] / 6.0;
  if (n > 4) {
    const std::size_t lo = 2, cnt = n - 4;
    std::vector<double> dg(cnt, 4.0), q(rhs2.begin() + lo, rhs2.begin() + lo + cnt);
    q[0] -= M[1];
    q[cnt - 1] -= M[n - 2];
    for (std::size_t k = 1; k < cnt; ++k) {  // forward elimination
      const double w = 1.0 / dg[k - 1];
      dg[k] -= w;
      q[k] -= w * q[k - 1];
    }
    M[lo + cnt - 1] = q[cnt - 1] / dg[cnt - 1];
    for (std::size_t k = cnt - 1; k-- > 0;) M[lo + k] = (q[k] - M[lo + k + 1]) / dg[k];
  }
  M[0] = 2.0 * M[1] - M[2];
  M[n - 1] = 2.0 * M[n - 2] - M[n - 3];
  Spline s;
  s.x0 = x0;
  s.h = h;
  s.seg.resize(7 * (n - 1));
  for (std::size_t i = 0; i + 1 < n; ++i) {
    double* c = &s.seg[7 * i];
    c[0] = (M[i + 1] - M[i]) / (6.0 * h);
    c[1] = 0.5 * M[i];
    c[2] = (y[i + 1] - y[i]) / h - h * (2.0 * M[i] + M[i + 1]) / 6.0;
    c[3] = y[i];
    c[4] = 3.0 * c[0];
    c[5] = 2.0 * c[1];
    c[6] = c[2];
  }
  return s;
}

namespace {

// whitespace tokenizer with the source line of every token, for the
// reference's "path:line: message" errors (potential.cpp:42-106)
class Tokens {
 public:
  explicit Tokens(const std::string& path) : path_(path), in_(path) {
    if (!in_) raise(CBX_RUNTIME, "cannot open potential file '" + path + "'");
  }
  std::string line() {
    std::string s;
    if (!std::getline(in_, s)) fail("unexpected end of file");
    ++line_;
    return s;
  }
  bool next(std::string& tok) {
    while (pos_ >= toks_.size()) {
      std::string s;
      if (!std::getline(in_, s)) return false;
      ++line_;
      toks_.clear();
      pos_ = 0;
      std::istringstream ss(s);
      std::string t;
      while (ss >> t) toks_.push_back(t);
    }
    tok = toks_[pos_++];
    return true;
  }
  [[noreturn]] void fail(const std::string& m) const {
    raise(CBX_RUNTIME, path_ + ":" + std::to_string(line_) + ": " + m);
  }

 private:
  std::string path_;
  std::ifstream in_;
  int line_ = 0;
  std::vector<std::string> toks_;
  std::size_t pos_ = 0;
};

std::vector<double> block(Tokens& t, long n, const char* what) {
  std::vector<double> v;
  v.reserve(n);
  for (long i = 0; i < n; ++i) {
    std::string tok;
    if (!t.next(tok))
      t.fail(std::string("table ") + what + " ends early: expected " + std::to_string(n) +
             " values, found " + std::to_string(i));
    char* end = nullptr;
    const double x = std::strtod(tok.c_str(), &end);
    if (end != tok.c_str() + tok.size() || !std::isfinite(x))
      t.fail(std::string("non-numeric entry in ") + what + " table: '" + tok + "'");
    v.push_back(x);
  }
  return v;
}

}  // namespace

Potential parse_potential(const std::string& path) {
  Tokens t(path);
  Potential p;
  p.comment = t.line();
  {
    std::istringstream ss(t.line());
    double z = 0.0;
    if (!(ss >> z >> p.mass >> p.lattice_const >> p.lattice_name))
      t.fail("element line needs: atomic-number mass lattice-constant name");
    if (z < 1.0 || z != std::floor(z)) t.fail("atomic number must be a positive integer");
    if (!(p.mass > 0.0)) t.fail("mass must be positive");
    if (!(p.lattice_const > 0.0)) t.fail("lattice constant must be positive");
    p.atomic_number = (int)z;
  }
  long nrho = 0, nr = 0;
  double drho = 0, dr = 0;
  {
    std::istringstream ss(t.line());
    if (!(ss >> nrho >> drho >> nr >> dr >> p.cutoff))
      t.fail("grid line needs: Nrho drho Nr dr cutoff");
    if (nrho < 4 || nr < 4) t.fail("node counts must be at least 4 (cubic spline)");
    if (!(drho > 0.0) || !(dr > 0.0)) t.fail("grid spacings must be positive");
    if (!(p.cutoff > 0.0)) t.fail("cutoff must be positive");
    if (std::abs((double)nr * dr - p.cutoff) > 1e-9)
      t.fail("cutoff does not match the r-table extent Nr*dr");
  }
  const std::vector<double> f = block(t, nrho, "embedding");
  const std::vector<double> z = block(t, nr, "pair z(r)");
  const std::vector<double> d = block(t, nr, "density");
  std::string extra;
  if (t.next(extra)) t.fail("trailing data after the tables: '" + extra + "'");
  p.embed = build_spline(0.0, drho, f);
  p.zr = build_spline(dr, dr, z);
  p.dens = build_spline(dr, dr, d);
  return p;
}

Offsets build_offsets(const cbx_box& b, double cutoff) {
  if (!(cutoff > 0.0)) raise(CBX_INVALID_ARGUMENT, "build_offsets: cutoff must be positive");
  if (cutoff > (double)b.ghost_width * b.a0) {
    char buf[200];
    std::snprintf(buf, sizeof buf,
                  "build_offsets: cutoff %f A exceeds the ghost reach ghost_width*a0 = %f A",
                  cutoff, b.ghost_width * b.a0);
    raise(CBX_INVALID_ARGUMENT, buf);
  }
  Offsets o;
  o.cutoff = cutoff;
  const long reach = (long)std::ceil(cutoff / b.a0) + 1;
  const double c2 = cutoff * cutoff;
  const long tx2 = 2 * (b.box_x + 2 * b.ghost_width);
  const int64_t sy = tx2, sz = (int64_t)tx2 * (b.box_y + 2 * b.ghost_width);
  // same-sublattice displacement (d)*a0; cross-sublattice (d +- 1/2)*a0
  for (long dz = -reach; dz <= reach; ++dz)
    for (long dy = -reach; dy <= reach; ++dy)
      for (long dx = -reach; dx <= reach; ++dx) {
        const double ds = (double)(dx * dx + dy * dy + dz * dz) * b.a0 * b.a0;
        if (ds <= c2 && !(dx == 0 && dy == 0 && dz == 0)) {
          const int64_t off = sz * dz + sy * dy + 2 * dx;
          for (int par = 0; par < 2; ++par)
            o.full[par].push_back({off, (int)dx, (int)dy, (int)dz, 0});
        }
        const double px = dx + 0.5, py = dy + 0.5, pz = dz + 0.5;
        if ((px * px + py * py + pz * pz) * b.a0 * b.a0 <= c2)
          o.full[0].push_back({sz * dz + sy * dy + (2 * dx + 1), (int)dx, (int)dy, (int)dz, 1});
        const double mx = dx - 0.5, my = dy - 0.5, mz = dz - 0.5;
        if ((mx * mx + my * my + mz * mz) * b.a0 * b.a0 <= c2)
          o.full[1].push_back({sz * dz + sy * dy + (2 * dx - 1), (int)dx, (int)dy, (int)dz, 1});
      }
  for (int par = 0; par < 2; ++par) {
    std::sort(o.full[par].begin(), o.full[par].end(),
              [](const Offset& a, const Offset& c) { return a.flat < c.flat; });
    for (const Offset& f : o.full[par])
      if (f.flat > 0) {
        o.half[par].push_back(f);
        o.z_reach = std::max<long>(o.z_reach, f.dz);
      }
  }
  return o;
}

Geo make_geo(const cbx_box& b) {
  Geo G{};
  G.bx = (int)b.box_x;
  G.by = (int)b.box_y;
  G.bz = (int)b.box_z;
  G.g = (int)b.ghost_width;
  G.tx = G.bx + 2 * G.g;
  G.ty = G.by + 2 * G.g;
  G.tz = G.bz + 2 * G.g;
  G.txy = G.tx * G.ty;
  G.NC = (long long)G.tx * G.ty * G.tz;
  G.NI = (long long)G.bx * G.by * G.bz;
  G.a0 = b.a0;
  G.lx = b.box_x * b.a0;
  G.ly = b.box_y * b.a0;
  G.lz = b.box_z * b.a0;
  G.kmx = (int)((b.ghost_width + b.box_x - 1) / b.box_x);
  G.kmy = (int)((b.ghost_width + b.box_y - 1) / b.box_y);
  G.kmz = (int)((b.ghost_width + b.box_z - 1) / b.box_z);
  G.zoff = 0;
  G.gbz = G.bz;
  G.gtz = G.tz;
  G.glz = G.lz;
  G.slab = 0;
  auto magic = [](unsigned d, unsigned long long& m, int& sh) {
    int l = 0;
    while ((1ull << l) < d) ++l;
    sh = 31 + l;
    m = ((1ull << sh) + d - 1) / d;
  };
  magic((unsigned)G.bx, G.mbx, G.sbx);
  magic((unsigned)G.by, G.mby, G.sby);
  G.col_units = ab_flag("CBX_COL_UNITS", 1);
  return G;
}

double accel_factor() { return accel_factor_c; }
double mv2_to_ev() { return 1.0 / accel_factor_c; }
double speed_factor() { return 98.22694750253277; }
double boltzmann_ev() { return boltzmann_ev_c; }

// init_bcc over the global box `b`; sites of global interior planes
// [z_lo, z_hi) are stored in the layout of `out_geo` shifted down by z_lo -
// out_geo.g planes (the whole box: z_lo = 0, out_geo = make_geo(b)).  The
// RNG stream and the momentum removal run over every global site in id
// order, so a slab gets exactly the single-box values of its planes.
static HostLattice init_bcc_planes(const cbx_box& b, const Geo& out_geo, long z_lo, long z_hi,
                                   double mass, double temperature, uint64_t seed) {
  const Geo G = make_geo(b);
  const double sigma =
      temperature > 0.0 ? std::sqrt(boltzmann_ev_c * temperature * accel_factor_c / mass) : 0.0;
  std::mt19937_64 gen(seed);
  double spare = 0.0;
  bool have = false;
  auto u01 = [&] { return (double)((gen() >> 11) + 1) * (1.0 / 9007199254740993.0); };
  auto gauss = [&] {  // Box-Muller, sim.cpp:28-38
    if (have) {
      have = false;
      return spare;
    }
    const double r = std::sqrt(-2.0 * std::log(u01()));
    const double a = 6.283185307179586476925286766559 * u01();
    spare = r * std::sin(a);
    have = true;
    return r * std::cos(a);
  };
  const Geo& O = out_geo;
  const long long S = 2 * O.NC;
  HostLattice L;
  L.pos.assign(3 * S, 0.0);
  L.vel.assign(3 * S, 0.0);
  L.tag.assign(S, 0);
  L.valid.assign(S, 0);
  uint64_t tag = 0;
  const double a = b.a0;
  double mx = 0, my = 0, mz = 0;  // net momentum, summed in global site-id order
  for (long z = G.g; z < G.g + G.bz; ++z) {
    const bool mine = z - G.g >= z_lo && z - G.g < z_hi;
    const long zl = z - z_lo;  // local plane (the halo offset g is shared)
    for (long y = G.g; y < G.g + G.by; ++y)
      for (long x = 2 * G.g; x < 2 * (G.g + G.bx); ++x) {
        double v[3];
        v[0] = sigma * gauss();
        v[1] = sigma * gauss();
        v[2] = sigma * gauss();
        mx += v[0];
        my += v[1];
        mz += v[2];
        const uint64_t t = tag++;
        if (!mine) continue;
        const long long id = ((long long)zl * O.ty + y) * (2 * O.tx) + x;
        double* p = &L.pos[3 * id];
        if (x % 2 == 0) {  // site_position, lattice.cpp:45-52
          p[0] = 0.5 * x * a;
          p[1] = y * a;
          p[2] = z * a;
        } else {
          p[0] = 0.5 * (x - 1) * a + 0.5 * a;
          p[1] = y * a + 0.5 * a;
          p[2] = z * a + 0.5 * a;
        }
        for (int k = 0; k < 3; ++k) L.vel[3 * id + k] = v[k];
        L.tag[id] = t;
        L.valid[id] = 1;
      }
  }
  L.n_atoms = (long)tag;
  // remove the net momentum (sim.cpp:122-128)
  const double inv = 1.0 / (double)L.n_atoms;
  mx *= inv;
  my *= inv;
  mz *= inv;
  for (long long id = 0; id < S; ++id)
    if (L.valid[id]) {
      L.vel[3 * id] -= mx;
      L.vel[3 * id + 1] -= my;
      L.vel[3 * id + 2] -= mz;
    }
  return L;
}

HostLattice init_bcc(const cbx_box& b, double mass, double temperature, uint64_t seed) {
  return init_bcc_planes(b, make_geo(b), 0, b.box_z, mass, temperature, seed);
}

HostLattice init_bcc_slab(const cbx_box& global, const Geo& local, double mass,
                          double temperature, uint64_t seed) {
  HostLattice L = init_bcc_planes(global, local, local.zoff, local.zoff + local.bz, mass,
                                  temperature, seed);
  long n = 0;
  for (uint8_t v : L.valid) n += v;
  L.n_atoms = n;  // atoms of this slab
  return L;
}

// ---- synthetic::write_table (synthetic.cpp:10-98, synthetic.h:19-32) ------
// The reference's own single-element test table: rho = A (rc - r)^3,
// phi = B exp(-s (r/rnn - 1)) ((rc - r)/(rc - rnn))^3, F = -C (sqrt(rho + e) -
// sqrt(e)).  Same constants, same operation order, same %.17g layout.
namespace {
namespace syn {
constexpr int atomic_number = 26;
constexpr double mass = 55.845;
constexpr double a0 = 2.8553;
constexpr double cutoff = 5.6;
constexpr double r_nn = 2.4727640449591856;
constexpr double rho_rc = 4.1;
constexpr double rho_amp = 0.02171868164588797;
constexpr double pair_slope = 6.5;
constexpr double pair_amp = 0.5123847826890735;
constexpr double embed_amp = 9.053882773088201;
constexpr double embed_reg = 0.09;
constexpr double rho_table_max = 4.0;

double density(double r) {
  if (r >= rho_rc) return 0.0;
  const double t = rho_rc - r;
  return rho_amp * t * t * t;
}
double zfun(double r) {
  if (r >= cutoff) return r * 0.0;
  const double damp = (cutoff - r) / (cutoff - r_nn);
  return r * (pair_amp * std::exp(-pair_slope * (r / r_nn - 1.0)) * damp * damp * damp);
}
double embedding(double rho) {
  return -embed_amp * (std::sqrt(rho + embed_reg) - std::sqrt(embed_reg));
}
}  // namespace syn
}  // namespace

void write_synthetic_table(const std::string& path, long nrho, long nr) {
  if (nrho < 4 || nr < 4)
    throw std::invalid_argument("write_table: need at least 4 knots per table");
  std::FILE* f = std::fopen(path.c_str(), "w");
  if (!f) throw std::runtime_error("write_table: cannot open '" + path + "' for writing");
  using namespace syn;
  std::fprintf(f,
               "synthetic Fe-like EAM: rho=%.17g*(%.17g-r)^3; "
               "phi=%.17g*exp(-%.17g*(r/%.17g-1))*((%.17g-r)/(%.17g-%.17g))^3; "
               "F=-%.17g*(sqrt(rho+%.17g)-sqrt(%.17g))\n",
               rho_amp, rho_rc, pair_amp, pair_slope, r_nn, cutoff, cutoff, r_nn, embed_amp,
               embed_reg, embed_reg);
  std::fprintf(f, "%d %.17g %.17g bcc\n", atomic_number, mass, a0);
  const double drho = rho_table_max / (double)(nrho - 1);
  const double dr = cutoff / (double)nr;
  std::fprintf(f, "%ld %.17g %ld %.17g %.17g\n", nrho, drho, nr, dr, cutoff);
  auto block = [f](long n, auto value) {  // four values per line
    for (long i = 0; i < n; ++i) std::fprintf(f, "%.17g%c", value(i), (i % 4 == 3) ? '\n' : ' ');
    if (n % 4 != 0) std::fputc('\n', f);
  };
  block(nrho, [&](long k) { return embedding(drho * (double)k); });
  block(nr, [&](long k) { return zfun(dr * (double)(k + 1)); });
  block(nr, [&](long k) { return density(dr * (double)(k + 1)); });
  if (std::fclose(f) != 0) throw std::runtime_error("write_table: write error on '" + path + "'");
}

}  // namespace cbx
