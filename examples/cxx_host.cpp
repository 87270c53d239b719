// C++ caller of the C ABI through include/cascade_b200.hpp: the shape of the
// reference-side integration.  Without a GPU it exercises
// the host-side setup and the error path only.
#include <cstdio>
#include <stdexcept>

#include "cascade_b200.hpp"

int main(int argc, char** argv) {
  if (argc < 2) {
    std::fprintf(stderr, "usage: %s potential.eam [gpu [slab]]\n", argv[0]);
    return 2;
  }
  using namespace cascade_b200;
  Potential pot(argv[1]);
  double ic = 0.0;
  const cbx_box box = make_box(8, 8, 8, pot, 0.0, 0, 0.05, &ic);
  Offsets idx(box, ic);
  std::printf("box %ld^3 g=%ld cutoff=%.4f index_cutoff=%.4f offsets %ld/%ld half %ld/%ld\n",
              box.box_x, box.ghost_width, pot.cutoff(), ic, idx.full_count(false),
              idx.full_count(true), idx.half_count(false), idx.half_count(true));
  try {
    Potential bad("/nonexistent.eam");
  } catch (const std::runtime_error& e) {
    std::printf("runtime_error: %s\n", e.what());
  }
  if (argc > 2) {  // device run: Simulation constructor + 10 steps
    Engine eng(box, pot, &idx, 0);
    const long n = eng.init_bcc(600.0, 12345);
    const auto e = eng.eval_forces();
    eng.measure();
    const cbx_state s = eng.step(1e-3, 10);
    std::printf("atoms %ld E_emb %.10f E_pair %.10f -> step %ld KE %.10f\n", n, e.embedding,
                e.pair, s.step, s.kinetic);
  }
  if (argc > 3) {  // one-rank z-slab over peer memory
    SlabEngine slab(box, pot, 0, 1, 0);
    slab.connect_p2p(slab.p2p_handle());
    const long n = slab.init_bcc(600.0, 12345);
    slab.eval_forces();
    slab.measure();
    const cbx_state s = slab.step(1e-3, 10);
    std::printf("slab atoms %ld -> step %ld KE %.10f\n", n, s.step, s.kinetic);
  }
  return 0;
}
