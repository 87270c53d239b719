"""Generate tests/golden/*.npz from the REAL reference core (oracle/_ref,
compiled from /root/reference by oracle/Makefile).  Run in the build
container (the reference tree is not on the GPU box):

    python tests/golden/make_golden.py
"""
import json
import os
import sys
import tempfile

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)

from oracle import oracle  # noqa: E402
from paper_2107_07866_b200.potential import write_baseline_table  # noqa: E402


def main():
    oracle.build(ref=True)
    path = write_baseline_table(os.path.join(tempfile.mkdtemp(), "baseline.eam"))
    meta = {"sim": {"box": [8, 8, 8], "temperature": 600.0, "seed": 12345,
                    "pka_energy_kev": 1.0, "pka_site": [4, 4, 4], "pka_dir": [1, 3, 5]},
            "dt0": 1e-3, "n0": 10, "dt1": 1e-4, "n1": 120,
            "note": "BASELINE table (rho_max 60), 600 K, 10 x 1 fs, 1 keV PKA, 120 x 0.1 fs"}
    s = oracle.Sim(path, kind="ref", **{k: tuple(v) if isinstance(v, list) else v
                                       for k, v in meta["sim"].items()})
    s.step(meta["dt0"], meta["n0"])
    s.inject_pka()
    s.step(meta["dt1"], meta["n1"])
    st = s.store()
    m = st.valid.astype(bool) & ~st.ghost.astype(bool)
    e = s.state()
    tab = sum(float(np.abs(s.spline(w)[2]).sum()) for w in range(3))
    np.savez_compressed(
        os.path.join(HERE, "cascade_8.npz"), meta=json.dumps(meta),
        slot_ids=np.nonzero(m)[0], slot_tag=st.tag[m], slot_pos=st.pos[m],
        slot_force=st.force[m], slot_rho=st.rho[m], clash_key=st.clash_key,
        clash_tag=st.clash_tag, clash_pos=st.clash_pos,
        energies=np.array([e["kinetic"], e["pair"], e["embedding"]]),
        defects=np.array(s.count_defects()), table_abs_sum=np.float64(tab))
    print("wrote cascade_8.npz; defects", s.count_defects(), "clash records", len(st.clash_key))


if __name__ == "__main__":
    main()
