"""Generate tests/golden/c3_cascade.npz from the REAL reference core
(oracle/_ref, compiled from /root/reference by oracle/Makefile).  Run in the
build container (the reference tree is not on the GPU box):

    python tests/golden/make_c3_cascade.py [--steps 1000] [--workers 8]

BASELINE config 3 as SURVEY.md §8(d) restates it: BCC Fe 100^3 cells
(2,000,000 atoms), init_bcc at 600 K from seed 12345 (sim.cpp:100-130), no
equilibration, a 10 keV PKA on the corner site of cell (50,50,50) along
(1,3,5)/sqrt(35) (sim.cpp:163-186), then 1000 x Simulation::step(1e-4)
(sim.cpp:248-273).  Every 100 steps the reference's Wigner-Seitz counts
(count_defects, analysis.cpp:40-56), the StepState energies, the clash
records (key, bucket index, tag) and a digest of the slot occupancy are
recorded; at the end also the 4096 fastest atoms (tag, position, velocity).
"""
import argparse
import json
import os
import sys
import tempfile
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)

from oracle import oracle  # noqa: E402
from paper_2107_07866_b200.potential import write_baseline_table  # noqa: E402


def occupancy_digest(site_ids: np.ndarray, tags: np.ndarray) -> int:
    """order-independent digest of the (site -> tag) map of occupied interior
    slots: sum over slots of mix(site, tag) mod 2^64 (shared with the GPU test)"""
    x = site_ids.astype(np.uint64) * np.uint64(0x9E3779B97F4A7C15)
    x ^= tags.astype(np.uint64) + np.uint64(0x632BE59BD9B4E019)
    x ^= x >> np.uint64(29)
    x *= np.uint64(0xBF58476D1CE4E5B9)
    x ^= x >> np.uint64(32)
    return int(x.sum(dtype=np.uint64))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--steps", type=int, default=1000)
    ap.add_argument("--every", type=int, default=100)
    ap.add_argument("--workers", type=int, default=os.cpu_count() or 1)
    ap.add_argument("--out", default=os.path.join(HERE, "c3_cascade.npz"))
    args = ap.parse_args()
    oracle.build(ref=True)
    path = write_baseline_table(os.path.join(tempfile.mkdtemp(), "baseline.eam"))
    meta = {"sim": {"box": [100, 100, 100], "temperature": 600.0, "seed": 12345,
                    "pka_energy_kev": 10.0, "pka_site": [50, 50, 50], "pka_dir": [1, 3, 5]},
            "dt": 1e-4, "steps": args.steps, "every": args.every,
            "workers": args.workers,
            "note": "BASELINE config 3: BASELINE table (rho_max 60), 600 K, 10 keV PKA "
                    "(1,3,5) at cell (50,50,50), 1000 x 0.1 fs; real reference (oracle/_ref)"}
    s = oracle.Sim(path, kind="ref", workers=args.workers,
                   **{k: tuple(v) if isinstance(v, list) else v for k, v in meta["sim"].items()})
    s.inject_pka()
    rows, clash, digests = [], [], []
    t0 = time.time()

    def record(step):
        e = s.state()
        st = s.store()
        m = st.valid.astype(bool) & ~st.ghost.astype(bool)
        ids = np.nonzero(m)[0]
        rows.append([step, e["kinetic"], e["pair"], e["embedding"], e["max_speed"],
                     *s.count_defects()])
        cm = st.clash_ghost == 0
        clash.append(np.stack([np.full(cm.sum(), step), st.clash_key[cm],
                               st.clash_idx[cm], st.clash_tag[cm].astype(np.int64)], axis=1))
        digests.append(occupancy_digest(ids, st.tag[m]))
        print(f"step {step}: defects {s.count_defects()} clash {cm.sum()} "
              f"E {e['kinetic'] + e['pair'] + e['embedding']:.10f} "
              f"({time.time() - t0:.0f} s)", flush=True)
        return st, m

    record(0)
    done = 0
    while done < args.steps:
        n = min(args.every, args.steps - done)
        s.step(meta["dt"], n)
        done += n
        st, m = record(done)
    # the fastest atoms at the end (slot + interior clash records)
    tags = np.concatenate([st.tag[m], st.clash_tag[st.clash_ghost == 0]]).astype(np.int64)
    pos = np.concatenate([st.pos[m], st.clash_pos[st.clash_ghost == 0]])
    vel = np.concatenate([st.vel[m], st.clash_vel[st.clash_ghost == 0]])
    sp = (vel * vel).sum(axis=1)
    top = np.argsort(-sp, kind="stable")[:4096]
    np.savez_compressed(
        args.out, meta=json.dumps(meta),
        rows=np.array(rows, dtype=np.float64),
        digests=np.array(digests, dtype=np.uint64),
        clash=np.concatenate(clash).astype(np.int64),
        fast_tag=tags[top], fast_pos=pos[top], fast_vel=vel[top])
    print("wrote", args.out, "in %.0f s" % (time.time() - t0))


if __name__ == "__main__":
    main()
