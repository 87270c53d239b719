"""shared comparison helpers (the oracle is the checker; see oracle/)."""
import numpy as np


def real_mask(s):
    return s.valid.astype(bool) & ~s.ghost.astype(bool)


def by_tag(s):
    """{tag: (pos, vel, force, rho, df)} over non-ghost atoms, slots + clash"""
    m = real_mask(s)
    out = {}
    for arrs, mask in (((s.tag, s.pos, s.vel, s.force, s.rho, s.df), m),
                       ((s.clash_tag, s.clash_pos, s.clash_vel, s.clash_force, s.clash_rho,
                         s.clash_df), s.clash_ghost == 0)):
        tag, pos, vel, frc, rho, df = arrs
        for i in np.nonzero(mask)[0]:
            out[int(tag[i])] = (pos[i], vel[i], frc[i], rho[i], df[i])
    return out


def structure(s):
    """slot occupancy (site -> tag) and clash buckets (key -> [tags]), non-ghost"""
    m = real_mask(s)
    slots = {int(i): int(s.tag[i]) for i in np.nonzero(m)[0]}
    buckets = {}
    for k, t, g in zip(s.clash_key, s.clash_tag, s.clash_ghost):
        buckets.setdefault(int(k), []).append((int(t), int(g)))
    return slots, buckets


def assert_store_parity(ref, dev, rel=1e-10, force_floor=1.0, pos_tol=0.0, what=""):
    """the north-star tolerances: structure bit-exact; rho, dF within rel;
    forces within rel*max(|f|, floor); positions exact (or pos_tol)"""
    sr, sd = structure(ref), structure(dev)
    assert sr[0] == sd[0], f"{what}: slot occupancy differs"
    assert sr[1] == sd[1], f"{what}: clash buckets differ"
    a, b = by_tag(ref), by_tag(dev)
    assert a.keys() == b.keys()
    worst = {"pos": 0.0, "rho": 0.0, "df": 0.0, "force": 0.0, "vel": 0.0}
    for t, (pa, va, fa, ra, da) in a.items():
        pb, vb, fb, rb, db = b[t]
        worst["pos"] = max(worst["pos"], float(np.abs(pa - pb).max()))
        worst["vel"] = max(worst["vel"], float(np.abs(va - vb).max() / max(1.0, np.abs(va).max())))
        worst["rho"] = max(worst["rho"], abs(ra - rb) / max(abs(ra), 1e-300))
        worst["df"] = max(worst["df"], abs(da - db) / max(abs(da), 1e-300))
        worst["force"] = max(worst["force"],
                             float(np.abs(fa - fb).max() / max(np.abs(fa).max(), force_floor)))
    assert worst["pos"] <= pos_tol, (what, worst)
    assert worst["rho"] <= rel and worst["df"] <= rel and worst["force"] <= rel, (what, worst)
    return worst
