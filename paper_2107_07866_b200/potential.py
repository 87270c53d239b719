"""BASELINE synthetic EAM table in the reference's funcfl layout.

BASELINE.json configs quote a synthetic tabulated EAM that the reference does
not ship (its own generator, core/src/synthetic.cpp:50-98, writes a different
smooth Fe-like table).  This writer produces the BASELINE recipe in exactly
the file format `parse_potential_file` reads (core/include/cascademd/
potential.h:62-69, core/src/potential.cpp:134-185), so the CUDA path and the
CPU checkers load the *same file*:

* pair:     phi(r) = D (exp(-2 alpha (r - r0)) - 2 exp(-alpha (r - r0))),
            D = 0.4 eV, alpha = 1.4 / A, r0 = 2.85 A, tabulated as z = r phi
* density:  rho(r) = exp(-2.0 (r - 2.48))
* embedding F(rho) = -sqrt(rho)
* 5000 knots per table, cutoff 5.6 A (dr = cutoff / 5000, r_k = (k+1) dr),
  F knots at k * drho with drho = rho_max / 4999, a0 = 2.855 A, mass 55.845 amu.

rho_max is the one free choice; the default 60.0 is about
5x the perfect-lattice density rho_bar_eq = 11.8096.
"""
from __future__ import annotations

import math

BASELINE_RHO_MAX = 60.0


def baseline_functions(D=0.4, alpha=1.4, r0=2.85, rho_r0=2.48, rho_k=2.0):
    def phi(r):
        return D * (math.exp(-2.0 * alpha * (r - r0)) - 2.0 * math.exp(-alpha * (r - r0)))

    def rho(r):
        return math.exp(-rho_k * (r - rho_r0))

    def emb(p):
        return -math.sqrt(p)

    return phi, rho, emb


def _block(vals):
    out = []
    for i, v in enumerate(vals):
        out.append("%.17g%s" % (v, "\n" if i % 4 == 3 else " "))
    if len(vals) % 4:
        out.append("\n")
    return "".join(out)


def write_baseline_table(path: str, rho_max: float = BASELINE_RHO_MAX, nrho: int = 5000,
                         nr: int = 5000, cutoff: float = 5.6, a0: float = 2.855,
                         mass: float = 55.845, rho_k: float = 2.0) -> str:
    """rho_k: the density decay constant (2.0 = BASELINE; tests use steeper
    tables to exercise the fp64 fallback of the compressed records)"""
    phi, rho, emb = baseline_functions(rho_k=rho_k)
    drho = rho_max / (nrho - 1)
    dr = cutoff / nr
    lines = [
        "BASELINE synthetic EAM: phi=Morse(D=0.4,alpha=1.4,r0=2.85); rho=exp(-%g(r-2.48)); "
        "F=-sqrt(rho); rho_max=%.17g\n" % (rho_k, rho_max),
        "26 %.17g %.17g bcc\n" % (mass, a0),
        "%d %.17g %d %.17g %.17g\n" % (nrho, drho, nr, dr, cutoff),
    ]
    lines.append(_block([emb(drho * k) for k in range(nrho)]))
    rs = [dr * (k + 1) for k in range(nr)]
    lines.append(_block([r * phi(r) for r in rs]))
    lines.append(_block([rho(r) for r in rs]))
    with open(path, "w") as f:
        f.write("".join(lines))
    return path
