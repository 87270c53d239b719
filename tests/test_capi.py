"""CPU: the C-ABI library loads without a GPU, exports every symbol that
include/cascade_b200.h declares, and its host-side setup (potential parser,
spline builder, offset builder, box derivation) equals the oracle's --
no compute calls here."""
import ctypes as C
import os
import re
import subprocess

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "cascade_b200.h")


def header_symbols():
    src = open(HEADER).read()
    return sorted(set(re.findall(r"CBX_API\s+[\w\s\*]+?\b(cbx_\w+)\s*\(", src)))


def test_library_exports_every_declared_symbol():
    from paper_2107_07866_b200 import _lib
    lib = _lib.load()
    syms = header_symbols()
    assert len(syms) >= 30
    out = subprocess.run(["nm", "-D", "--defined-only", _lib.LIB_PATH], capture_output=True,
                         text=True).stdout
    exported = set(re.findall(r"\bT (cbx_\w+)", out))
    assert set(syms) <= exported, set(syms) - exported
    assert set(syms) == {n for n, _, _ in _lib.SIGNATURES}
    for s in syms:
        getattr(lib, s)
    # nothing but the C ABI leaks out of the shared object
    assert all(n.startswith("cbx_") for n in exported)
    assert lib.cbx_abi_version() == 1


def test_library_is_sm100a():
    from paper_2107_07866_b200 import _lib
    out = subprocess.run(["cuobjdump", "--list-elf", _lib.LIB_PATH], capture_output=True,
                         text=True).stdout
    assert "sm_100a" in out


def test_potential_tables_equal_oracle(tables):
    """parse_potential_file + build_spline restated in the library's host
    code give bit-identical coefficient tables"""
    from oracle import oracle
    from paper_2107_07866_b200 import EamPotential
    for name in ("baseline", "synthetic"):
        p = EamPotential.load(tables[name])
        s = oracle.Sim(tables[name], box=(4, 4, 4), init_lattice=False)
        for w, which in enumerate(("embed", "zr", "dens")):
            x0, h, seg = p.table(which)
            ox0, oh, oseg = s.spline(w)
            assert (x0, h) == (ox0, oh)
            assert np.array_equal(seg, oseg)
        assert p.cutoff == 5.6 and p.mass == 55.845


def test_offsets_equal_oracle(tables):
    from oracle import oracle
    from paper_2107_07866_b200 import build_offsets
    for box in [(8, 8, 8), (1, 1, 1), (6, 5, 3)]:
        s = oracle.Sim(tables["synthetic"], box=box, init_lattice=False)
        dims, a0, g = s.box
        mine = build_offsets((*dims, a0, g), s.index_cutoff)
        ref = s.offsets()
        for k in ("even_full", "odd_full", "even_half", "odd_half"):
            assert np.array_equal(mine[k], ref[k]), k
        assert mine["z_reach"] == ref["z_reach"]


def test_make_box_and_errors(tables):
    from paper_2107_07866_b200 import EamPotential, SimConfig, make_box, pka_speed
    from paper_2107_07866_b200._lib import CbxInvalidArgument, CbxRuntimeError
    pot = EamPotential.load(tables["baseline"])
    box, ic = make_box(SimConfig(box_x=20, box_y=20, box_z=20), pot)
    assert (box.box_x, box.ghost_width, box.a0) == (20, 3, 2.855)
    assert ic == 5.6 + 0.3 * 2.855
    with pytest.raises(CbxInvalidArgument, match="half the lattice constant"):
        make_box(SimConfig(max_disp=1.43), pot)
    with pytest.raises(CbxRuntimeError, match="cannot open potential file"):
        EamPotential.load("/nonexistent.eam")
    assert pka_speed(1000.0, 55.845) == pytest.approx(587.8323710323659, rel=1e-14)


def test_parser_line_numbered_errors(tmp_path, tables):
    from paper_2107_07866_b200 import EamPotential
    from paper_2107_07866_b200._lib import CbxRuntimeError
    lines = open(tables["baseline"]).read().splitlines()
    bad = tmp_path / "bad.eam"
    bad.write_text("\n".join(lines[:3] + ["1.0 2.0 nope"] + lines[4:]) + "\n")
    with pytest.raises(CbxRuntimeError, match=r"bad.eam:4: non-numeric entry in embedding"):
        EamPotential.load(str(bad))
    short = tmp_path / "short.eam"
    short.write_text("\n".join(lines[:10]) + "\n")
    with pytest.raises(CbxRuntimeError, match="ends early"):
        EamPotential.load(str(short))


def test_create_without_gpu_fails_loudly(tables):
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    from paper_2107_07866_b200 import DeviceStore, EamPotential
    from paper_2107_07866_b200._lib import CbxError
    with pytest.raises(CbxError):
        DeviceStore((4, 4, 4, 2.855, 3), EamPotential.load(tables["baseline"]))


def test_cxx_host_header_compiles_and_runs(tmp_path, tables):
    """include/cascade_b200.hpp: the C++ mirror compiles against the C ABI
    and rethrows the reference's exception types (host-side calls only)"""
    from paper_2107_07866_b200 import _lib
    _lib.load()
    exe = str(tmp_path / "cxx_host")
    libdir = os.path.dirname(_lib.LIB_PATH)
    subprocess.run(["g++", "-std=c++17", "-O1", "-I", os.path.join(ROOT, "include"),
                    os.path.join(ROOT, "examples", "cxx_host.cpp"), "-L", libdir,
                    "-l:libcascade_b200.so", f"-Wl,-rpath,{libdir}", "-o", exe], check=True)
    out = subprocess.run([exe, tables["baseline"]], capture_output=True, text=True, check=True)
    assert "offsets 112/112 half 46/66" in out.stdout
    assert "runtime_error: cannot open potential file" in out.stdout


@pytest.mark.gpu
def test_cxx_engine_and_slab_engine_on_device(tmp_path, tables):
    """the C++ mirror drives the single-box Engine and a one-rank SlabEngine
    (peer-memory transport to itself) to the same trajectory"""
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2107_07866_b200 import _lib
    _lib.load()
    exe = str(tmp_path / "cxx_host")
    libdir = os.path.dirname(_lib.LIB_PATH)
    subprocess.run(["g++", "-std=c++17", "-O1", "-I", os.path.join(ROOT, "include"),
                    os.path.join(ROOT, "examples", "cxx_host.cpp"), "-L", libdir,
                    "-l:libcascade_b200.so", f"-Wl,-rpath,{libdir}", "-o", exe], check=True)
    out = subprocess.run([exe, tables["baseline"], "gpu", "slab"], capture_output=True,
                         text=True, check=True, timeout=300).stdout
    box = [ln for ln in out.splitlines() if ln.startswith("atoms")][0]
    slab = [ln for ln in out.splitlines() if ln.startswith("slab atoms")][0]
    assert box.split()[1] == slab.split()[2] == "1024"
    ke_box, ke_slab = float(box.split()[-1]), float(slab.split()[-1])
    assert box.split()[-3] == slab.split()[-3] == "10"
    assert abs(ke_box - ke_slab) <= 1e-9 * ke_box
