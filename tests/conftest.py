import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200, sm_100a)")


@pytest.fixture(scope="session")
def tables(tmp_path_factory):
    """the BASELINE table and the reference's own synthetic table, written once"""
    from oracle import oracle
    from paper_2107_07866_b200.potential import write_baseline_table
    d = tmp_path_factory.mktemp("tables")
    base = write_baseline_table(str(d / "baseline.eam"))
    base40 = write_baseline_table(str(d / "baseline40.eam"), rho_max=40.0)
    syn = str(d / "synthetic.eam")
    oracle.write_synthetic_table(syn)
    return {"baseline": base, "baseline40": base40, "synthetic": syn}


@pytest.fixture(scope="session")
def have_ref():
    from oracle import oracle
    return os.path.exists(oracle.REF_LIB)
