import json
import os
import sys

import numpy as np
import pytest

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
for p in (HERE, ROOT):
    if p not in sys.path:
        sys.path.insert(0, p)

GOLDEN = os.path.join(HERE, "golden")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200) and libglsim_cuda.so")


def golden_names():
    with open(os.path.join(GOLDEN, "index.json")) as f:
        return sorted(json.load(f))


def load_golden(name):
    """(docs, outputs dict) of one reference-generated fixture."""
    import gen
    z = np.load(os.path.join(GOLDEN, f"{name}.npz"))
    meta = json.loads(bytes(z["meta"]).decode())
    docs = gen.Docs(meta["lib"], meta["net"], meta["sdf"], meta["vcd"], meta["period"],
                    meta["pct"], meta["avg"])
    out = {k: z[k] for k in z.files if k != "meta"}
    out["saif"] = bytes(out["saif"]).decode()
    out["report"] = json.loads(bytes(out["report"]).decode())
    return docs, out


@pytest.fixture(scope="session")
def oracle_lib():
    from oracle import port
    port.build()
    return port
collect_ignore = ["reference_suite"]
