import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

GOLDEN = os.path.join(ROOT, "tests", "golden")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200)")


def load_golden(name):
    """Golden fixture -> (problem namespace, outputs dict)."""
    from types import SimpleNamespace

    z = np.load(os.path.join(GOLDEN, name + ".npz"))
    p = SimpleNamespace(
        twojmax=int(z["twojmax"]), rcut=float(z["rcut"]), rmin0=float(z["rmin0"]),
        rfac0=float(z["rfac0"]), wself=float(z["wself"]), self_flag=int(z["self_flag"]),
        beta=z["beta"], weights=z["weights"], numneigh=z["numneigh"], nbr=z["nbr"],
        disp=z["disp"], types=z["types"] if "types" in z else None,
        positions=z["positions"] if "positions" in z else None,
        box=z["box"] if "box" in z else None)
    out = {k[4:]: z[k] for k in z.files if k.startswith("out_")}
    if "etotal" in out:
        out["etotal"] = float(out["etotal"])
    extra = {k: z[k] for k in z.files if not k.startswith("out_")}
    return p, out, extra


def golden_names():
    return sorted(f[:-4] for f in os.listdir(GOLDEN)
                  if f.endswith(".npz") and f != "tables.npz")


@pytest.fixture(scope="session")
def port():
    import oracle

    return oracle.Port()


def fnv1a(x):
    """common.hpp:81-99 fnv1a_bits over the IEEE bytes, hex like checksum_hex."""
    h = 0xcbf29ce484222325
    for b in np.ascontiguousarray(x, np.float64).tobytes():
        h ^= b
        h = (h * 0x100000001b3) & 0xFFFFFFFFFFFFFFFF
    return "%016x" % h


def gpu_available():
    try:
        import torch

        return torch.cuda.is_available()
    except Exception:
        return False
