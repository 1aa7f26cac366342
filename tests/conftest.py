import json
import sys
from pathlib import Path

import numpy as np
import pytest

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
GOLDEN = ROOT / "tests" / "golden"

# Reference 4-state graph (reference tests/conftest.py F1) and the silence
# self-loop graph (F2), restated as text.
F1_TEXT = "0 1 1 1 0.5\n0 3 3 3 0.9\n1 2 2 2 0.3\n1 3 0 0 0.1\n3 2 2 2 0.7\n2 0.0\n3 0.4\n"
F2_TEXT = "0 1 1 1 0.1\n1 1 2 0 0.0\n1 0.0\n"


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (runs the CUDA library)")


def gpu_available() -> bool:
    try:
        from paper_2306_15685_b200 import _lib
        import ctypes
        n = ctypes.c_int32()
        return _lib.load().ab_device_count(ctypes.byref(n)) == 0 and n.value > 0
    except Exception:
        return False


def pytest_collection_modifyitems(config, items):
    # GPU tests fail loudly (not skip) when selected with -m gpu on a GPU-less box,
    # except that under "-m 'not gpu'" they are deselected by the marker itself.
    pass


def load_json(name: str):
    return json.loads((GOLDEN / name).read_text())


def fx(s: str) -> float:
    return float.fromhex(s)


def case_inputs(c: dict, exact: bool = False):
    """(csr, scores[T, L] f64, ctx or None, cfg) of one golden case, as package objects.
    exact: DecoderConfig.exact_counters (every candidate relaxed, so len(store)
    and eps_truncations are the reference's too)."""
    import paper_2306_15685_b200 as ab

    g = c["graph"]
    finals = {int(s): fx(w) for s, w in g["finals"]}
    csr = ab.csr_from_arrays(g["start"], g["row_offsets"], g["ilabels"], g["olabels"],
                             g["next_states"], [fx(w) for w in g["weights"]], finals,
                             fingerprint="")
    if c.get("scores"):
        scores = np.array([[fx(v) for v in row] for row in c["scores"]], dtype=np.float64)
    else:
        scores = np.zeros((0, max(c.get("width", 1), 1)), dtype=np.float64)
    ctx = None
    if c.get("ctx") is not None:
        ctx = ab.BiasingContext(id="r", arc_indices=np.array(c["ctx"]["arc_indices"], dtype=np.int64),
                                discount=fx(c["ctx"]["discount"]))
    cfg = ab.DecoderConfig(**c["cfg"], exact_counters=exact)
    return csr, scores, ctx, cfg


def expect_hyps(e: dict):
    return [(h["words"], fx(h["cost"]), h["frame"], h["kind"], h["fallback"]) for h in e["hyps"]]


@pytest.fixture(params=[False, True], ids=["cutoff", "exact"])
def exact(request):
    """Both decode modes: the expansion-time cutoff (default; hypotheses and
    surviving tokens exact) and exact_counters (every candidate relaxed;
    len(store) and eps_truncations exact too)."""
    return request.param


@pytest.fixture(scope="session")
def small_cases():
    return load_json("small_cases.json")
