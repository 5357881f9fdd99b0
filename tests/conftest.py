import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (sm_100a) GPU and the built CUDA library")
    config.addinivalue_line("markers", "slow: long-running CPU test")


@pytest.fixture(scope="session")
def oracle_mod():
    import oracle
    oracle.build()
    return oracle


# ---------------------------------------------------------------- parity error log
# GPU parity tests record their normwise error per (config, layer, op, math) here; the session writes
# them to gpurun_out/parity_errors.json so the margin against the 1e-5 / 5e-3 bars is visible
# (copied to profiles/ per round).
_PARITY_ROWS = []


@pytest.fixture(scope="session")
def parity_log():
    return _PARITY_ROWS


def pytest_sessionfinish(session, exitstatus):
    if not _PARITY_ROWS:
        return
    import json
    out = os.path.join(ROOT, "gpurun_out", "parity_errors.json")
    try:
        os.makedirs(os.path.dirname(out), exist_ok=True)
        old = []
        if os.path.exists(out):
            try:
                old = json.load(open(out)).get("rows", [])
            except Exception:
                old = []
        keys = {(r["config"], r["layer"], r["op"], r["math"], r.get("check")) for r in _PARITY_ROWS}
        rows = [r for r in old if (r["config"], r["layer"], r["op"], r["math"], r.get("check")) not in keys]
        json.dump({"rows": rows + _PARITY_ROWS}, open(out, "w"), indent=1)
    except Exception:
        pass
