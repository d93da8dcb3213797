"""pytest plugin: run the reference's own tests with tilefusion's kernels
bound to libtfb200 (integration/tilefusion_kernels_b200.py).

    PYTHONPATH=baseline/_ref:integration:. python -m pytest -p pytest_b200_shim \
        baseline/_ref_tests/test_tsdf.py

At the end it writes the per-kernel call counts to $TFB200_SHIM_REPORT
(JSON), so a caller can check the B200 kernels actually ran.
"""

import json
import os


def pytest_configure(config):
    import tilefusion

    import tilefusion_kernels_b200 as shim
    shim.install(tilefusion)


def pytest_unconfigure(config):
    import tilefusion_kernels_b200 as shim
    out = os.environ.get("TFB200_SHIM_REPORT")
    if out:
        with open(out, "w") as fh:
            json.dump(shim.CALLS, fh)
