"""The reference's own C-ABI client test suite (tests/test_capi.cpp of the
reference: 8 doctest cases, 56 assertions) compiled against THIS
repository's include/dynbatch/dynbatch.h and linked to its libdynbatch.so
(oracle/Makefile `capi`; tests/cpp/doctest.h stands in for doctest). The
binary is built in the dev container and travels with the repo; the
reference sources are not needed at run time."""
import os
import re
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
BIN = os.path.join(ROOT, "oracle", "_ref", "test_capi_ours")
needs_bin = pytest.mark.skipif(not os.path.exists(BIN), reason="oracle/_ref/test_capi_ours not built")

# cases that execute on the device (db_execute, db_moe_run, db_verify_run)
DEVICE_CASES = {"generate, schedule, verify, execute through handles",
                "moe runs agree between naive and batched and respect call counts",
                "verification entry point runs and reports"}


def _run():
    out = subprocess.run([BIN], capture_output=True, text=True, timeout=600)
    failed = set(re.findall(r'TEST CASE "(.*)" FAILED', out.stdout))
    m = re.search(r"test cases: (\d+) \| (\d+) passed", out.stdout)
    return out, failed, (int(m.group(1)), int(m.group(2))) if m else None


@needs_bin
def test_reference_capi_suite_host_cases_pass_without_gpu():
    """Without a GPU the device cases fail loudly (no CPU fallback); every
    other reference case passes against this library."""
    from dbtest import gpu_available
    if gpu_available():
        pytest.skip("GPU present: the full suite runs in the gpu test")
    out, failed, counts = _run()
    assert counts is not None and counts[0] == 8, out.stdout
    assert failed <= DEVICE_CASES, out.stdout


@needs_bin
@pytest.mark.gpu
def test_reference_capi_suite_passes_on_the_device():
    out, failed, counts = _run()
    assert out.returncode == 0 and not failed, out.stdout
    assert counts == (8, 8), out.stdout
