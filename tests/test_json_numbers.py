"""JSON number layout byte-compatible with the reference's nlohmann dump(2)
(src/serialize.cpp:153-158): tests/cpp/json_numbers.cpp prints
moe_config_to_json for numbers that take every branch of the layout (fixed
with ".0", fixed with a fraction, "0.000…", exponent form, subnormals,
extremes), built against the compiled reference and against this library
(oracle/Makefile `jsonnum`). Host code only: runs without a GPU."""
import os
import subprocess

import pytest

REF_DIR = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "oracle", "_ref")


def _out(name):
    path = os.path.join(REF_DIR, name)
    if not os.path.exists(path):
        pytest.skip(f"{name} not built (oracle/Makefile jsonnum needs /root/reference)")
    return subprocess.run([path], capture_output=True, text=True, check=True, timeout=60).stdout


def test_json_numbers_match_reference_bytes():
    ours, ref = _out("json_numbers_ours"), _out("json_numbers_ref")
    assert ours.count('"m"') == 24
    assert ours == ref
    # the shapes the %g form got wrong
    for text in ('"m": 10.0', '"m": 120.0', '"m": 1e+15', '"m": 123456789012345.0', '"m": 1.5e-05'):
        assert text in ours
