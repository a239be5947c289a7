"""The reference's OWN test modules, run against the GPU-backed drop-in through the
INTEGRATION.md §1 module swap (SURVEY.md §8(b) "who calls it"): every test of
``pkg/tests/test_attention.py`` and acceptance criterion 6
(``pkg/tests/test_acceptance.py:178-225``), unmodified, with ``prefixbatch.attention``
resolved to ``paper_2412_03594_b200.attention`` (numpy in -> float64 GPU path).

The reference and its tests come from ``baseline/_ref`` (tools/install_reference.sh:
the unmodified reference, git-ignored, shipped to the GPU box with the snapshot);
skipped when it is not installed."""

import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
REF = os.path.join(ROOT, "baseline", "_ref")
REF_TESTS = os.path.join(REF, "ref_tests")


@pytest.mark.timeout(900)
@pytest.mark.parametrize("target", ["test_attention.py",
                                    "test_acceptance.py::test_criterion_6_attention_oracle_equivalence"])
def test_reference_suite_through_module_swap(target, tmp_path):
    if not os.path.isfile(os.path.join(REF_TESTS, target.split("::")[0])):
        pytest.skip("reference not installed in baseline/_ref (tools/install_reference.sh)")
    env = dict(os.environ)
    env["PYTHONPATH"] = os.pathsep.join([REF, REF_TESTS, os.path.join(ROOT, "tests", "refswap"),
                                         ROOT, env.get("PYTHONPATH", "")])
    cmd = [sys.executable, "-m", "pytest", "-p", "swap_plugin", "-q", "-s", "-p", "no:cacheprovider",
           "--rootdir", str(tmp_path), "-c", os.devnull, os.path.join(REF_TESTS, target)]
    res = subprocess.run(cmd, capture_output=True, text=True, env=env, cwd=str(tmp_path),
                         timeout=850)
    log = res.stdout + res.stderr
    assert res.returncode == 0, log[-4000:]
    assert "SWAPPED prefixbatch.attention -> paper_2412_03594_b200.attention" in log
    assert "loaded=True" in log, "the drop-in never touched libpsa.so"
    assert " passed" in log and " failed" not in log
