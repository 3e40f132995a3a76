"""The reference's OWN test suite, run unchanged against the drop-in.

SURVEY.md section 8(b) "Conformance": with ``paper_1912_06976_b200/compat``
first on ``sys.path``, ``import bttb`` resolves to the GPU drop-in, and the
reference tests (/root/reference/pkg/tests, copied next to the reference
install in ``baseline/_ref/ref_tests`` by ``tools/install_reference.sh``)
exercise it through the reference's public API.  Dense assembly comes from the
unmodified reference install (the shim re-exports it), so every
dense-vs-transform comparison below is reference numpy entries vs the GPU
operator.

Required (verdict round 1): test_multiply.py in full, the
TestBuildTransformStack shape/count cases (test_transform.py:84-96) and
acceptance criteria 1 and 4 (test_acceptance.py:37-55, :103-117).  The whole
suite is also run and every outcome is printed; ``EXPECTED_FAIL`` lists the
tests that cannot pass against a GPU build, with the reason.
"""
import os
import subprocess
import sys
import xml.etree.ElementTree as ET

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
REF = os.environ.get("BTTB_REFERENCE_INSTALL", os.path.join(ROOT, "baseline", "_ref"))
REF_TESTS = os.path.join(REF, "ref_tests")
COMPAT = os.path.join(ROOT, "paper_1912_06976_b200", "compat")

pytestmark = [
    pytest.mark.gpu,
    pytest.mark.skipif(not os.path.isdir(REF_TESTS),
                       reason="reference install missing (tools/install_reference.sh)"),
]

REQUIRED_FILES = ["test_multiply.py"]
REQUIRED_IDS = [
    "test_transform.py::TestBuildTransformStack::test_shapes_problem_one",
    "test_transform.py::TestBuildTransformStack::test_element_count",
    "test_acceptance.py::test_criterion_1_oracle_equivalence",
    "test_acceptance.py::test_criterion_4_adjoint",
]
# tests that are expected to fail against the GPU build, with the reason
EXPECTED_FAIL = {}


def _run(args, tmp_path, name):
    xml = tmp_path / f"{name}.xml"
    env = dict(os.environ)
    env["PYTHONPATH"] = os.pathsep.join([COMPAT, ROOT, env.get("PYTHONPATH", "")])
    env["PYTHONDONTWRITEBYTECODE"] = "1"
    cmd = [sys.executable, "-m", "pytest", "-q", "-p", "no:cacheprovider", "-o", "addopts=",
           "--rootdir", REF_TESTS, f"--junitxml={xml}", *args]
    proc = subprocess.run(cmd, cwd=REF_TESTS, env=env, capture_output=True, text=True, timeout=1800)
    outcomes = {}
    if xml.exists():
        for case in ET.parse(xml).getroot().iter("testcase"):
            cid = f"{case.get('file') or case.get('classname')}::{case.get('name')}"
            cls = case.get("classname", "")
            short = cls.split(".")[-1]
            mod = cls.split(".")[0]
            key = f"{mod}.py::{short}::{case.get('name')}" if short != mod else f"{mod}.py::{case.get('name')}"
            state = "passed"
            for child in case:
                if child.tag in ("failure", "error"):
                    state = "failed"
                elif child.tag == "skipped":
                    state = "skipped"
            outcomes[key] = state
            del cid
    return proc, outcomes


def test_reference_suite_required_subset(tmp_path):
    args = [os.path.join(REF_TESTS, f) for f in REQUIRED_FILES]
    args += [os.path.join(REF_TESTS, i) for i in REQUIRED_IDS]
    proc, outcomes = _run(args, tmp_path, "required")
    print(proc.stdout[-3000:])
    assert proc.returncode == 0, proc.stdout[-5000:] + proc.stderr[-2000:]
    assert len(outcomes) >= 20, outcomes
    assert all(v == "passed" for v in outcomes.values()), outcomes


def test_reference_suite_full(tmp_path):
    proc, outcomes = _run([REF_TESTS], tmp_path, "full")
    failed = sorted(k for k, v in outcomes.items() if v == "failed")
    passed = sum(v == "passed" for v in outcomes.values())
    print(f"reference suite against the drop-in: {passed} passed, {len(failed)} failed, "
          f"{sum(v == 'skipped' for v in outcomes.values())} skipped")
    for k in failed:
        print("  FAILED", k, "(expected: " + EXPECTED_FAIL[k] + ")" if k in EXPECTED_FAIL else "")
    assert outcomes, proc.stdout[-5000:] + proc.stderr[-2000:]
    unexpected = [k for k in failed if k not in EXPECTED_FAIL]
    assert not unexpected, proc.stdout[-8000:]
