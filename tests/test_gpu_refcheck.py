"""GPU: the reference's OWN unit tests (proj/tests/test_*.cpp, 120 test cases)
and acceptance suite, compiled unchanged and linked against the drop-in C++
adapter (paper_2506_10092_b200/adapter/runq_adapter.cpp) so every
runq::compute / enc / masks / agg / kernels call runs on the B200 through
librunq_b200.so (tests/refcheck/Makefile). The same test binary linked with
the reference's own operator objects (bin/runq_tests_cpu) passes 120/120 on
the CPU — the control that the doctest stand-in is faithful."""
import os
import re
import subprocess

import pytest

pytestmark = pytest.mark.gpu

BIN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "refcheck", "bin")


def _run(name, *args, timeout=900):
    exe = os.path.join(BIN, name)
    if not os.path.exists(exe):
        pytest.skip(f"{exe} not built (make -C tests/refcheck, needs /root/reference at build time)")
    return subprocess.run([exe, *args], capture_output=True, text=True, timeout=timeout)


def test_reference_unit_tests_on_device():
    r = _run("runq_tests")
    print(r.stdout[-2000:], r.stderr[-4000:])
    m = re.search(r"test cases: (\d+) \| (\d+) passed \| (\d+) failed", r.stdout)
    assert m, r.stdout[-2000:]
    total, passed, failed = map(int, m.groups())
    assert total == 120 and failed == 0 and r.returncode == 0, r.stderr[-4000:]


def test_reference_acceptance_on_device():
    r = _run("runq_acceptance")
    print(r.stdout)
    lines = {l.split("  ")[1].split(".")[0]: l.startswith("PASS") for l in r.stdout.splitlines()
             if l.startswith(("PASS", "FAIL"))}
    # 1 paper fixtures (< 1 s), 2 randomized differential suite, 3 run
    # statistics, 4 size accounting + bounds, 6 invariant suites; 5 needs the
    # reference's data directory, absent on the GPU box
    for c in ("1", "2", "3", "4", "6"):
        assert lines.get(c), r.stdout
