"""Builds and runs tests/cpp/planner_internal.cpp against the host sources
(the reference's acceptance criteria 1-3 at the C++ level)."""
import os
import subprocess

from conftest import ROOT


def test_planner_internals(tmp_path):
    from paper_1509_04394_b200 import build as B
    exe = tmp_path / "planner_internal"
    host = os.path.join(B.CSRC, "host")
    cmd = [B.CXX, "-std=c++20", "-O1", "-ffp-contract=off", f"-I{host}",
           f"-I{os.path.join(ROOT, 'include')}",
           f"-I{B.JSON_DIR}", os.path.join(ROOT, "tests", "cpp", "planner_internal.cpp"),
           os.path.join(host, "model.cpp"), os.path.join(host, "planner.cpp"),
           "-o", str(exe)]
    subprocess.run(cmd, check=True)
    r = subprocess.run([str(exe)], capture_output=True, text=True, timeout=120)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "OK" in r.stdout
