"""The C++ host path (include/kbgrid.hpp over the C-ABI) on the GPU."""
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
BIN = os.path.join(ROOT, "tests", "cpp", "grid_pass_demo")


def test_cpp_host_builds(built):
    assert os.path.exists(BIN)


@pytest.mark.gpu
def test_cpp_host_runs(built):
    env = dict(os.environ)
    env["LD_LIBRARY_PATH"] = os.path.join(ROOT, "paper_1402_4247_b200", "lib") + ":" + env.get("LD_LIBRARY_PATH", "")
    r = subprocess.run([BIN], capture_output=True, text=True, env=env, timeout=300)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "grid_pass_demo ok" in r.stdout
