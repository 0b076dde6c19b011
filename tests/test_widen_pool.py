"""Host unit test of the int32 -> int64 row expansion (csrc/widen_pool.h) that the host path of
axb_compute_host_finish runs on CPU threads while result chunks cross PCIe.  Pure host code: compiled
with g++ and run here, no GPU needed."""
import os
import subprocess

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_widen_pool_expands_rows_exactly(tmp_path):
    exe = tmp_path / "widen_pool_test"
    src = os.path.join(ROOT, "tests", "native", "widen_pool_test.cpp")
    subprocess.run(["g++", "-O2", "-std=c++17", "-pthread", "-o", str(exe), src], check=True)
    out = subprocess.run([str(exe)], capture_output=True, text=True, timeout=120)
    assert out.returncode == 0, out.stdout + out.stderr
    assert "bad=0" in out.stdout
