"""The INTEGRATION.md C++ shim: same signatures as the reference's
decode_stream, compiled against the reference headers (CPU) and run (GPU)."""
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
REF_INC = "/root/reference/proj/core/include"
DEMO = os.path.join(ROOT, "examples", "shim_demo")


@pytest.mark.skipif(not os.path.isdir(REF_INC), reason="reference headers absent")
def test_shim_compiles_against_reference_headers(tmp_path):
    out = tmp_path / "demo"
    subprocess.run(["g++", "-std=c++20", f"-I{REF_INC}", f"-I{ROOT}/include", f"-I{ROOT}/examples",
                    os.path.join(ROOT, "examples", "shim_demo.cpp"), f"-L{ROOT}/paper_1503_07387_b200",
                    "-lmvb_cuda", "-o", str(out)], check=True)
    assert out.exists()


@pytest.mark.gpu
def test_shim_demo_runs_on_gpu():
    if not os.path.exists(DEMO):
        pytest.fail("examples/shim_demo not built (run __graft_entry__.build() where /root/reference exists)")
    r = subprocess.run([DEMO], capture_output=True, text=True, env={**os.environ,
                        "LD_LIBRARY_PATH": os.path.join(ROOT, "paper_1503_07387_b200")})
    assert r.returncode == 0, r.stdout + r.stderr
    assert "128 386 16 32" in r.stdout
