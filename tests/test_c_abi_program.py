"""The C ABI used from a plain C program (examples/sma_c_demo.c): no Python,
no torch in the process.  CPU: it compiles and links against include/sma.h and
libsma.so.  GPU: it runs, and its z matches the oracle."""
import os
import subprocess

import numpy as np
import pytest

import sma_inputs

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _build(tmp_path):
    from paper_1901_02244_b200 import _build as B
    B.build()
    exe = str(tmp_path / "sma_c_demo")
    subprocess.check_call(["gcc", "-O2", "-Wall", "-Werror", "-I", os.path.join(ROOT, "include"),
                           os.path.join(ROOT, "examples", "sma_c_demo.c"),
                           "-L", os.path.join(ROOT, "paper_1901_02244_b200"), "-lsma",
                           f"-Wl,-rpath,{os.path.join(ROOT, 'paper_1901_02244_b200')}", "-o", exe])
    return exe


def test_c_program_compiles_and_links(tmp_path):
    assert os.path.exists(_build(tmp_path))


@pytest.mark.gpu
def test_c_program_matches_oracle(tmp_path, orc):
    exe = _build(tmp_path)
    d, k, R = 100_003, 4, 10
    zpath = str(tmp_path / "z.bin")
    out = subprocess.run([exe, str(d), str(k), str(R), zpath], capture_output=True, text=True,
                         timeout=120)
    assert out.returncode == 0, out.stderr
    z = np.fromfile(zpath, dtype=np.float32)
    assert z.size == d
    z4 = np.array([float(v) for v in out.stdout.split("z[0..3]=")[1].split()[:4]])
    assert np.array_equal(z4.astype(np.float32), z[:4])
    F = lambda x: float(np.float32(x))  # noqa: E731
    st = orc.State.init(np.zeros(d), k)     # the demo starts from w0 = 0
    for i in range(R):
        st.round(np.stack([sma_inputs.grad(i, j, k, d) for j in range(k)]), F(1 / k), F(0.1), F(0.9))
    # every element of z, element-wise, within the north_star tolerance
    assert np.max(np.abs(z - st.z) / (1 + np.abs(st.z))) <= 1e-5
