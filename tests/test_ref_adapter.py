"""The reference's own plug-in point on the device: tests/cpp/ref_model_adapter.cpp
runs the reference's UNMODIFIED ipm_solve (ipm.cpp:270-341) over an IpmModel whose
newton_solve is bound to oc_newton_solve (include/optcon_b200_ref.hpp:
make_steady_model / make_spacetime_model, to_b200 converters) and compares it
with the stock reference model on the same inputs (C1 minres-pd and gmres-pt,
C4 convection-diffusion, C3-style state box + partial observation, heat), to
1e-10 in u, y and J with equal Newton counts. The binary is built by
oracle/Makefile next to the reference library (oracle/_ref/) and travels to
the GPU box with it."""
import os
import subprocess

import pytest

from conftest import ROOT

EXE = os.path.join(ROOT, "oracle", "_ref", "ref_model_adapter")
REF_INC = "/root/reference/proj/include"


@pytest.mark.skipif(not os.path.isdir(REF_INC), reason="reference headers not present")
def test_adapter_header_compiles_against_reference_headers(tmp_path):
    src = tmp_path / "inc.cpp"
    src.write_text('#include "optcon_b200_ref.hpp"\nint main() { return 0; }\n')
    subprocess.run(["g++", "-std=c++20", "-fsyntax-only", f"-I{ROOT}/include", f"-I{REF_INC}",
                    f"-I{ROOT}/oracle/shim", str(src)], check=True)


@pytest.mark.gpu
def test_reference_ipm_solve_over_device_newton_solve():
    if not os.path.exists(EXE):
        pytest.skip("oracle/_ref/ref_model_adapter not built (make -C oracle)")
    out = subprocess.run([EXE], capture_output=True, text=True, timeout=900)
    print(out.stdout)
    assert out.returncode == 0, out.stdout + out.stderr
    assert "ALL PASS" in out.stdout
    assert out.stdout.count("PASS ") == 5
