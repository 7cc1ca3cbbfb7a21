"""Host setup shortcut: the grid-constant stencils (mass scaled by h^2, Q1
Poisson h-independent), the lumped mass and M f computed from the stencil are
bitwise the full assembly (tests/cpp/assembly_shortcut.cpp, CPU only)."""
import os
import subprocess

from conftest import ROOT


def test_stencil_shortcuts_are_bitwise_the_full_assembly(tmp_path):
    exe = tmp_path / "assembly_shortcut"
    subprocess.run(["g++", "-std=c++17", "-O2", os.path.join(ROOT, "tests", "cpp", "assembly_shortcut.cpp"),
                    os.path.join(ROOT, "paper_1806_05896_b200", "csrc", "assembly.cpp"), "-o", str(exe)],
                   check=True)
    out = subprocess.run([str(exe)], capture_output=True, text=True, timeout=300)
    assert out.returncode == 0, out.stdout
    assert out.stdout.strip().endswith("ok")
