"""The C++ façade (include/optcon_b200.hpp) compiles against the C ABI and, on
a GPU, reproduces the reference's known answer through it."""
import os
import subprocess

import pytest

from conftest import ROOT

SRC = os.path.join(ROOT, "tests", "cpp", "facade_known_answer.cpp")
LIBDIR = os.path.join(ROOT, "paper_1806_05896_b200", "_lib")


def build(tmp_path):
    exe = tmp_path / "facade_known_answer"
    subprocess.run(["g++", "-std=c++17", "-O2", f"-I{ROOT}/include", SRC, f"-L{LIBDIR}",
                    "-loptcon_b200", f"-Wl,-rpath,{LIBDIR}", "-o", str(exe)], check=True)
    return exe


def test_facade_compiles_and_links(tmp_path):
    assert build(tmp_path).exists()


@pytest.mark.gpu
def test_facade_known_answer_on_device(tmp_path):
    exe = build(tmp_path)
    out = subprocess.run([str(exe)], capture_output=True, text=True, timeout=300)
    assert out.returncode == 0, out.stdout + out.stderr
    assert "nli=9" in out.stdout
