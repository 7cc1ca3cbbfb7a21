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


def test_exit_hook_closes_problems_before_contexts():
    """The atexit hook closes every live device object, problems and
    hierarchies before contexts (a context must outlive what it owns)."""
    from paper_1806_05896_b200 import optcon

    order = []

    class Fake:
        def __init__(self, tag):
            self.tag = tag

        def close(self):
            order.append(self.tag)

    ctx, prob, mg = Fake("ctx"), Fake("prob"), Fake("mg")
    optcon._live_contexts.add(ctx)
    optcon._live_objects.add(prob)
    optcon._live_objects.add(mg)
    try:
        optcon._close_live_objects()
    finally:
        optcon._live_contexts.discard(ctx)
        optcon._live_objects.discard(prob)
        optcon._live_objects.discard(mg)
    assert sorted(order[:2]) == ["mg", "prob"] and order[2:] == ["ctx"]
