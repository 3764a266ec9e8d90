"""The drop-in boundary compiles next to the reference's own declarations
(CPU, no GPU needed): the reference's public names (namespace bmg, Eigen-free
stand-ins in tests/cpp/ref_mock, declared after /root/reference/proj/include/
blockmg/*.hpp) and the device facade (include/bmg/blockmg.hpp, namespace
bmg::cuda) in one translation unit, with the reference-side adapter
(tests/cpp/bmg_device_adapter.hpp) that INTEGRATION.md quotes verbatim."""
import os
import shutil
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CPP = os.path.join(ROOT, "tests", "cpp")


def _cxx():
    return "/usr/bin/g++" if os.path.exists("/usr/bin/g++") else shutil.which("g++")


@pytest.mark.skipif(_cxx() is None, reason="no C++ compiler")
def test_adapter_and_facade_compile_in_one_tu(tmp_path):
    out = subprocess.run([_cxx(), "-std=c++20", "-Wall", "-Wextra", "-Werror", "-c",
                          "-I" + os.path.join(ROOT, "include"), "-I" + CPP, "-I" + os.path.join(CPP, "ref_mock"),
                          os.path.join(CPP, "adapter_compile_test.cpp"), "-o", str(tmp_path / "a.o")],
                         capture_output=True, text=True)
    assert out.returncode == 0, out.stderr


def test_facade_declares_nothing_in_the_reference_namespace():
    # every facade declaration sits inside namespace bmg::cuda
    txt = open(os.path.join(ROOT, "include", "bmg", "blockmg.hpp")).read()
    body = txt[txt.index("namespace bmg {"):]
    assert body.startswith("namespace bmg {\nnamespace cuda {\n")
    assert body.rstrip().endswith("}  // namespace cuda\n}  // namespace bmg")


def test_integration_doc_quotes_the_compiled_adapter():
    doc = open(os.path.join(ROOT, "INTEGRATION.md")).read()
    src = open(os.path.join(CPP, "bmg_device_adapter.hpp")).read()
    body = src[src.index("namespace bmg_adapter {"):src.index("}  // namespace bmg_adapter")]
    assert body in doc, "INTEGRATION.md must quote tests/cpp/bmg_device_adapter.hpp verbatim"
