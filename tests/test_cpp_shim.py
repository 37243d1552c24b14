"""The C++ shim (include/fsagp_b200.hpp) compiles and links against the C ABI
library on CPU; on the GPU it runs a reference-shaped fit objective."""
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
EXE = os.path.join(ROOT, "build", "shim_example")


def build_example():
    os.makedirs(os.path.dirname(EXE), exist_ok=True)
    lib = os.path.join(ROOT, "paper_2405_14492_b200")
    subprocess.run(["g++", "-std=c++17", "-O2", "-I", os.path.join(ROOT, "include"),
                    os.path.join(ROOT, "tests", "cpp", "shim_example.cpp"), "-L", lib, "-lfsa_b200",
                    f"-Wl,-rpath,{lib}", "-o", EXE], check=True)
    return EXE


def test_shim_compiles_and_links():
    assert os.path.exists(build_example())


@pytest.mark.gpu
def test_shim_runs_on_gpu():
    out = subprocess.run([build_example()], check=True, capture_output=True, text=True).stdout
    assert out.startswith("nll ")
