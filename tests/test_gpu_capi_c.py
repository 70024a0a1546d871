"""GPU: the C ABI driven from a plain C program (tests/c/capi_demo.c): no Python on the compute path.

Adjointness of fsld_project / fsld_backproject and the brick-sorted fused loss+grad against the tile
kernel, all through include/fsld_b200.h + libfsld_b200.so (what a non-Python host binds)."""
import os
import subprocess

import pytest

from conftest import ROOT

pytestmark = pytest.mark.gpu


def build_demo() -> str:
    out_dir = os.path.join(ROOT, "tests", "c", "_build")
    os.makedirs(out_dir, exist_ok=True)
    exe = os.path.join(out_dir, "capi_demo")
    src = os.path.join(ROOT, "tests", "c", "capi_demo.c")
    lib_dir = os.path.join(ROOT, "paper_2311_16100_b200", "_lib")
    cuda = os.environ.get("CUDA_HOME", "/usr/local/cuda")
    cmd = ["gcc", "-O2", "-std=c11", "-Wall", src, "-I", os.path.join(ROOT, "include"), "-I",
           os.path.join(cuda, "include"), "-L", lib_dir, "-lfsld_b200", "-L", os.path.join(cuda, "lib64"),
           "-lcudart", "-lm", f"-Wl,-rpath,{lib_dir}", "-o", exe]
    subprocess.run(cmd, check=True, capture_output=True, text=True)
    return exe


def test_c_program_drives_the_abi():
    exe = build_demo()
    r = subprocess.run([exe], capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "capi_demo" in r.stdout
    print(r.stdout.strip())
