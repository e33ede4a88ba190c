"""include/fasttrig/gpu.hpp composes with the real reference headers (CPU only)."""
import os
import subprocess

import pytest

from conftest import ROOT

REF_INC = "/root/reference/proj/include"


@pytest.mark.parametrize("with_ref", [True, False])
def test_gpu_hpp_compiles(with_ref):
    if with_ref and not os.path.isdir(os.path.join(REF_INC, "fasttrig")):
        pytest.skip("reference headers not present")
    cmd = ["g++", "-std=c++20", "-fsyntax-only", "-Wall", "-Werror", "-I" + os.path.join(ROOT, "include")]
    if with_ref:
        cmd.append("-I" + REF_INC)
    cmd.append(os.path.join(ROOT, "tests", "cpp", "test_gpu_api.cpp"))
    subprocess.run(cmd, check=True)
