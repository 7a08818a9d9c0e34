"""In-tree build of the sm_100a library (nvcc via csrc/Makefile).

The shared library lands next to this file (paper_2301_03989_b200/libpswarm_b200.so)
so it travels with the repository snapshot to the GPU box.
"""
from __future__ import annotations

import os
import subprocess

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")


def build_library(jobs: int = 4) -> str:
    subprocess.run(["make", "-s", f"-j{jobs}", "-C", CSRC], check=True)
    return os.path.join(HERE, "libpswarm_b200.so")


if __name__ == "__main__":
    print(build_library())
