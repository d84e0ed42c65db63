"""Build the in-tree CUDA library (nvcc, sm_100a) -- no JIT cache involved."""

import os
import subprocess

HERE = os.path.dirname(os.path.abspath(__file__))


def build_library(force: bool = False) -> str:
    csrc = os.path.join(HERE, "csrc")
    if force:
        subprocess.run(["make", "-s", "-C", csrc, "clean"], check=True)
    subprocess.run(["make", "-s", "-j4", "-C", csrc], check=True)
    return os.path.join(HERE, "_ptap_b200.so")


if __name__ == "__main__":
    print(build_library())
