"""Build liboracle.so (TEST INFRASTRUCTURE ONLY -- see oracle.h). Plain g++, -O2 -ffp-contract=off, no fast-math.

The oracle links the synth generator only through a function-pointer callback supplied by the caller; it
contains no CUDA and shares no code with paper_2004_08532_b200/csrc.
"""
import os
import subprocess

HERE = os.path.dirname(os.path.abspath(__file__))
LIB = os.path.join(HERE, "liboracle.so")


def build(force: bool = False) -> str:
    src = [os.path.join(HERE, "oracle.cpp")]
    deps = src + [os.path.join(HERE, "oracle.h")]
    if not force and os.path.exists(LIB) and all(os.path.getmtime(LIB) >= os.path.getmtime(p) for p in deps):
        return LIB
    cmd = ["g++", "-O2", "-std=c++17", "-ffp-contract=off", "-fno-fast-math", "-fopenmp", "-fPIC", "-shared",
           "-Wall", "-o", LIB] + src
    subprocess.check_call(cmd)
    return LIB


if __name__ == "__main__":
    print(build(force=True))
