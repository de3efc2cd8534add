"""Build libsynth.so: the seeded synthetic-graph generator shared by the oracle's tests and the CUDA path's
tests / bench (input generation only; see synth.h)."""
import os
import subprocess

HERE = os.path.dirname(os.path.abspath(__file__))
LIB = os.path.join(HERE, "libsynth.so")


def build(force: bool = False) -> str:
    deps = [os.path.join(HERE, "synth.c"), os.path.join(HERE, "synth.h")]
    if not force and os.path.exists(LIB) and all(os.path.getmtime(LIB) >= os.path.getmtime(p) for p in deps):
        return LIB
    subprocess.check_call(["gcc", "-O2", "-fopenmp", "-fPIC", "-shared", "-Wall", "-o", LIB,
                           os.path.join(HERE, "synth.c"), "-lm"])
    return LIB


if __name__ == "__main__":
    print(build(force=True))
