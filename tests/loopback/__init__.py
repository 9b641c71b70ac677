"""Builds the test-only loopback NCCL stand-in (loopback_nccl.cpp)."""
import os
import subprocess

HERE = os.path.dirname(os.path.abspath(__file__))
SO = os.path.join(HERE, "libloopback_nccl.so")


def build() -> str:
    src = os.path.join(HERE, "loopback_nccl.cpp")
    if not os.path.exists(SO) or os.path.getmtime(SO) < os.path.getmtime(src):
        tmp = SO + f".tmp{os.getpid()}"
        subprocess.check_call(["g++", "-O2", "-std=c++17", "-shared", "-fPIC", "-I/usr/local/cuda/include", src,
                               "-o", tmp, "-L/usr/local/cuda/lib64/stubs", "-lcuda", "-lpthread"])
        os.replace(tmp, SO)
    return SO
