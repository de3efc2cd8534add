"""B200-native (sm_100a) DGL-KE mini-batch KGE training step (arXiv 2004.08532).

The product is libkge.so (C-ABI, include/kge.h) built from csrc/; `kge` is its thin ctypes binding.
"""
from . import kge  # noqa: F401
from .kge import Config, Handle, KgeError, init  # noqa: F401

__all__ = ["kge", "Config", "Handle", "KgeError", "init"]
