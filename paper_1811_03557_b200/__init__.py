"""B200-native DPM hot path (arXiv 1811.03557): libdpm.so (CUDA, sm_100a) + thin binding.

Importing the package does not require a GPU; ``paper_1811_03557_b200.api`` loads
libdpm.so and raises if it is missing (no CPU fallback exists).
"""
import os

LIB_PATH = os.path.join(os.path.dirname(os.path.abspath(__file__)), "libdpm.so")


def load():
    from . import api  # noqa: F401  (raises ImportError if libdpm.so is missing)
    return api
