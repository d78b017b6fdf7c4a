"""paper_1408_1605_b200 -- B200-native level-synchronous 2D-partitioned BFS (arXiv 1408.1605).

The product is the C-ABI library ``libbfs200.so`` (``include/bfs200.h``); ``bfs`` is its thin
ctypes binding.  ``inputs`` is the seeded input generator shared with the tests.  Nothing here
falls back to a CPU implementation: without the CUDA library every call raises.
"""
import importlib

__all__ = ["bfs", "inputs"]


def __getattr__(name):
    if name in __all__:
        return importlib.import_module(f"{__name__}.{name}")
    raise AttributeError(name)
