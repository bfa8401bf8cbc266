"""sk200: a B200-native sparse-convolution engine for the TorchSparse++ hot path
(arXiv 2311.12862), behind the sparsekit operator API (/root/reference/proj).

The compute lives in libsk200.so (hand-written sm_100a CUDA behind the C ABI
in include/sk200.h); this package is the host-side mirror of the reference
interface. Import of the torch-facing API is lazy so the C-ABI checks run
without a GPU.
"""
__version__ = "0.1.0"


def __getattr__(name):
    if name in ("sparse",):
        import importlib
        return importlib.import_module(f".{name}", __name__)
    raise AttributeError(name)
