"""paper_2507_11424_b200 -- B200-native boundary-MPS bitstring sampling (arXiv 2507.11424).

The product path is libtnsample.so (CUDA, sm_100a) behind the C ABI of include/tnsample.h;
this package is the thin ctypes binding (argument marshalling only, _lib.py) plus the
multi-GPU driver (dist.py: state broadcast, contiguous sample shards, gather of bits and
ln q over torch.distributed). There is no CPU fallback.
"""
from ._lib import TNError, TNState, lib, load_library, observables  # noqa: F401

__all__ = ["TNState", "TNError", "lib", "load_library", "observables", "dist"]
