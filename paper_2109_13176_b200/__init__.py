"""B200-native G-VOM per-scan voxel-map update (arXiv 2109.13176).

The product is the C-ABI CUDA library ``lib/libgvom.so`` (include/gvom.h);
``gvom`` is its thin ctypes binding and ``synth`` the seeded input generator.
"""
from .gvom import GvomMap, GvomError, SensorOutside, LAYERS, load_library  # noqa: F401
