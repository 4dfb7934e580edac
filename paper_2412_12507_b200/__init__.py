"""B200-native (sm_100a) 3DGUT forward rasterizer: UT projection, tile binning,
(tile, depth) onesweep radix sort, 3D max-response compositing.

The product is libgut.so behind the C ABI in include/gut.h; `gut` is its thin
ctypes binding.  Build with `python -m paper_2412_12507_b200.build`.
"""
from . import gut  # noqa: F401
