"""Phase timing of diag128 (debug build tools/libhsolve_cuda_diagtiming.so,
compiled with -DHS_DIAG_TIMING): prints clock64 cycles per phase."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2605_13209_b200 import _lib  # noqa: E402

_lib.lib_path = lambda: os.path.join(os.path.dirname(os.path.abspath(__file__)),
                                     "libhsolve_cuda_diagtiming.so")
import paper_2605_13209_b200 as hs  # noqa: E402

rt = hs.Runtime()
m = hs.generate_spd_device(rt, 512, 512, seed=42)
hs.potrf_device(rt, m)
rt.close()
