"""A/B helper: run bench.py's main() against an alternative build of the CUDA
library (HS_LIB=path), e.g. the previous commit's, for interleaved timing
comparisons on one box. Not used by the product or the tests."""
import os
import runpy
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
if os.environ.get("HS_LIB"):
    from paper_2605_13209_b200 import _lib
    _lib.lib_path = lambda: os.environ["HS_LIB"]
sys.argv = [os.path.join(ROOT, "bench.py")] + sys.argv[1:]
runpy.run_path(os.path.join(ROOT, "bench.py"), run_name="__main__")
