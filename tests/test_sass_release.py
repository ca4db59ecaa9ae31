"""Every TMA-fed kernel in the CUDA library releases a shared-memory stage
only after the reads of that stage have completed (no consumer `mbarrier`
arrive ahead of the consumers of a pending LDS) -- the ordering bug that gave
wrong 64 x 64 GEMM tiles under outside memory load. Static SASS check (no
GPU): tools/sass_release_check.py over the built libhsolve_cuda.so."""
import os
import shutil
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
LIB = os.path.join(ROOT, "paper_2605_13209_b200", "libhsolve_cuda.so")
sys.path.insert(0, os.path.join(ROOT, "tools"))


@pytest.mark.skipif(not os.path.exists(LIB) or not shutil.which("cuobjdump"),
                    reason="needs the built library and cuobjdump")
def test_no_stage_release_ahead_of_pending_shared_loads(capsys):
    import sass_release_check
    assert sass_release_check.main(LIB) == 0, capsys.readouterr().out


def test_checker_flags_the_unfenced_pattern():
    import sass_release_check
    unfenced = """
        /*0100*/ SYNCS.PHASECHK.TRANS64.TRYWAIT P0, [R3+URZ+0x18000], R54 ;
        /*0110*/ LDS.64 R60, [R56+0x4000] ;
        /*0120*/ LDS.64 R58, [R56+0x4400] ;
        /*0130*/ DMMA.8x8x4 R32, R52, R60, R32 ;
        /*0140*/ @!P0 SYNCS.ARRIVE.TRANS64.A1T0 RZ, [R3+URZ+0x18018], RZ ;
        /*0150*/ DMMA.8x8x4 R20, R52, R58, R20 ;
        /*0160*/ EXIT ;
    """.split("\n")
    fenced = list(unfenced)
    fenced.insert(4, "        /*0138*/ MEMBAR.ALL.CTA ;")
    assert len(sass_release_check.check(unfenced)) == 1
    assert sass_release_check.check(fenced) == []
