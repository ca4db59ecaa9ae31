"""BSPD1 matrix / vector files (reference matrix_io.hpp:9-19).

CPU: the C-ABI format code (hs_bspd1_*, hs_vector_*) against the compiled
reference (oracle/_ref: save_matrix / load_matrix from the unmodified
matrix_io.cpp) — files are byte-identical in both directions, and every
corruption the reference's tests make (test_genmat.cpp:115-163) is rejected
with the same error kind and payload.

GPU: hs_matrix_load_bspd1 streams a file into HBM tiles bit-exactly (row
sharded and block-cyclic layouts), hs_matrix_save_bspd1 writes the same bytes
as the host writer, and a solve on a loaded matrix equals one on the uploaded
matrix.
"""
import os

import numpy as np
import pytest

import paper_2605_13209_b200 as hs
from paper_2605_13209_b200 import _lib
from oracle import packed_len

KIND = {1: "config_error", 7: "format_error", 8: "version_mismatch", 9: "truncated_file",
        10: "io_error"}


def random_packed(n, b, seed):
    """Packed values with awkward bit patterns (signed zeros, inf, nan,
    subnormals) so a byte-level round trip is really checked."""
    rng = np.random.default_rng(seed)
    v = rng.standard_normal(packed_len(n, b))
    special = np.array([0.0, -0.0, np.inf, -np.inf, np.nan, 5e-324, -1.7976931348623157e308])
    idx = rng.integers(0, v.size, size=min(v.size, 16))
    v[idx] = special[rng.integers(0, special.size, size=idx.size)]
    return v


def our_status(fn, *args):
    try:
        fn(*args)
    except hs.HsolveError as e:
        return e
    return None


@pytest.mark.parametrize("n,b,seed", [(1, 1, 0), (20, 4, 3), (45, 8, 1), (75, 12, 9),
                                      (130, 64, 2)])
def test_files_identical_to_reference(reference, tmp_path, n, b, seed):
    v = random_packed(n, b, seed)
    ours, theirs = str(tmp_path / "ours.bspd"), str(tmp_path / "ref.bspd")
    hs.save_matrix(hs.BlockedSPDMatrix(n, b, v.copy()), ours)
    reference.save_matrix(n, b, v, theirs)
    assert open(ours, "rb").read() == open(theirs, "rb").read()
    # each side loads the other's file bit-exactly
    m = hs.load_matrix(theirs)
    assert (m.n, m.b) == (n, b)
    assert m.values.tobytes() == v.tobytes()
    st, rn, rb, rv, _, _ = reference.load_matrix(ours)
    assert st == 0 and (rn, rb) == (n, b) and rv.tobytes() == v.tobytes()


def test_round_trip_random_shapes(tmp_path):
    # test_genmat.cpp:98-114 (shapes from a seeded generator)
    rng = np.random.default_rng(1234)
    for trial in range(5):
        n = 16 + int(rng.integers(0, 60))
        b = 1 + int(rng.integers(0, 12))
        v = random_packed(n, b, trial)
        p = str(tmp_path / f"rt{trial}.bspd")
        hs.save_matrix(hs.BlockedSPDMatrix(n, b, v.copy()), p)
        back = hs.load_matrix(p)
        assert (back.n, back.b) == (n, b)
        assert back.values.tobytes() == v.tobytes()


def corruptions(good: bytes):
    """The reference's BSPD1 error cases (test_genmat.cpp:115-158) plus a few
    more header cuts."""
    yield "wrong magic", b"X" + good[1:]
    yield "version mismatch", good[:4] + b"\x02" + good[5:]
    yield "truncated block region", good[:-100]
    yield "truncated header", good[:10]
    yield "implausible n", good[:5] + b"\xff" * 8 + good[13:]
    yield "zero b", good[:13] + b"\x00" * 8 + good[21:]
    yield "magic only", good[:4]
    yield "empty", b""
    yield "one byte short", good[:-1]


def test_error_kinds_match_reference(reference, tmp_path):
    v = random_packed(20, 4, 3)
    p = str(tmp_path / "good.bspd")
    reference.save_matrix(20, 4, v, p)
    good = open(p, "rb").read()
    bad = str(tmp_path / "bad.bspd")
    for name, data in corruptions(good):
        open(bad, "wb").write(data)
        st, _, _, _, ea, eb = reference.load_matrix(bad)
        err = our_status(hs.load_matrix, bad)
        assert st != 0 and err is not None, name
        assert err.kind == KIND[st], (name, err.kind, KIND[st])
        if st == 9:  # truncated_file carries (expected, actual) bytes
            assert (err.expected_bytes, err.actual_bytes) == (ea, eb), name
    # the reference's own expectations for the block-region cut
    open(bad, "wb").write(good[:-100])
    err = our_status(hs.load_matrix, bad)
    assert isinstance(err, hs.TruncatedFileError)
    assert (err.expected_bytes, err.actual_bytes) == (len(good), len(good) - 100)
    open(bad, "wb").write(good[:4] + b"\x02" + good[5:])
    err = our_status(hs.load_matrix, bad)
    assert isinstance(err, hs.VersionMismatchError) and (err.expected, err.actual) == (1, 2)


def test_missing_file_is_io_error():
    err = our_status(hs.load_matrix, "/tmp/hsolve_does_not_exist.bspd")
    assert isinstance(err, hs.IoError)
    err = our_status(hs.save_matrix, hs.BlockedSPDMatrix(4, 2), "/nonexistent_dir/x.bspd")
    assert isinstance(err, hs.IoError)


def test_vector_round_trip_and_reference_bytes(reference, tmp_path):
    # test_genmat.cpp:165-175
    v = hs.generate_rhs(33, 8, 9)
    p, q = str(tmp_path / "vec.bin"), str(tmp_path / "vref.bin")
    hs.save_vector(v, p)
    reference.save_vector(33, 8, v.values, q)
    assert open(p, "rb").read() == open(q, "rb").read()
    back = hs.load_vector(p, 8)
    assert back.n == 33 and back.values.tobytes() == v.values.tobytes()
    open(q, "wb").write(open(p, "rb").read()[:-3])
    assert isinstance(our_status(hs.load_vector, q, 8), hs.TruncatedFileError)
    open(q, "wb").write(b"\x00" * 8)
    assert isinstance(our_status(hs.load_vector, q, 8), hs.FormatError)


def test_cpp_matrix_io_header_matches_reference_signatures():
    src = open(os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))),
                            "include", "hsolve", "matrix_io.hpp")).read()
    for sig in ["void save_matrix(const BlockedSPDMatrix& m, const std::string& path);",
                "BlockedSPDMatrix load_matrix(const std::string& path);",
                "void save_vector(const BlockVector& v, const std::string& path);",
                "BlockVector load_vector(const std::string& path, std::size_t block_size);"]:
        assert sig in src


# ---------------------------------------------------------------------------
# device streaming path


@pytest.mark.gpu
@pytest.mark.parametrize("n,b,cyclic", [(1000, 128, False), (1000, 128, True),
                                        (4096, 512, False), (300, 7, False),
                                        (9000, 256, True)])
def test_device_load_bit_exact(rt, tmp_path, n, b, cyclic):
    v = random_packed(n, b, n)
    p = str(tmp_path / "m.bspd")
    hs.save_matrix(hs.BlockedSPDMatrix(n, b, v.copy()), p)
    d = hs.DeviceMatrix.load_bspd1(rt, p, cyclic=cyclic)
    assert (d.n, d.b) == (n, b)
    assert d.download().tobytes() == v.tobytes()
    q = str(tmp_path / "back.bspd")
    d.save_bspd1(q)
    assert open(q, "rb").read() == open(p, "rb").read()
    d.free()


@pytest.mark.gpu
def test_device_save_over_longer_file_truncates(rt, tmp_path):
    p = str(tmp_path / "m.bspd")
    big = hs.BlockedSPDMatrix(512, 64, random_packed(512, 64, 1))
    hs.save_matrix(big, p)
    small = hs.generate_spd_device(rt, 256, 64, seed=5)
    small.save_bspd1(p)
    back = hs.load_matrix(p)
    assert (back.n, back.b) == (256, 64)
    assert back.values.tobytes() == small.download().tobytes()
    assert os.path.getsize(p) == 21 + packed_len(256, 64) * 8


@pytest.mark.gpu
def test_device_load_errors(rt, tmp_path):
    p = str(tmp_path / "m.bspd")
    hs.save_matrix(hs.BlockedSPDMatrix(64, 16, random_packed(64, 16, 2)), p)
    good = open(p, "rb").read()
    for name, data in corruptions(good):
        open(p, "wb").write(data)
        with pytest.raises(hs.HsolveError) as ei:
            hs.DeviceMatrix.load_bspd1(rt, p)
        try:
            hs.load_matrix(p)
        except hs.HsolveError as e:
            assert type(e) is type(ei.value), name
    with pytest.raises(hs.IoError):
        hs.DeviceMatrix.load_bspd1(rt, "/tmp/hsolve_does_not_exist.bspd")


@pytest.mark.gpu
def test_solve_on_loaded_matrix_matches_generated(rt, tmp_path):
    import torch
    n, b = 2048, 128
    m = hs.generate_spd_device(rt, n, b, seed=42)
    p = str(tmp_path / "gp.bspd")
    m.save_bspd1(p)
    host = hs.load_matrix(p)
    assert host.values.tobytes() == m.download().tobytes()
    d = hs.DeviceMatrix.load_bspd1(rt, p)
    rhs = torch.from_numpy(hs.generate_rhs(n, b, 42).values).cuda()
    x1, x2 = torch.zeros_like(rhs), torch.zeros_like(rhs)
    cfg = hs.SolverConfig(block_size=b, eps=1e-6)
    s1 = hs.solve_cg_device(rt, m, rhs.data_ptr(), x1.data_ptr(), cfg)
    s2 = hs.solve_cg_device(rt, d, rhs.data_ptr(), x2.data_ptr(), cfg)
    assert s1.iterations == s2.iterations and s1.converged
    assert torch.equal(x1, x2)  # same bytes in, deterministic kernels
    m.free()
    d.free()
