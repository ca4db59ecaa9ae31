"""The C++ shim (include/hsolve/*.hpp, libhsolve_b200.so) builds against
unchanged reference-style caller code and passes reference assertions."""
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
PKG = os.path.join(ROOT, "paper_2605_13209_b200")


def _build(tmp_path):
    exe = str(tmp_path / "test_hsolve_api")
    subprocess.run(["g++", "-std=c++20", "-O1", "-I", os.path.join(ROOT, "include"),
                    os.path.join(ROOT, "tests", "cpp", "test_hsolve_api.cpp"), "-o", exe,
                    "-L", PKG, "-lhsolve_b200", "-lhsolve_cuda", f"-Wl,-rpath,{PKG}"],
                   check=True)
    return exe


def test_cpp_shim_compiles(tmp_path):
    if not os.path.exists(os.path.join(PKG, "libhsolve_b200.so")):
        pytest.skip("shim not built")
    assert os.path.exists(_build(tmp_path))


@pytest.mark.gpu
def test_cpp_shim_runs_reference_assertions(tmp_path):
    exe = _build(tmp_path)
    out = subprocess.run([exe], capture_output=True, text=True, timeout=300)
    print(out.stdout)
    assert out.returncode == 0 and "ALL PASSED" in out.stdout, out.stdout + out.stderr


def _build_io(tmp_path):
    exe = str(tmp_path / "test_io_cli")
    subprocess.run(["g++", "-std=c++20", "-O1", "-I", os.path.join(ROOT, "include"),
                    os.path.join(ROOT, "tests", "cpp", "test_io_cli.cpp"), "-o", exe,
                    "-L", PKG, "-lhsolve_b200", "-lhsolve_cuda", f"-Wl,-rpath,{PKG}"],
                   check=True)
    return exe


def test_cpp_matrix_io_and_cli_host_part(tmp_path):
    """matrix_io.hpp / bench.hpp drop-in: format, error kinds, usage errors
    (no GPU needed)."""
    if not os.path.exists(os.path.join(PKG, "libhsolve_b200.so")):
        pytest.skip("shim not built")
    out = subprocess.run([_build_io(tmp_path)], capture_output=True, text=True, timeout=300)
    assert out.returncode == 0 and "ALL PASSED" in out.stdout, out.stdout + out.stderr


@pytest.mark.gpu
def test_cpp_matrix_io_and_cli_gpu_part(tmp_path):
    out = subprocess.run([_build_io(tmp_path), "--gpu"], capture_output=True, text=True,
                         timeout=600)
    assert out.returncode == 0 and "ALL PASSED" in out.stdout, out.stdout + out.stderr


@pytest.mark.gpu
def test_cpp_multigpu_runtime(tmp_path):
    """SolverConfig::gpus = 2 through the reference API (in-process transport
    on a one-GPU box, NCCL with two GPUs)."""
    exe = str(tmp_path / "test_hsolve_multigpu")
    subprocess.run(["g++", "-std=c++20", "-O1", "-I", os.path.join(ROOT, "include"),
                    os.path.join(ROOT, "tests", "cpp", "test_hsolve_multigpu.cpp"), "-o", exe,
                    "-L", PKG, "-lhsolve_b200", "-lhsolve_cuda", f"-Wl,-rpath,{PKG}"],
                   check=True)
    out = subprocess.run([exe], capture_output=True, text=True, timeout=600)
    print(out.stdout)
    assert out.returncode == 0 and "ALL PASSED" in out.stdout, out.stdout + out.stderr


def _build_named(tmp_path, name):
    exe = str(tmp_path / name)
    subprocess.run(["g++", "-std=c++20", "-O1", "-ffp-contract=off", "-I",
                    os.path.join(ROOT, "include"),
                    os.path.join(ROOT, "tests", "cpp", name + ".cpp"), "-o", exe,
                    "-L", PKG, "-lhsolve_b200", "-lhsolve_cuda", f"-Wl,-rpath,{PKG}"],
                   check=True)
    return exe


def test_cpp_block_kernels_api_compiles(tmp_path):
    """block_kernels.hpp / dd.hpp drop-in headers compile against the shim."""
    if not os.path.exists(os.path.join(PKG, "libhsolve_b200.so")):
        pytest.skip("shim not built")
    assert os.path.exists(_build_named(tmp_path, "test_block_kernels_api"))


@pytest.mark.gpu
def test_cpp_block_kernels_api(tmp_path):
    """hsolve::kernels on the GPU: the reference's closed forms and bitwise
    agreement with its loops (test_block_kernels.cpp)."""
    out = subprocess.run([_build_named(tmp_path, "test_block_kernels_api")], capture_output=True,
                         text=True, timeout=600)
    print(out.stdout)
    assert out.returncode == 0 and "ALL PASSED" in out.stdout, out.stdout + out.stderr
