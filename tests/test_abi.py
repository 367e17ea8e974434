"""CPU-side checks of the C-ABI boundary: the library loads, exports every symbol
include/ising.h declares, and reports errors without a GPU."""
import os
import re

import pytest

from paper_1906_06297_b200 import ising

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def declared_functions():
    src = open(os.path.join(ROOT, "include", "ising.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(ising_[a-z0-9_]+)\s*\(", src)))


def test_header_declares_the_north_star_calls():
    names = declared_functions()
    for call in ["ising_create", "ising_set_beta", "ising_init_random", "ising_init_cold",
                 "ising_sweep", "ising_read_lattice", "ising_observables", "ising_destroy"]:
        assert call in names


def test_library_exports_every_declared_symbol():
    lib = ising.load()
    for name in declared_functions():
        assert hasattr(lib, name), name
    assert set(declared_functions()) == set(ising.SIGNATURES)


def test_library_is_sm100a_only():
    # the cubin inside libising.so targets sm_100a (no PTX / other-arch fallback)
    import subprocess

    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", ising.LIB_PATH],
                         capture_output=True, text=True)
    if out.returncode != 0:
        pytest.skip("cuobjdump unavailable")
    assert "sm_100a" in out.stdout
    arches = set(re.findall(r"sm_\d+a?", out.stdout))
    assert arches == {"sm_100a"}, arches


def test_errors_without_gpu_or_with_bad_args():
    lib = ising.load()
    assert lib.ising_strerror(ising.ISING_ERR_ARG) == b"invalid argument"
    assert lib.ising_destroy(None) == ising.ISING_OK
    # shape validation happens before any device call
    for N, M, n in [(63, 64, 1), (64, 48, 1), (64, 64, 3), (2, 64, 2), (0, 64, 1)]:
        with pytest.raises(ising.IsingError) as ei:
            ising.ising_create(N, M, 1, n)
        assert ei.value.status == ising.ISING_ERR_ARG
    with pytest.raises(ising.IsingError) as ei:
        ising.ising_create(64, 64, 1, 0)
    assert ei.value.status == ising.ISING_ERR_ARG


def test_no_device_is_an_error_not_a_fallback():
    import torch

    if torch.cuda.is_available():
        pytest.skip("GPU present")
    with pytest.raises(ising.IsingError) as ei:
        ising.ising_create(64, 64, 1, 1)
    assert ei.value.status in (ising.ISING_ERR_CUDA, ising.ISING_ERR_DEVICE)
