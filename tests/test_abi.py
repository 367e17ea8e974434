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


def test_shapes_beyond_the_draw_counter_or_int32_slab_rows_are_rejected():
    """The draw counter (reading R6) holds the global row and the plane column / 4 in 32-bit
    words, and slab rows are int32 in the kernels: L_rows > 2^32, L_cols > 2^35 and slab rows
    > 2^30 must be ARG errors from every constructor, before any device call (no GPU here)."""
    big_rows = [(1 << 33, 64, 1), (1 << 31, 64, 1), ((1 << 31) + 2, 64, 1)]  # R >= 2^31
    big_cols = [(64, 1 << 36, 1), (64, (1 << 35) + 64, 1)]                # M > 2^35
    slab_rows = [((1 << 30) + 2, 64, 1), (1 << 32, 64, 2)]               # R > 2^30
    for N, M, n in big_rows + big_cols + slab_rows:
        with pytest.raises(ising.IsingError) as ei:
            ising.ising_create(N, M, 1, n)
        assert ei.value.status == ising.ISING_ERR_ARG, (N, M, n)
        with pytest.raises(ising.IsingError) as ei:
            ising.ising_create_rank_p2p(N, M, 1, 0, n, 0)
        assert ei.value.status == ising.ISING_ERR_ARG, (N, M, n)
        with pytest.raises(ising.IsingError) as ei:
            ising.ising_create_rank(N, M, 1, 0, 1, 0, None)
        assert ei.value.status == ising.ISING_ERR_ARG, (N, M)
        with pytest.raises(ising.IsingError) as ei:
            ising.ising_create_rank_lsa(N, M, 1, 0, 1, 0, None)
        assert ei.value.status == ising.ISING_ERR_ARG, (N, M)
    # 2^32 rows in 4 slabs of 2^30 is within every limit: it gets past the shape check and
    # fails only at the device (none here)
    with pytest.raises(ising.IsingError) as ei:
        ising.ising_create(1 << 32, 64, 1, 4)
    assert ei.value.status in (ising.ISING_ERR_CUDA, ising.ISING_ERR_DEVICE)
    for N, M in [(1 << 33, 64), (64, 1 << 36), ((1 << 32) + 2, 64)]:
        with pytest.raises(ising.IsingError) as ei:
            ising.ising_create_basic(N, M, 1, 0)
        assert ei.value.status == ising.ISING_ERR_ARG, (N, M)


def test_connect_local_argument_errors():
    lib = ising.load()
    assert lib.ising_p2p_connect_local(None, 2) == ising.ISING_ERR_ARG
    arr = (ising._VP * 2)(None, None)
    assert lib.ising_p2p_connect_local(arr, 2) == ising.ISING_ERR_ARG
    assert lib.ising_p2p_connect_local(arr, 0) == ising.ISING_ERR_ARG
    assert lib.ising_p2p_connect_local(arr, 9) == ising.ISING_ERR_ARG


def test_batch_shape_rules_without_gpu():
    # ising_batch_create validates the shape (one CTA, or a cluster of <= 16 CTAs whose row
    # bands + halos fit 200 KB each) before any device call
    for N, M in [(63, 64), (64, 96), (64, 32), (4096, 4096), (2048, 4096), (3, 8192), (0, 64),
                 (2, 65536)]:  # (2, 65536): more column pairs per row than a CTA has threads
        with pytest.raises(ising.IsingError) as ei:
            ising.IsingBatch(N, M, [1])
        assert ei.value.status == ising.ISING_ERR_ARG, (N, M)
    with pytest.raises(ising.IsingError) as ei:
        ising.IsingBatch(64, 64, [])          # no lattices
    assert ei.value.status == ising.ISING_ERR_ARG
    import torch

    if not torch.cuda.is_available():         # valid shapes reach the device: an error here
        for N, M in [(64, 64), (640, 640), (1024, 1024), (2048, 2048)]:
            with pytest.raises(ising.IsingError) as ei:
                ising.IsingBatch(N, M, [1, 2])
            assert ei.value.status in (ising.ISING_ERR_CUDA, ising.ISING_ERR_DEVICE), (N, M)


def test_batch_calls_reject_null_handles_without_gpu():
    lib = ising.load()
    assert lib.ising_batch_destroy(None) == ising.ISING_OK
    assert lib.ising_batch_create(None, 64, 64, 1, None, 0) == ising.ISING_ERR_ARG
    assert lib.ising_batch_set_beta(None, None, 0) == ising.ISING_ERR_ARG
    assert lib.ising_batch_init_random(None) == ising.ISING_ERR_ARG
    assert lib.ising_batch_init_cold(None) == ising.ISING_ERR_ARG
    assert lib.ising_batch_sweep(None, 1) == ising.ISING_ERR_ARG
    assert lib.ising_batch_sweep_measure(None, 1, 1, None, None) == ising.ISING_ERR_ARG
    assert lib.ising_batch_observables(None, None, None) == ising.ISING_ERR_ARG
    assert lib.ising_batch_read_lattice(None, 0, None, 0) == ising.ISING_ERR_ARG
    assert lib.ising_batch_write_lattice(None, 0, None, 0, 0) == ising.ISING_ERR_ARG
    assert lib.ising_batch_last_sweep_ms(None, None) == ising.ISING_ERR_ARG
    assert lib.ising_batch_get_sweep(None, None) == ising.ISING_ERR_ARG


def test_every_handle_call_rejects_a_null_handle():
    # every exported call that takes a handle returns ISING_ERR_ARG for NULL (destroy: a no-op),
    # with NULL / zero for the remaining arguments — no crash, no device access
    import ctypes

    lib = ising.load()
    no_handle = {"ising_create", "ising_create_slabs", "ising_create_rank", "ising_nccl_unique_id",
                 "ising_create_rank_p2p", "ising_create_rank_lsa", "ising_create_basic",
                 "ising_probe_philox", "ising_strerror", "ising_last_error", "ising_batch_create",
                 "ising_p2p_connect_local"}
    for name, (_, args) in ising.SIGNATURES.items():
        if name in no_handle:
            continue
        vals = [None if (a is ctypes.c_void_p or (isinstance(a, type) and issubclass(a, ctypes._Pointer)))
                else 0 for a in args]
        want = ising.ISING_OK if name.endswith("destroy") else ising.ISING_ERR_ARG
        assert getattr(lib, name)(*vals) == want, name
