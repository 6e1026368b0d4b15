"""The drop-in boundary: libfheconv.so loads and exports every entry point
declared in include/fheconv.h (no compute without a GPU)."""
import ctypes as C
import os
import re
import subprocess

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def header_functions():
    src = open(os.path.join(ROOT, "include", "fheconv.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(fhe_[a-z0-9_]+)\s*\(", src)))


def test_every_declared_symbol_is_exported(product_lib):
    names = header_functions()
    assert len(names) >= 40
    for n in names:
        assert hasattr(product_lib, n), n
    out = subprocess.run(["nm", "-D", "--defined-only", os.path.join(ROOT, "paper_2306_09189_b200", "libfheconv.so")],
                         capture_output=True, text=True, check=True).stdout
    exported = set(re.findall(r"\b(fhe_[a-z0-9_]+)\b", out))
    assert set(names) <= exported


def test_ctypes_binding_covers_header():
    from paper_2306_09189_b200 import _lib
    assert sorted(_lib.EXPORTED) == header_functions()


def test_library_is_sm100a_only():
    lib = os.path.join(ROOT, "paper_2306_09189_b200", "libfheconv.so")
    out = subprocess.run(["cuobjdump", "--list-elf", lib], capture_output=True, text=True).stdout
    assert "sm_100a" in out
    for other in ("sm_80", "sm_90"):
        assert f"{other}." not in out


def test_no_cpu_fallback_without_gpu(product_lib):
    import torch
    if torch.cuda.is_available():
        pytest.skip("a GPU is present")
    from paper_2306_09189_b200 import Context, FheError
    with pytest.raises(FheError) as e:
        Context.from_config("cfg1")
    assert e.value.code == -3  # FHE_E_CUDA


def test_host_decomposition_matches_reference(product_lib, golden):
    from paper_2306_09189_b200 import decompose
    for s in (4096, 8192):
        lens, sums, first = golden[f"decomp{s}/lens"], golden[f"decomp{s}/sums"], golden[f"decomp{s}/steps_lt1024"]
        for strat in (0, 1):
            for n in range(0, s, 7):
                st = decompose(strat, n, s)
                assert len(st) == lens[strat, n] and sum(st) == sums[strat, n]
                if n < 1024:
                    assert st == [int(x) for x in first[strat, n, : len(st)]]
    with pytest.raises(ValueError):
        decompose(0, 4096, 4096)


def test_cxx_wrapper_compiles():
    """include/fheconv.hpp (Engine-shaped C++ wrapper) compiles against the C ABI."""
    src = os.path.join(ROOT, "tests", "cxx", "engine_demo.cpp")
    out = "/tmp/fheconv_engine_demo"
    subprocess.run(["g++", "-std=c++17", "-O1", "-I", os.path.join(ROOT, "include"), src, "-o", out,
                    "-L", os.path.join(ROOT, "paper_2306_09189_b200"), "-lfheconv",
                    f"-Wl,-rpath,{os.path.join(ROOT, 'paper_2306_09189_b200')}"], check=True)
    assert os.path.exists(out)


def test_context_rejects_more_than_eight_digits(product_lib):
    """dnum = ceil(n_q / n_p) > 8 has no keyed-kernel instantiation: rejected up front
    (before any device work), never silently skipped."""
    from paper_2306_09189_b200 import Context, FheError
    with pytest.raises(FheError) as e:
        Context(log_n=13, q_bits=[50] * 9, p_bits=[60], log_scale=40)
    assert e.value.code == -1  # FHE_E_INVALID, not the no-GPU FHE_E_CUDA: the check runs first
