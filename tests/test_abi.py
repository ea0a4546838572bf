"""CPU checks of the drop-in boundary: libbmg.so loads, exports exactly what
include/bandmatch_gpu.h declares, and its host-side entry points behave like
the reference's (no compute calls -- there is no GPU here)."""
import ctypes as C
import re
import subprocess
from pathlib import Path

import numpy as np
import pytest

import paper_2505_22089_b200 as bm
from paper_2505_22089_b200 import _lib

ROOT = Path(__file__).resolve().parents[1]
HEADER = ROOT / "include" / "bandmatch_gpu.h"


def declared_symbols():
    text = HEADER.read_text()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(bmg_[a-z0-9_]+)\s*\(", text)))


def test_library_exports_every_declared_symbol():
    lib = _lib.load()
    syms = declared_symbols()
    assert len(syms) >= 30
    for s in syms:
        assert hasattr(lib, s), s
    out = subprocess.run(["nm", "-D", "--defined-only", str(_lib.LIB_PATH)], capture_output=True,
                         text=True).stdout
    exported = set(re.findall(r" T (bmg_\w+)", out))
    assert set(syms) <= exported
    assert set(_lib.EXPORTED) <= exported


def test_library_targets_sm100a():
    out = subprocess.run(["cuobjdump", "--list-elf", str(_lib.LIB_PATH)], capture_output=True,
                         text=True).stdout
    assert "sm_100a" in out


def test_status_names_mirror_reference_codes():
    lib = _lib.load()
    names = [lib.bmg_status_name(i).decode() for i in range(9)]
    assert names == ["Ok", "InvalidArgument", "HashMismatch", "CapacityExceeded", "NotResident",
                     "CudaError", "OutOfMemory", "Unsupported", "InvalidScene"]
    assert lib.bmg_abi_version() == 1


def test_seed_for_and_hash_functions_match_oracle(oracle):
    for root, tag in [(42, "matching"), (0, ""), (2 ** 64 - 1, "hash.fine"), (7, "scene.world")]:
        assert bm.seed_for(root, tag) == oracle.seed_for(root, tag)
    for seed, p in [(bm.seed_for(42, "matching"), (6, 8, 128)), (3, (2, 5, 70)), (9, (1, 32, 1))]:
        hf = bm.make_hash_functions(seed, bm.HashParams(*p))
        c, f = oracle.make_hash_functions(seed, *p)
        assert np.array_equal(hf.coarse.view(np.uint32), c.view(np.uint32))
        assert np.array_equal(hf.fine.view(np.uint32), f.view(np.uint32))


def test_hash_function_errors():
    for p in [(0, 8, 128), (6, 0, 128), (6, 33, 128), (6, 8, 0)]:
        with pytest.raises(bm.BandmatchError) as e:
            bm.make_hash_functions(1, bm.HashParams(*p))
        assert e.value.code == "InvalidArgument"


def test_no_cpu_fallback_without_a_device():
    import torch
    if torch.cuda.is_available():
        pytest.skip("a GPU is present")
    hf = bm.make_hash_functions(1)
    with pytest.raises(bm.BandmatchError) as e:
        bm.Matcher(hf)
    assert e.value.code == "CudaError" and "no CPU fallback" in str(e.value)
    with pytest.raises(bm.BandmatchError):
        bm.compute_codes(bm.FeatureSet(1, np.zeros((2, 128), np.float32)), hf,
                         np.zeros(128, np.float32))


def test_null_arguments_are_rejected_without_crashing():
    lib = _lib.load()
    assert lib.bmg_create(None, None) == 1
    assert lib.bmg_upload(None, 1, None, 0) == 1
    assert lib.bmg_row(None, None, 0, None) == 1
    assert lib.bmg_destroy(None) == 0
    assert lib.bmg_result_pair_count(None) == 0
    assert b"null" in lib.bmg_last_error() or lib.bmg_last_error() != b""
