"""CPU-side checks of the C ABI: the library loads, exports every symbol the
header declares, and its GPU-free host logic (slab split, layout, state
machine, error reporting) behaves as include/gscl.h documents.  No kernels run."""
from __future__ import annotations

import ctypes
import os
import re

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def G():
    from paper_1207_1746_b200 import build
    build.build()
    from paper_1207_1746_b200 import gscl
    return gscl


def _declared():
    src = open(os.path.join(ROOT, "include", "gscl.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(gscl_[a-z0-9_]+)\s*\(", src)))


def test_header_declares_the_north_star_calls():
    names = _declared()
    for n in ["gscl_grid_create", "gscl_grid_destroy", "gscl_do_all", "gscl_do_reduce",
              "gscl_halo_exchange", "gscl_jacobi_run", "gscl_init", "gscl_finalize"]:
        assert n in names


def test_every_declared_symbol_is_exported(G):
    lib = ctypes.CDLL(G.LIB_PATH)
    missing = [n for n in _declared() if not hasattr(lib, n)]
    assert not missing, missing


def test_binding_names_match_header(G):
    # the thin binding wraps exactly the header's entry points (no extra compute paths)
    declared = set(_declared())
    import inspect
    src = inspect.getsource(G)
    used = set(re.findall(r"\b(gscl_[a-z0-9_]+)\b", src))
    assert used <= declared | {"gscl_error"}, used - declared


def test_library_is_sm100a_only():
    so = os.path.join(ROOT, "paper_1207_1746_b200", "libgscl.so")
    import subprocess
    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", so], capture_output=True,
                         text=True).stdout
    archs = set(re.findall(r"sm_(\d+a?)", out))
    assert archs == {"100a"}, archs


def test_sass_uses_tma_and_mbarrier():
    so = os.path.join(ROOT, "paper_1207_1746_b200", "libgscl.so")
    import subprocess
    sass = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "-sass", so], capture_output=True,
                          text=True).stdout
    assert "UTMALDG" in sass, "TMA loads (cp.async.bulk.tensor) missing from the sweep kernels"
    assert "SYNCS" in sass, "mbarrier operations missing"


def test_sweep_kernels_never_contract_to_fma():
    # DESIGN.md R3: every + - * of the trees is a separate IEEE operation.
    so = os.path.join(ROOT, "paper_1207_1746_b200", "libgscl.so")
    import subprocess
    sass = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "-sass", so], capture_output=True,
                          text=True).stdout
    funcs = re.split(r"\n\s*Function : ", sass)[1:]
    sweeps = [f for f in funcs if "sweep" in f.split("\n", 1)[0]]
    assert len(sweeps) >= 24
    for f in sweeps:
        name = f.split("\n", 1)[0]
        # LAP27 (op 3) and RESID27 (op 4, rv 1) divide by 30: the correctly rounded
        # IEEE division routine uses FMA internally; its result is still exact-RN.
        # (also the fp32 JACOBI27 two-sweep pass with its RESID27 check, rv 1)
        if "ILi3E" in name or "ILi4ELi1E" in name or "sweep2k_tmaILi1Ef" in name:
            continue
        assert not re.search(r"\b(DFMA|FFMA)\b", f), name


@pytest.mark.parametrize("nz,P", [(10, 4), (512, 1), (768, 8), (7, 3), (1024, 8)])
def test_slab_rule(G, nz, P):
    bounds = [G.slab_range(nz, r, P) for r in range(P)]
    assert bounds[0][0] == 0 and bounds[-1][1] == nz
    for (a0, a1), (b0, _) in zip(bounds, bounds[1:]):
        assert a1 == b0
    sizes = [b - a for a, b in bounds]
    rem = nz % P
    assert sizes == [nz // P + (1 if r < rem else 0) for r in range(P)]


def test_layout_bytes(G):
    # fp64 512^3 halo 1: pitch = round_up(16+512+1, 16) = 544; 514 rows; 514 planes
    assert G.grid_bytes(512, 512, 512, 1, G.F64) == 544 * 514 * 514 * 8
    # fp32: origin offset 32 floats (128 B); pitch = round_up(32+512+1, 32) = 576
    assert G.grid_bytes(512, 512, 512, 1, G.F32) == 576 * 514 * 514 * 4
    # halo 0 coefficient grid: pitch = round_up(16+768, 16) = 784
    assert G.grid_bytes(768, 768, 768, 0, G.F64) == 784 * 768 * 768 * 8
    # slab of rank 3 of 8 at 768 planes: 96 planes + 2 halo planes
    assert G.grid_bytes(768, 768, 768, 1, G.F64, 3, 8) == 800 * 770 * 98 * 8


def test_layout_errors(G):
    with pytest.raises(G.GsclError) as e:
        G.grid_bytes(0, 4, 4, 1)
    assert e.value.name == "GSCL_E_INVALID_DOMAIN"
    with pytest.raises(G.GsclError) as e:
        G.grid_bytes(4, 4, 4, 17)
    assert e.value.name == "GSCL_E_INVALID_DOMAIN"
    with pytest.raises(G.GsclError) as e:
        G.grid_bytes(4, 4, 3, 1, G.F64, 3, 4)  # rank 3 of 4 gets no plane
    assert e.value.name == "GSCL_E_INVALID_DOMAIN"


def test_state_machine_before_init(G):
    lib = G.lib
    h = ctypes.c_void_p()
    assert lib.gscl_grid_create(4, 4, 4, 1, 0, ctypes.byref(h)) == 8  # GSCL_E_STATE
    assert b"gscl_init" in lib.gscl_last_error()
    assert lib.gscl_sync() == 8
    assert lib.gscl_finalize() == 8
    assert lib.gscl_do_all(2, None, 1, None, None, None, 0) == 8
    assert lib.gscl_jacobi_run(2, None, None, None, 0, 1, 0, None) == 8
    n = ctypes.c_size_t()
    assert lib.gscl_peer_export(None, None, None, 0, ctypes.byref(n)) == 8
    assert lib.gscl_peer_import(None, None, None, 0) == 8
    assert lib.gscl_do_all_pass2(2, None, None, None, 1, 1, None) == 8
    it, conv = ctypes.c_int(), ctypes.c_int()
    assert lib.gscl_converge_run(0, None, None, 1e-6, 10, 1, ctypes.byref(it), ctypes.byref(conv)) == 8


def test_pass_units_host_side(G):
    # boundary units per side of a two-sweep pass = its x-y tiles: 60 x 28
    # output tiles for fp64 (V = 2), 120 x 28 for fp32 (V = 4)
    assert G.pass_units(512, 512) == 9 * 19
    assert G.pass_units(512, 512, G.F32) == 5 * 19
    assert G.pass_units(60, 28) == 1 and G.pass_units(61, 29) == 4
    with pytest.raises(G.GsclError):
        G.pass_units(0, 5)


def test_init_without_gpu_fails_cleanly(G):
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    st = G.lib.gscl_init(0, 1, None, 0, None)
    assert st == 10  # GSCL_E_CUDA, returned, not aborted
    assert G.lib.gscl_last_error()
    assert G.lib.gscl_sync() == 8  # still not initialised


def test_init_argument_validation(G):
    assert G.lib.gscl_init(2, 2, None, 0, None) == 1  # rank out of range
    # world > 1 without an NCCL id is valid (peer-memory transport only); with
    # no GPU it fails later, at the device, never with OK
    import torch
    if torch.cuda.is_available():
        return  # (on a GPU box that init is legitimate)
    assert G.lib.gscl_init(0, 2, None, 0, None) != 0


def test_version(G):
    assert "sm_100a" in G.version()
