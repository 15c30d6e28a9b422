"""The C-ABI library loads and exports every symbol include/spdp.h declares (CPU-only)."""
import ctypes
import os
import re
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "spdp.h")


def declared_symbols():
    text = open(HEADER).read()
    return sorted(set(re.findall(r"SPDP_API\s+[\w\s\*]+?\b(spdp_\w+)\s*\(", text)))


@pytest.fixture(scope="module")
def spdp():
    import __graft_entry__
    __graft_entry__.build()
    import paper_2511_18022_b200 as m
    return m


def test_header_declares_the_north_star_entry_points():
    syms = declared_symbols()
    for name in ("spdp_split_eval", "spdp_split_eval_batch", "spdp_saa_mean", "spdp_irp_dp"):
        assert name in syms


def test_library_exports_every_declared_symbol(spdp):
    lib = ctypes.CDLL(spdp.LIB_PATH)
    for name in declared_symbols():
        assert hasattr(lib, name), name
    assert set(declared_symbols()) == set(spdp.SYMBOLS)
    out = subprocess.run(["nm", "-D", "--defined-only", spdp.LIB_PATH], capture_output=True, text=True).stdout
    exported = set(re.findall(r"\bT (spdp_\w+)", out))
    assert exported == set(declared_symbols())


def test_library_is_sm100a_only(spdp):
    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", spdp.LIB_PATH], capture_output=True,
                         text=True).stdout
    assert "sm_100a" in out
    assert not re.search(r"sm_(?!100a)\d+", out)


def test_host_only_entry_points(spdp):
    # spdp_saa_mean is host code: exact finalize of a partial, no GPU needed
    p = spdp.SaaPartial(3, 1, 6, 14, 0, 0)  # costs 1, 2, 3 (+1 infeasible)
    e = spdp.SaaEstimate()
    assert spdp.lib().spdp_saa_mean(ctypes.byref(p), ctypes.byref(e)) == 0
    assert (e.m, e.infeasible, e.mean, e.var) == (3, 1, 2.0, 1.0)
    z = spdp.SaaPartial(0, 5, 0, 0, 0, 0)
    assert spdp.lib().spdp_saa_mean(ctypes.byref(z), ctypes.byref(e)) == spdp.SPDP_E_DATA
    assert b"infeasible" in spdp.lib().spdp_last_error()
    assert spdp.workspace_bytes(100, 10**6, 1) > 0
    assert spdp.workspace_bytes(0, 10, 1) == 0


def test_usage_errors_before_any_device_work(spdp):
    L = spdp.lib()
    # NULL pointers / bad sizes are rejected on the host, before touching CUDA
    rc = L.spdp_split_eval(None, None, 10, None, 8, 8, 5, None, None, 0, None, 0, 0, None)
    assert rc == spdp.SPDP_E_USAGE
    rc = L.spdp_split_eval(None, None, 0, None, 8, 8, 5, None, None, 0, None, 0, 0, None)
    assert rc == spdp.SPDP_E_USAGE
    rc = L.spdp_split_eval(None, None, spdp.MAX_N + 1, None, 8, 8, 5, None, None, 0, None, 0, 0, None)
    assert rc == spdp.SPDP_E_RESOURCE


def test_product_never_imports_oracle():
    """The product (package, kernels, header) never imports, includes or links the oracle."""
    pat = re.compile(r"(^\s*(import|from)\s+oracle\b)|liboracle|#\s*include[^\n]*oracle|oracle\.c\b", re.M)
    roots = [os.path.join(ROOT, "paper_2511_18022_b200"), os.path.join(ROOT, "include")]
    for root in roots:
        for dirpath, _, files in os.walk(root):
            for f in files:
                if f.endswith((".py", ".cu", ".cuh", ".h", ".cpp")):
                    text = open(os.path.join(dirpath, f)).read()
                    assert not pat.search(text), os.path.join(dirpath, f)


def test_usage_errors_of_the_next_rows(spdp):
    """f3 / f4 entry points reject bad arguments on the host, before any device work."""
    L = spdp.lib()
    assert L.spdp_split_values(None, None, 10, None, 8, 8, 5, None, None, None, 0, None) == spdp.SPDP_E_USAGE
    assert L.spdp_split_values(None, None, 0, None, 8, 8, 5, None, None, None, 0, None) == spdp.SPDP_E_USAGE
    assert L.spdp_split_eval_neighbours(None, None, None, None, 4, None, 10, None, 8, 8, 5, None, None, 0, None, 0, 0,
                                        None) == spdp.SPDP_E_USAGE
    assert L.spdp_split_eval_neighbours(None, None, None, None, 0, None, 10, None, 8, 8, 5, None, None, 0, None, 0, 0,
                                        None) == spdp.SPDP_E_USAGE
    assert L.spdp_split_eval_limits(None, None, 10, None, 8, 8, 5, -1, 0, None, None, None, 0, 0, None) == spdp.SPDP_E_USAGE
    assert L.spdp_split_eval_limits(None, None, 10, None, 8, 8, 0, -1, 0, None, None, None, 0, 0, None) == spdp.SPDP_E_USAGE
    assert b"Q=0" in L.spdp_last_error()
    assert L.spdp_values_workspace_bytes(0, 5) == 0 and L.spdp_values_workspace_bytes(10, 5) > 0
    assert L.spdp_neighbour_workspace_bytes(10, 5, 0) == 0 and L.spdp_neighbour_workspace_bytes(10, 5, 3) > 0
