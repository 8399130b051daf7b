"""The C-ABI library loads and exports every function include/*.h declares (no GPU needed)."""
import ctypes
import glob
import os
import re

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
LIB = os.path.join(ROOT, "paper_1502_07451_b200", "libhetsched_b200.so")


def declared_functions():
    names = set()
    for h in glob.glob(os.path.join(ROOT, "include", "*.h")):
        text = open(h).read()
        text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
        for m in re.finditer(r"\b(hs_[a-z0-9_]+|METIS_[A-Za-z]+)\s*\(", text):
            names.add(m.group(1))
    return sorted(names)


def test_header_declares_entry_points():
    names = declared_functions()
    for must in ("hs_evaluate2", "hs_simulate_batch", "hs_levels", "hs_fm2", "hs_brute2",
                 "hs_partition_kway", "hs_exact_totals", "hs_last_error",
                 "hs_partition_kway_dist", "hs_symmetrize_range", "hs_kway_dist_arena_bytes",
                 "METIS_PartGraphKway"):
        assert must in names


def test_library_exports_every_declared_symbol():
    lib = ctypes.CDLL(LIB)
    missing = [n for n in declared_functions() if not hasattr(lib, n)]
    assert not missing, f"declared but not exported: {missing}"


def test_library_is_sm100a():
    import subprocess
    out = subprocess.run(["cuobjdump", "--list-elf", LIB], capture_output=True, text=True)
    assert out.returncode == 0, out.stderr
    assert "sm_100a" in out.stdout


def test_status_plumbing_without_gpu():
    lib = ctypes.CDLL(LIB)
    lib.hs_version.restype = ctypes.c_char_p
    assert b"sm_100a" in lib.hs_version()
    lib.hs_simulate_batch.restype = ctypes.c_int
    # null batch -> HS_EINVAL with a message, no device touched
    rc = lib.hs_simulate_batch(None, 0, None, 3, 1, *([None] * 10))
    assert rc == -1
    lib.hs_last_error.restype = ctypes.c_char_p
    assert b"null" in lib.hs_last_error()


def test_sharded_partition_validates_before_touching_the_device():
    lib = ctypes.CDLL(LIB)
    lib.hs_last_error.restype = ctypes.c_char_p
    lib.hs_kway_dist_arena_bytes.restype = ctypes.c_int64
    lib.hs_kway_dist_arena_bytes.argtypes = [ctypes.c_int32]
    assert lib.hs_kway_dist_arena_bytes(10_000_000) >= 24 * 10_000_000
    fn = lib.hs_partition_kway_dist
    fn.restype = ctypes.c_int
    rc = fn(None, 0, 10, None, 2, None, ctypes.c_double(0.03), ctypes.c_uint64(0), None, None,
            None)
    assert rc == -1 and b"null" in lib.hs_last_error()
