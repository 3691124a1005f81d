"""C-ABI library: loads on a CPU-only host and exports every entry point
declared in include/he_rotfree.h (no compute calls without a GPU)."""
import ctypes
import os
import re
import subprocess

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HDR = os.path.join(ROOT, "include", "he_rotfree.h")
LIB = os.path.join(ROOT, "paper_2409_05205_b200", "libhe_rotfree.so")


def declared():
    src = open(HDR).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(he_[a-z0-9_]+)\s*\(", src)))


def test_library_builds_and_exports_header_symbols():
    from paper_2409_05205_b200 import build
    build.build()
    lib = ctypes.CDLL(LIB)
    names = declared()
    assert len(names) >= 19
    for n in names:
        assert hasattr(lib, n), n


def test_binding_covers_header():
    import paper_2409_05205_b200 as he
    assert sorted(he.EXPORTED) == declared()


def test_status_strings():
    import paper_2409_05205_b200 as he
    for s in range(6):
        assert he._lib.he_status_str(s).decode().startswith("HE_")


def test_sass_is_sm100a():
    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", LIB],
                         capture_output=True, text=True).stdout
    assert "sm_100a" in out


def _create(primes, log2N, t=65537):
    import paper_2409_05205_b200 as he
    arr = (ctypes.c_uint64 * len(primes))(*primes)
    r = he.RingDesc(log2N, len(primes),
                    ctypes.cast(arr, ctypes.POINTER(ctypes.c_uint64)), t)
    h = ctypes.c_void_p()
    st = he._lib.he_ctx_create(ctypes.byref(r), 0, ctypes.byref(h))
    if st == he.HE_OK:
        he._lib.he_ctx_destroy(h)
    return st


def test_ring_validation_host_side():
    """Parameter checks run before any CUDA call: on a GPU-less host valid
    rings get as far as the device step (HE_ECUDA), invalid ones HE_EPARAM."""
    import torch
    import paper_2409_05205_b200 as he
    import synth
    ok = he.HE_OK if torch.cuda.is_available() else he.HE_ECUDA
    for cfg in synth.CONFIGS.values():
        assert _create(list(cfg.primes), cfg.log2N, cfg.t) == ok
    assert _create([7681, 12289], 8) == ok
    assert _create([7681, 7681], 8) == he.HE_EPARAM          # duplicate
    assert _create([7683], 8) == he.HE_EPARAM                # composite
    assert _create([7681], 9) == he.HE_EPARAM                # != 1 mod 2N
    assert _create([(1 << 50) + 1], 8) == he.HE_EPARAM       # >= 2^50
    assert _create([7681], 8, t=65536) == he.HE_EPARAM       # t even
    assert _create([7681], 7) == he.HE_EPARAM                # N too small
    assert _create([7681], 16) == he.HE_EPARAM               # N too large
