"""The C-ABI library builds for sm_100a, loads, and exports every symbol the header declares."""
import os
import re
import subprocess

from paper_2402_19481_b200 import _native as N

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "pp_b200.h")


def declared():
    src = open(HEADER).read()
    return sorted(set(re.findall(r"PP_API\s+[\w\s\*]+?\b(pp_\w+)\s*\(", src)))


def test_header_declares_the_boundary():
    names = declared()
    for must in ("pp_runner_create", "pp_runner_step", "pp_runner_sample", "pp_run_sampling",
                 "pp_conv2d_region", "pp_partition_rows", "pp_derive_patch_spec",
                 "pp_last_error"):
        assert must in names


def test_library_exports_every_declared_symbol():
    lib = N.lib()
    missing = [n for n in declared() if not hasattr(lib, n)]
    assert not missing, missing
    out = subprocess.run(["nm", "-D", "--defined-only", N.LIB_PATH], capture_output=True,
                         text=True).stdout
    exported = {ln.split()[-1] for ln in out.splitlines() if " T " in ln}
    assert set(declared()) <= exported
    # nothing but the C ABI is exported (hidden visibility for the C++ internals)
    assert all(s.startswith("pp_") or not s.startswith("_ZN2pp") for s in exported)


def test_python_binding_covers_the_header():
    assert set(declared()) <= set(N.SIGNATURES)


def test_cubin_is_sm100a_with_tcgen05_and_tma():
    sass = subprocess.run(["cuobjdump", "-sass", N.LIB_PATH], capture_output=True, text=True).stdout
    assert "sm_100a" in subprocess.run(["cuobjdump", "-lelf", N.LIB_PATH], capture_output=True,
                                       text=True).stdout or "sm_100" in sass
    assert "UTCHMMA" in sass or "UTCQMMA" in sass or "UTCMMA" in sass   # tcgen05.mma
    assert "UTMALDG" in sass                                             # TMA tensor loads
    assert "LDTM" in sass                                                # tcgen05.ld
    assert "HMMA" not in sass.replace("UTCHMMA", "")                     # no legacy mma.sync


def test_version_and_error_plumbing():
    lib = N.lib()
    assert lib.pp_version() >= 1
    rc = lib.pp_partition_rows(8, 3, 8, None)
    assert rc == N.PP_EINVAL
    assert "not divisible" in N.last_error()
