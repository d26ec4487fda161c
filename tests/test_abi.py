"""C-ABI library: builds for sm_100a, loads, exports every symbol include/s3bfs.h declares,
and rejects bad arguments on the host (CPU only -- no compute call needs a GPU here)."""
import ctypes
import os
import re
import subprocess

import pytest

import paper_2209_08764_b200 as pkg
from paper_2209_08764_b200 import build as cuda_build

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "s3bfs.h")


def declared_functions():
    text = open(HEADER).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(s3bfs_[a-z_0-9]+)\s*\(", text)))


@pytest.fixture(scope="module")
def lib():
    cuda_build.build()
    return pkg.load()


def test_header_declares_the_north_star_calls():
    names = declared_functions()
    for must in ("s3bfs_create", "s3bfs_run", "s3bfs_destroy"):
        assert must in names


def test_library_exports_every_declared_symbol(lib):
    out = subprocess.check_output(["nm", "-D", "--defined-only", pkg.LIB_PATH], text=True)
    exported = {line.split()[-1] for line in out.splitlines() if line.strip()}
    missing = [f for f in declared_functions() if f not in exported]
    assert not missing, missing
    for f in declared_functions():
        assert hasattr(lib, f)
    assert set(pkg.EXPORTED) <= set(declared_functions())


def test_sm100a_sass_present_and_no_atomics_on_discovery_path(lib):
    sass = subprocess.check_output(["cuobjdump", "-sass", pkg.LIB_PATH], text=True)
    assert "sm_100a" in subprocess.check_output(["cuobjdump", "-lelf", pkg.LIB_PATH], text=True) \
        or "arch = sm_100a" in sass
    funcs = {}
    cur = None
    for line in sass.splitlines():
        m = re.search(r"Function : (\S+)", line)
        if m:
            cur = m.group(1)
            funcs[cur] = []
        elif cur:
            funcs[cur].append(line)
    explore = [k for k in funcs if "k_explore" in k]
    small = [k for k in funcs if "k_small" in k]
    assert explore and small
    # P:15 "no locks and atomic-instructions" (DESIGN R17): the discovery kernel k_explore
    # has no atomic instruction at all; the single-CTA tier k_small only publishes visited
    # bits of already-deduplicated vertices with an OR (no counter, CAS or exchange).
    for k in explore + small:
        ops = []
        for line in funcs[k]:
            m = re.search(r"\*/\s+(?:@!?U?P\w+\s+)?([A-Z][A-Z0-9_.]*)", line)
            if m:
                ops.append(m.group(1))
        assert ops, k
        atomics = sorted({op for op in ops if op.split(".")[0] in
                          ("ATOM", "ATOMG", "ATOMS", "RED", "REDG")})
        if k in explore:
            assert not atomics, (k, atomics)
        else:
            assert all(".OR" in op for op in atomics), (k, atomics)


def test_status_strings(lib):
    assert pkg.s3bfs_status_string(0) == "ok"
    assert pkg.s3bfs_status_string(1) == "invalid argument"
    assert pkg.s3bfs_status_string(99) == "unknown status"


def test_host_side_argument_rejection(lib):
    h = ctypes.c_void_p()
    # n <= 0, nnz < 0, NULL pointers: rejected before any device work (S:81 style errors)
    assert lib.s3bfs_create(ctypes.byref(h), 0, 0, 1, 1, None, None) == 1
    assert lib.s3bfs_create(ctypes.byref(h), 4, -1, 1, 1, None, None) == 1
    assert lib.s3bfs_create(ctypes.byref(h), 4, 3, None, None, None, None) == 1
    assert lib.s3bfs_create(None, 4, 3, 1, 1, None, None) == 1
    assert h.value is None
    # host memory is not device memory: rejected, no CPU fallback
    buf = (ctypes.c_int32 * 8)()
    assert lib.s3bfs_create(ctypes.byref(h), 4, 3, ctypes.addressof(buf), ctypes.addressof(buf),
                            None, None) == 1
    assert lib.s3bfs_run(None, 0, None, None, None) == 1
    assert lib.s3bfs_destroy(None) == 0
    assert lib.s3bfs_debug_exclusive_scan(None, None, 5, None) == 1
    assert lib.s3bfs_debug_find_start_points(None, 1, 1, 1, None, None, None) == 1
    msg = ctypes.c_char_p()
    assert lib.s3bfs_last_error(None, ctypes.byref(msg)) == 0 and msg.value


def test_product_path_never_touches_the_oracle():
    """Only tests/, __graft_entry__.smoke() and bench.py's CPU legs may use oracle/: the
    package and the experiment scripts never import or link it (any import form)."""
    imp = re.compile(r"^\s*(from\s+oracle\b|import\s+[^\n#]*\boracle\b)", re.M)
    for d in ("paper_2209_08764_b200", "scripts", "include"):
        for dirpath, _, files in os.walk(os.path.join(ROOT, d)):
            for f in files:
                if f.endswith((".py", ".cu", ".cuh", ".h", ".cpp", ".sh")):
                    text = open(os.path.join(dirpath, f)).read()
                    assert not imp.search(text), os.path.join(dirpath, f)
                    assert "s3bfs_oracle" not in text and "liboracle" not in text, f


def test_options_struct_matches_header():
    # the ctypes mirror must list the header's int32 fields in the header's order
    hdr = open(HEADER).read()
    body = hdr[hdr.index("typedef struct {\n  int32_t edges_per_cta"):]
    body = body[: body.index("} s3bfs_options;")]
    names = re.findall(r"int32_t\s+(\w+);", re.sub(r"/\*.*?\*/", "", body, flags=re.S))
    assert [f[0] for f in pkg.Options._fields_] == names
    assert ctypes.sizeof(pkg.Options) == len(names) * 4
    assert ctypes.sizeof(pkg.LevelStat) == 8 * 4 + 4 * 8
