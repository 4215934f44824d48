"""C-ABI checks that need no GPU: the library loads, exports every symbol that
include/dsr.h declares, and its host-side layout agrees with what the paper
fixes (the oracle's N_T, columns, block size, block-count bound) and with the
invariants of the parts the paper leaves open."""
import ctypes
import random
import re
from pathlib import Path

import pytest

from conftest import ROOT, split_fields


def declared_functions():
    txt = (ROOT / "include" / "dsr.h").read_text()
    txt = re.sub(r"/\*.*?\*/", "", txt, flags=re.S)
    return sorted(set(re.findall(r"^\s*(?:const\s+)?[a-z_0-9]+\s*\*?\s*(dsr_[a-z_0-9]+)\s*\(", txt, flags=re.M)))


@pytest.fixture(scope="module")
def L():
    from paper_1810_11765_b200 import build, dsr
    build.build()
    return dsr


def test_library_exports_every_declared_symbol(L):
    names = declared_functions()
    assert len(names) >= 20
    lib = ctypes.CDLL(str(L.LIBPATH))
    for n in names:
        assert hasattr(lib, n), n
    assert L.lib().dsr_build_info().startswith(b"sm_100a")


def test_status_strings(L):
    assert L.status_str(L.OK) == "DSR_OK"
    assert L.status_str(L.ERR_OOM) == "DSR_ERR_OOM"


def level_words(n):
    """u64 containers per level of an n-bit hierarchical bitmap."""
    out = []
    while True:
        out.append((n + 63) // 64)
        if n <= 64:
            return out
        n = (n + 63) // 64


def check_gpu_layout(L, O, tf, heap, parents=None):
    """The library's layout against what the paper and the R-LAYOUT reading
    fix (the oracle's or_layout), and against invariants for everything the
    paper leaves to the implementation (where its regions go): same N_T,
    columns and block size; M at most the paper-derived bound and within 1 %
    of it; every region holds its M-sized array, in order, disjoint, inside the
    buffer after the control page; bitmap levels sized per P:501."""
    a = L.layout_compute(tf, heap, parents)
    b = O.layout(tf, heap)
    T = len(tf)
    assert a["cap"] == b["cap"]
    assert [a["col_off"][t][:len(tf[t])] for t in range(T)] == b["col_off"]
    assert a["block_bytes"] == b["block_bytes"]
    M = a["M"]
    assert M <= b["M"]
    assert M >= 0.99 * b["M"] - 8, (M, b["M"], heap)
    assert a["level_words"] == level_words(M) and a["nlevels"] == len(level_words(M))
    assert a["bitmap_words"] >= sum(level_words(M))
    regs = [(a["off_data"], M * a["block_bytes"]), (a["off_alloc_bm"], 8 * M), (a["off_iter_bm"], 8 * M),
            (a["off_type"], M), (a["off_R"], 4 * M), (a["off_bitmaps"], (1 + 2 * T) * a["bitmap_words"] * 8)]
    assert a["off_data"] >= 4096                                          # after the control page
    for (o1, s1), (o2, _) in zip(regs, regs[1:]):
        assert o1 % 256 == 0 and o1 + s1 <= o2
    assert regs[-1][0] + regs[-1][1] <= a["total_bytes"] <= heap
    return a


def test_gpu_layout_within_paper_bounds(L, O):
    rnd = random.Random(11)
    cases = [[[4, 4, 4], [4, 4, 4, 4], [4] * 6], [[4, 1, 1], [4, 1]], [[4, 4, 4], [4, 4, 4, 4], [4, 8, 1, 1, 1, 1, 1]],
             [[4] * 7 + [4, 4, 4, 1]]]
    for _ in range(150):
        T = rnd.randint(1, 8)
        tf = [[rnd.choice([1, 2, 4, 8, 16]) for _ in range(rnd.randint(1, 16))] for _ in range(T)]
        if max(map(sum, tf)) <= 64 * min(map(sum, tf)):
            cases.append(tf)
    for tf in cases:
        for heap in (1 << 20, 123456789, 1 << 31):
            check_gpu_layout(L, O, tf, heap)


def test_inheritance_layout_is_the_flattened_layout(L, O):
    """a subtype's data segment begins with the SOA columns of its
    inherited fields, then its own; so a hierarchy lays out exactly like the
    flattened field lists (the oracle has no notion of a base type)."""
    tf = [[4, 4], [4, 4, 8], [4, 4, 1], [4, 4, 8, 4], [4, 4, 8, 4, 2, 2]]
    parents = [None, 0, 0, 1, 3]
    for heap in (1 << 20, 1 << 28):
        a = check_gpu_layout(L, O, tf, heap, parents)
        assert a == L.layout_compute(tf, heap)


def test_inheritance_rejects_invalid(L):
    with pytest.raises(L.DsrError):
        L.layout_compute([[4, 4], [4, 8, 8]], 1 << 20, [None, 0])      # inherited prefix differs
    with pytest.raises(L.DsrError):
        L.layout_compute([[4, 4, 8], [4, 4]], 1 << 20, [1, None])      # base declared later
    with pytest.raises(L.DsrError):
        L.layout_compute([[4, 4]], 1 << 20, [0])                       # own base


def test_layout_rejects_invalid(L):
    with pytest.raises(ValueError):
        L.layout_compute([[4], [16] * 16 + [4]], 1 << 20)        # > 16 fields (binding)
    with pytest.raises(L.DsrError):
        L.layout_compute([[4], [3]], 1 << 20)                     # field size 3
    with pytest.raises(L.DsrError):
        L.layout_compute([[2], [16] * 9], 1 << 20)                # 144 B > 64 x 2 B
    with pytest.raises(L.DsrError):
        L.layout_compute([[4]], 4096)                             # no room for a block


def test_product_path_fails_loudly_without_gpu(L):
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    with pytest.raises(RuntimeError):
        L.Heap([[4]], 1 << 20)


def test_product_package_never_imports_the_oracle():
    pkg = ROOT / "paper_1810_11765_b200"
    for p in list(pkg.rglob("*.py")) + list(pkg.rglob("*.cu")) + list(pkg.rglob("*.cuh")) + list(pkg.rglob("*.h")):
        txt = p.read_text()
        assert not re.search(r"(^|\n)\s*(from|import)\s+oracle|liboracle|oracle\.h|oracle/", txt), p


def test_binding_ids_and_flags_mirror_the_header():
    """Every DSR_F_* flag and DSR_[MKC]_* id of include/dsr.h has the same
    value under the same name (prefix dropped) in the ctypes binding."""
    import re
    from pathlib import Path
    from paper_1810_11765_b200 import dsr
    hdr = (Path(__file__).resolve().parents[1] / "include" / "dsr.h").read_text()
    found = {}
    for name, val in re.findall(r"#define DSR_(F_[A-Z0-9_]+)\s+(0x[0-9a-fA-F]+)u", hdr):
        found[name] = int(val, 16)
    for name, val in re.findall(r"\bDSR_([MKC]_[A-Z0-9_]+)\s*=\s*(\d+)", hdr):
        found[name] = int(val)
    assert len(found) > 40
    missing = [n for n in found if not hasattr(dsr, n)]
    assert not missing, missing
    wrong = {n: (v, getattr(dsr, n)) for n, v in found.items() if getattr(dsr, n) != v}
    assert not wrong, wrong
