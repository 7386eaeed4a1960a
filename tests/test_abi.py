"""Boundary checks that need no GPU: the C-ABI library loads, exports every symbol
include/pp_loader.h declares, and rejects bad descriptors without side effects."""
import ctypes
import os
import re

import pytest

import __graft_entry__ as ge

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def pp():
    ge.build()
    import paper_2504_13266_b200 as pp

    return pp


def header_symbols():
    src = open(os.path.join(ROOT, "include", "pp_loader.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(pp_[a-z_0-9]+)\s*\(", src)))


def test_every_header_symbol_exported(pp):
    syms = header_symbols()
    assert len(syms) >= 15
    L = ctypes.CDLL(pp.LIB_PATH)
    for s in syms:
        assert hasattr(L, s), s
    from paper_2504_13266_b200 import _abi

    assert sorted(_abi.EXPORTS) == syms


def test_built_for_sm100a(pp):
    import subprocess

    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", pp.LIB_PATH], capture_output=True, text=True)
    assert "sm_100a" in out.stdout


def _header_define(name):
    import re

    hdr = open(os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "include",
                            "pp_loader.h")).read()
    return int(re.search(rf"#define {name} (\d+)", hdr).group(1))


def test_abi_version_and_footprint(pp):
    assert pp.pp_abi_version() == _header_define("PP_ABI_VERSION") == 6
    assert pp.IPC_HANDLE_BYTES == _header_define("PP_IPC_HANDLE_BYTES") == 256
    assert pp.NCCL_ID_BYTES == _header_define("PP_NCCL_ID_BYTES") == 128
    # input expansion K(R+1)x: 400 GB at R = 3, K = 1 -> 1.6 TB
    n = 100_000_000
    assert pp.pp_footprint_bytes(n, 1000, 4, 1, 0) == 400 * 10**9
    assert pp.pp_footprint_bytes(n, 1000, 4, 1, 3) == 1600 * 10**9
    assert pp.pp_footprint_bytes(-1, 1, 1, 1, 1) == -1


@pytest.mark.parametrize("kw,msg", [
    (dict(batch_size=0), "batch_size"),
    (dict(num_nodes=0), "num_nodes"),
    (dict(num_hops=0), "num_hops"),
    (dict(out_dtype=1, dtype=2), "dtype pair"),
    (dict(world_size=2, rank=0, peers=0), "peers"),
    (dict(world_size=1, rank=1), "rank"),
    (dict(node_set=[0, 5, 10]), "out of range"),
    (dict(peers=3), "nccl_unique_id"),
    (dict(peers=1), "world_size == 1"),
    (dict(peers=7), "unknown peers"),
])
def test_invalid_descriptors(pp, kw, msg):
    base = dict(num_nodes=10, num_hops=2, feat_dim=4, batch_size=2)
    base.update(kw)
    with pytest.raises(pp.PPError) as ei:
        pp.pp_loader_create(**base)
    assert ei.value.status == pp.PP_ERR_INVALID
    assert msg in str(ei.value)


def test_null_handle_calls(pp):
    lib = pp.lib()
    assert lib.pp_epoch_permute(None, 1, 1, None) == pp.PP_ERR_INVALID
    assert lib.pp_next_batch(None, None, None, None, None, None) == pp.PP_ERR_INVALID
    assert lib.pp_loader_destroy(None) == pp.PP_OK
    assert b"NULL" in lib.pp_last_error()


def test_product_package_never_imports_oracle():
    pkg = os.path.join(ROOT, "paper_2504_13266_b200")
    for dirpath, _, files in os.walk(pkg):
        for f in files:
            if f.endswith((".py", ".cu", ".cuh", ".h", ".cpp")):
                text = open(os.path.join(dirpath, f)).read()
                assert "oracle" not in re.sub(r"(#|//).*", "", text).replace("oracle/", ""), f


def test_struct_layouts_match_header(tmp_path):
    # the ctypes mirrors must have the header's exact layout (sizes and field offsets), checked by
    # compiling a probe against include/pp_loader.h with the host C compiler
    import ctypes
    import shutil
    import subprocess

    from paper_2504_13266_b200 import _abi

    cc = shutil.which("gcc") or shutil.which("cc")
    if cc is None:
        pytest.skip("no host C compiler")
    structs = {"pp_hop_desc": _abi.pp_hop_desc, "pp_loader_desc": _abi.pp_loader_desc,
               "pp_loader_info": _abi.pp_loader_info}
    lines = ['#include <stdio.h>', '#include <stddef.h>', '#include "pp_loader.h"', "int main(void) {"]
    for name, cls in structs.items():
        lines.append(f'  printf("{name} size %zu\\n", sizeof({name}));')
        for field, _ in cls._fields_:
            lines.append(f'  printf("{name} {field} %zu\\n", offsetof({name}, {field}));')
    lines += ["  return 0;", "}"]
    src = tmp_path / "probe.c"
    src.write_text("\n".join(lines) + "\n")
    exe = tmp_path / "probe"
    subprocess.check_call([cc, "-I", os.path.join(ROOT, "include"), "-o", str(exe), str(src)])
    got = {}
    for line in subprocess.check_output([str(exe)], text=True).splitlines():
        name, what, val = line.split()
        got[(name, what)] = int(val)
    for name, cls in structs.items():
        assert got[(name, "size")] == ctypes.sizeof(cls), name
        for field, _ in cls._fields_:
            assert got[(name, field)] == getattr(cls, field).offset, (name, field)
