"""The C-ABI library loads and exports every symbol include/rgnn.h declares (no GPU needed)."""
import ctypes
import os
import re

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def declared_functions():
    with open(os.path.join(ROOT, "include", "rgnn.h")) as f:
        src = re.sub(r"/\*.*?\*/", "", f.read(), flags=re.S)
    return sorted(set(re.findall(r"^\s*(?:const\s+)?[a-z_0-9]+\s*\*?\s*(rgnn_\w+|rgcn_\w+|rgat_\w+|hgt_\w+)\s*\(", src, flags=re.M)))


def test_header_declares_the_boundary():
    names = declared_functions()
    for n in ["rgnn_graph_create", "rgcn_forward", "rgat_forward", "rgnn_backward", "rgnn_comm_create"]:
        assert n in names


def test_library_exports_every_declared_symbol():
    lib = ctypes.CDLL(os.path.join(ROOT, "paper_2301_06284_b200", "librgnn.so"))
    for n in declared_functions():
        assert hasattr(lib, n), n


def test_binding_names_match_header():
    from paper_2301_06284_b200 import _binding
    assert sorted(_binding.EXPORTED) == declared_functions()


def test_host_only_entry_points():
    import numpy as np
    import paper_2301_06284_b200 as m
    assert "sm_100a" in m.version()
    b = m.partition_dst(np.r_[0, np.cumsum([5, 0, 1, 1, 9, 2, 2])], 3)
    assert b[0] == 0 and b[-1] == 7 and list(b) == sorted(b)
    # error path without a device: NULL descriptor
    from paper_2301_06284_b200 import _binding as B
    st = B.lib.rgnn_graph_bytes(None, None, None)
    assert st == B.RGNN_E_INVALID_ARG and b"desc" in B.lib.rgnn_last_error()


def test_binding_struct_layouts_match_header(tmp_path):
    """ctypes mirrors of rgnn_graph_desc / rgnn_graph_view have the C layout (size and every offset)."""
    import subprocess
    from paper_2301_06284_b200 import _binding as B
    structs = {"rgnn_graph_desc": B.rgnn_graph_desc, "rgnn_graph_view": B.rgnn_graph_view}
    lines = ['#include <stdio.h>', '#include <stddef.h>', '#include "rgnn.h"', "int main(void) {"]
    for name, cls in structs.items():
        lines.append(f'  printf("{name} size %zu\\n", sizeof({name}));')
        for f, _ in cls._fields_:
            lines.append(f'  printf("{name} {f} %zu\\n", offsetof({name}, {f}));')
    lines.append("  return 0; }")
    src = tmp_path / "layout.c"
    src.write_text("\n".join(lines))
    exe = tmp_path / "layout"
    subprocess.run(["gcc", "-I", os.path.join(ROOT, "include"), str(src), "-o", str(exe)], check=True)
    out = subprocess.run([str(exe)], check=True, capture_output=True, text=True).stdout.split("\n")
    got = {tuple(l.split()[:2]): int(l.split()[2]) for l in out if l.strip()}
    for name, cls in structs.items():
        assert got[(name, "size")] == ctypes.sizeof(cls), name
        for f, _ in cls._fields_:
            assert got[(name, f)] == getattr(cls, f).offset, (name, f)
