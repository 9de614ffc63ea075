"""The C-ABI library loads and exports every symbol include/rgnn.h declares (no GPU needed)."""
import ctypes
import os
import re

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def declared_functions():
    with open(os.path.join(ROOT, "include", "rgnn.h")) as f:
        src = re.sub(r"/\*.*?\*/", "", f.read(), flags=re.S)
    return sorted(set(re.findall(r"^\s*(?:const\s+)?[a-z_0-9]+\s*\*?\s*(rgnn_\w+|rgcn_\w+|rgat_\w+)\s*\(", src, flags=re.M)))


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
