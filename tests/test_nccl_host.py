"""The NCCL transport's host side without a GPU: libpjds dlopens the same libnccl.so.2 torch ships,
resolves every symbol it uses, and creates the 128-byte ncclUniqueId that DistPjds.create broadcasts."""
import ctypes

import pytest


def test_nccl_load_and_unique_id():
    import build_native
    build_native.build_pjds()
    import paper_1112_5588_b200 as pj
    path = pj._nccl_path()
    if path is None:
        pytest.skip("nvidia-nccl package not installed")
    pj.call("pjds_nccl_load", path)
    a, b = (ctypes.c_char * 128)(), (ctypes.c_char * 128)()
    pj.call("pjds_nccl_unique_id", a)
    pj.call("pjds_nccl_unique_id", b)
    assert bytes(a) != bytes(128) and bytes(a) != bytes(b)
    assert pj.lib().pjds_nccl_load(b"/nonexistent/libnccl.so.2") == 0  # already loaded: no-op
