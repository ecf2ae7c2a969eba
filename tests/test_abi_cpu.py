"""CPU checks of the boundary: libhmc.so loads and exports every symbol include/hmc.h declares;
the binding marshals structs with the C layout.  No compute calls (no GPU here)."""
import ctypes
import os
import re
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HDR = os.path.join(ROOT, "include", "hmc.h")


def declared_functions():
    src = open(HDR).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(hmc_[a-z_]+)\s*\(", src)))


def test_header_declares_boundary_calls():
    names = declared_functions()
    for must in ("hmc_setup", "hmc_grad", "hmc_trajectory", "hmc_sample", "hmc_destroy"):
        assert must in names


def test_library_exports_every_declared_symbol():
    from paper_2507_14652_b200 import abi
    if not os.path.exists(abi.LIB_PATH):
        subprocess.check_call(["make", "-C", ROOT], stdout=subprocess.DEVNULL)
    L = ctypes.CDLL(abi.LIB_PATH)
    for name in declared_functions():
        assert hasattr(L, name), name
    assert set(abi.EXPORTS) == set(declared_functions())
    out = subprocess.check_output(["nm", "-D", "--defined-only", abi.LIB_PATH]).decode()
    for name in declared_functions():
        assert re.search(rf"\bT {name}\b", out), name


def test_struct_layouts_match_header():
    from paper_2507_14652_b200 import abi
    # hmc_net: int32 + 3 pointers (padded) ; hmc_arch: kind + 2 nets + has_b0
    assert ctypes.sizeof(abi.hmc_net) == 32
    assert abi.hmc_arch.net.offset == 8
    assert ctypes.sizeof(abi.hmc_data) == 10 * 8 and abi.hmc_data.q_per_pair.offset == 9 * 8
    assert abi.hmc_config.exchange.offset == abi.hmc_config.nccl_id.offset + 8
    assert ctypes.sizeof(abi.hmc_config) == abi.hmc_config.exchange.offset + 8


def test_c_struct_sizes_via_compiler(tmp_path):
    """Compile a tiny C program against include/hmc.h and compare sizeof/offsetof with ctypes."""
    from paper_2507_14652_b200 import abi
    c = tmp_path / "s.c"
    c.write_text('#include <stdio.h>\n#include <stddef.h>\n#include "hmc.h"\nint main(){printf("%zu %zu %zu %zu %zu %zu\\n",'
                 'sizeof(hmc_net),sizeof(hmc_arch),sizeof(hmc_data),sizeof(hmc_config),offsetof(hmc_config,seed),'
                 'offsetof(hmc_config,exchange));}\n')
    exe = tmp_path / "s"
    subprocess.check_call(["gcc", "-I", os.path.join(ROOT, "include"), str(c), "-o", str(exe)])
    vals = [int(v) for v in subprocess.check_output([str(exe)]).split()]
    assert vals == [ctypes.sizeof(abi.hmc_net), ctypes.sizeof(abi.hmc_arch), ctypes.sizeof(abi.hmc_data),
                    ctypes.sizeof(abi.hmc_config), abi.hmc_config.seed.offset, abi.hmc_config.exchange.offset]


def test_product_path_does_not_import_oracle():
    pkg = os.path.join(ROOT, "paper_2507_14652_b200")
    for dp, _, fs in os.walk(pkg):
        for f in fs:
            if f.endswith((".py", ".cu", ".cuh", ".h", ".cpp")):
                txt = open(os.path.join(dp, f)).read()
                assert "oracle" not in re.sub(r"#.*|//.*", "", txt).replace("no CPU fallback", ""), f
