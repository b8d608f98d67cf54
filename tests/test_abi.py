"""C-ABI library checks that need no GPU: it loads, exports every symbol
include/ltlgrid_gpu.h declares, is built for sm_100a, and its host-only
validator reproduces the reference's messages."""
import ctypes as C
import json
import os
import re
import subprocess

import numpy as np
import pytest

from conftest import GOLDEN, ROOT, has_gpu
from paper_1810_02612_b200 import _native as N

HEADER = os.path.join(ROOT, "include", "ltlgrid_gpu.h")


def declared_functions():
    src = open(HEADER).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(ltlg_[a-z0-9_]+)\s*\(", src)))


def test_header_declares_what_python_binds():
    assert declared_functions() == sorted(N.EXPORTS)


def test_library_loads_and_exports_every_symbol():
    L = N.lib()
    out = subprocess.run(["nm", "-D", "--defined-only", N.GPU_SO], capture_output=True, text=True, check=True).stdout
    exported = set(re.findall(r"\bT (ltlg_\w+)", out))
    for name in declared_functions():
        assert name in exported, name
        assert getattr(L, name) is not None
    assert L.ltlg_abi_version() == 1


def test_library_is_sm100a_only():
    out = subprocess.run(["cuobjdump", "--list-elf", N.GPU_SO], capture_output=True, text=True).stdout
    assert "sm_100a" in out
    assert "sm_90" not in out and "sm_80" not in out


def test_product_library_leaves_out_the_ab_variants():
    # the A/B-only kernels (dev knobs) live in libltlgrid_gpu_ab.so; the product
    # library carries the default dispatch's kernels only
    def kernels(so):
        out = subprocess.run(["cuobjdump", "-sass", so], capture_output=True, text=True).stdout
        return set(re.findall(r"Function : \S*?(label_\w+?_kernel|tc_build_kernel)", out))
    if subprocess.run(["which", "cuobjdump"], capture_output=True).returncode:
        pytest.skip("cuobjdump not on PATH")
    prod, ab = kernels(N.GPU_SO), kernels(N.AB_SO)
    dev_only = {"label_stream_kernel", "label_stream_tma_kernel", "label_pl_kernel", "label_tc_kernel", "tc_build_kernel"}
    assert {"label_wm_kernel", "label_wm1_kernel", "label_stream64_kernel"} <= prod
    assert not prod & dev_only
    assert dev_only <= ab and prod <= ab


def test_no_cpu_fallback_without_device():
    if has_gpu():
        pytest.skip("a GPU is present")
    from paper_1810_02612_b200 import LabelEngine, LtlgError

    with pytest.raises(LtlgError, match="no CUDA device"):
        LabelEngine()


def test_host_validator_matches_reference_messages():
    L = N.lib()
    with open(os.path.join(GOLDEN, "validate.json")) as f:
        cases = json.load(f)
    for c in cases:
        off = np.array(c["offsets"], np.uint64)
        idx = np.array(c["indices"], np.uint32)
        buf = C.create_string_buffer(256)
        st = L.ltlg_validate_csr(c["rows"], c["cols"], off.ctypes.data, off.size, idx.ctypes.data, idx.size, buf, 256)
        if c["error"] is None:
            assert st == N.LTLG_OK, c
        else:
            assert st == N.LTLG_EINVAL and buf.value.decode() == c["error"], c
    off = np.array([0, 1, 3], np.uint64)
    idx = np.array([4, 1, 2], np.uint32)
    buf = C.create_string_buffer(256)
    assert L.ltlg_validate_csr(2, 5, off.ctypes.data, 3, idx.ctypes.data, 3, buf, 256) == N.LTLG_OK


def test_struct_layouts_match_the_header(tmp_path):
    """The ctypes mirrors of the header's structs (sizes and field offsets)
    equal what a C compiler lays out for include/ltlgrid_gpu.h."""
    structs = {
        "ltlg_options": (N.Options, ["sort_rows", "stream_task_pairs", "batch_task_pairs", "profile",
                                     "readback_chunks", "reserved"]),
        "ltlg_info": (N.Info, ["rows", "cols", "nnz", "words", "pairs", "t_bytes", "n_devices", "props", "frames",
                               "label_bytes", "label_words", "reserved"]),
        "ltlg_grid2": (N.Grid2, ["depth", "lo0", "hi0", "lo1", "hi1"]),
        "ltlg_pose2": (N.Pose2, ["dx", "dy", "cos_t", "sin_t"]),
        "ltlg_gridk": (N.GridK, ["dims", "depth", "lo", "hi"]),
        "ltlg_footprint": (N.Footprint, ["length", "width", "ref_offset"]),
        "ltlg_scenario": (N.Scenario, ["loop_cx", "loop_cy", "loop_radius", "lane_width", "agent_count",
                                       "agent_speed_min", "agent_speed_max", "agent_length", "agent_width",
                                       "lateral_spread", "horizon", "seed"]),
    }
    lines = ['#include <stdio.h>', '#include <stddef.h>', f'#include "{HEADER}"', 'int main(void) {']
    for cname, (_, fields) in structs.items():
        lines.append(f'printf("{cname} size %zu\\n", sizeof({cname}));')
        for f in fields:
            lines.append(f'printf("{cname} {f} %zu\\n", offsetof({cname}, {f}));')
    lines.append("return 0; }")
    src = tmp_path / "layout.c"
    src.write_text("\n".join(lines))
    exe = tmp_path / "layout"
    subprocess.run(["gcc", "-std=c11", "-o", str(exe), str(src)], check=True)
    got = {}
    for line in subprocess.run([str(exe)], capture_output=True, text=True, check=True).stdout.splitlines():
        name, key, val = line.split()
        got[(name, key)] = int(val)
    for cname, (py, fields) in structs.items():
        assert C.sizeof(py) == got[(cname, "size")], cname
        for f in fields:
            assert getattr(py, f).offset == got[(cname, f)], (cname, f)


def test_trajectory_inputs_both_forms():
    """swept_volume's trajectory argument: (sample_offsets, samples) or a list
    of per-edge State5 arrays give the same flat arrays."""
    from paper_1810_02612_b200.label import _trajectories

    rows = [np.arange(10.0).reshape(2, 5), np.zeros((0, 5)), np.ones((3, 5))]
    off, smp = _trajectories(rows)
    assert off.tolist() == [0, 2, 2, 5] and smp.shape == (5, 5)
    off2, smp2 = _trajectories((off, smp))
    assert np.array_equal(off2, off) and np.array_equal(smp2, smp)
    off3, smp3 = _trajectories([])
    assert off3.tolist() == [0] and smp3.shape == (0, 5)
