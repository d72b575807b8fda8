"""The C-ABI boundary on CPU: the sm_100a library loads, exports every entry
point include/oserve_gpu.h declares, carries sm_100a code, and refuses to run
without a device (no CPU fallback).  The device-free protocol helpers are
exercised directly."""
import os
import re
import subprocess

import pytest
import torch

from paper_2602_12151_b200 import _native, core

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "oserve_gpu.h")


def declared_symbols():
    src = open(HEADER).read()
    return sorted(set(re.findall(r"\b(oserve_(?:gpu|shard|key|forecast|nccl)\w*)\s*\(", src)))


def test_library_exports_every_declared_symbol():
    lib = _native.load_library()
    syms = declared_symbols()
    assert len(syms) >= 25
    missing = [s for s in syms if not hasattr(lib, s)]
    assert missing == []
    assert set(syms) == set(_native.EXPORTS)


def test_library_carries_sm100a_code():
    out = subprocess.run(["cuobjdump", "--list-elf", _native.LIB_PATH], capture_output=True, text=True)
    if out.returncode != 0:
        pytest.skip("cuobjdump unavailable")
    assert "sm_100a" in out.stdout


@pytest.mark.skipif(torch.cuda.is_available(), reason="checks the no-device behaviour")
def test_no_cpu_fallback_without_device():
    with pytest.raises(core.CudaError):
        _native.GpuContext(core.cluster(1, 8), core.model_140gb())


def test_shard_mapping_partitions_the_plan_order():
    for total in (0, 1, 61, 4096, 4097, 933_333, 3 * 4096 + 7):
        for world in (1, 2, 3, 4, 8):
            seen = []
            for r in range(world):
                n = _native.shard_count(total, r, world)
                seen += [_native.shard_global_rank(i, r, world) for i in range(0, n, max(1, n // 50))]
                if n:
                    assert _native.shard_global_rank(n - 1, r, world) < total
            assert sum(_native.shard_count(total, r, world) for r in range(world)) == total
            assert len(set(seen)) == len(seen)


def test_key_layout_orders_like_the_reference():
    lay = _native.key_layout(1000, 7, 8, 16)
    k = lambda o, p, s, l: _native.pack_key(lay, o, p, s, l)
    assert k(606, 3, 5, 2) < k(605, 0, 0, 0)      # higher objective first
    assert k(606, 2, 9, 9) < k(606, 3, 0, 0)      # then earlier partition
    assert k(606, 3, 4, 9) < k(606, 3, 5, 0)      # then smaller total pp
    assert k(606, 3, 5, 1) < k(606, 3, 5, 2)      # then lower combo rank
    assert k(1000, 6, 8, 15) < (1 << 63)
    with pytest.raises(core.TooLarge):
        _native.key_layout(2 ** 31, 2 ** 20, 1024, 2 ** 40)
