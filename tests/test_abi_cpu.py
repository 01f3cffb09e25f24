"""CPU-side checks of the C ABI: the library builds for sm_100a, loads, exports every symbol
include/espo.h declares, and its struct layouts match the header (no GPU compute here)."""
import ctypes
import os
import re
import subprocess
import tempfile

import pytest

from paper_2512_07710_b200.build import build_library, LIB_PATH

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "espo.h")


@pytest.fixture(scope="module")
def lib():
    build_library()
    return ctypes.CDLL(LIB_PATH)


def declared_functions():
    src = open(HEADER).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(espo_[a-z0-9_]+)\s*\(", src)))


def test_every_declared_symbol_is_exported(lib):
    names = declared_functions()
    assert len(names) >= 14
    for n in names:
        assert hasattr(lib, n), n
    out = subprocess.run(["nm", "-D", "--defined-only", LIB_PATH], capture_output=True,
                         text=True).stdout
    for n in names:
        assert re.search(rf"\bT {n}\b", out), n
    from paper_2512_07710_b200.espo import EXPORTED_SYMBOLS
    assert sorted(EXPORTED_SYMBOLS) == names


def test_binary_targets_sm100a():
    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", LIB_PATH],
                         capture_output=True, text=True).stdout
    assert "sm_100a" in out


def test_struct_layout_matches_header(lib):
    """Compile a C probe against the header and compare with the ctypes mirror."""
    from paper_2512_07710_b200.espo import Config, STATS_LEN
    probe = r'''
#include <stdio.h>
#include <stddef.h>
#include "espo.h"
int main(void) {
  printf("%zu %zu %zu %zu %zu %zu\n", sizeof(espo_config), offsetof(espo_config, adv_eps),
         offsetof(espo_config, logit_scale), offsetof(espo_config, zero_fill_inactive_rows),
         sizeof(espo_stats), offsetof(espo_stats, clip_frac));
  return 0;
}'''
    with tempfile.TemporaryDirectory() as d:
        c = os.path.join(d, "p.c")
        open(c, "w").write(probe)
        exe = os.path.join(d, "p")
        subprocess.run(["gcc", "-std=c99", "-I", os.path.join(ROOT, "include"), c, "-o", exe],
                       check=True)
        vals = [int(x) for x in subprocess.run([exe], capture_output=True, text=True,
                                               check=True).stdout.split()]
    assert vals[0] == ctypes.sizeof(Config)
    assert vals[1] == Config.adv_eps.offset
    assert vals[2] == Config.logit_scale.offset
    assert vals[3] == Config.zero_fill_inactive_rows.offset
    assert vals[4] == STATS_LEN * 8
    assert vals[5] == 8 * 8


def test_host_only_entry_points(lib):
    from paper_2512_07710_b200.espo import Config
    lib.espo_status_string.restype = ctypes.c_char_p
    assert lib.espo_status_string(0) == b"ESPO_OK"
    assert lib.espo_status_string(5) == b"ESPO_ERR_NONFINITE_INPUT"
    cfg = Config()
    lib.espo_config_default(ctypes.byref(cfg), 151936)
    assert cfg.vocab == 151936 and abs(cfg.alpha - 0.4) < 1e-7 and cfg.n_buckets == 2
    assert (cfg.split_num, cfg.split_den) == (4, 5) and cfg.adv_eps == 1e-6
    # argument validation happens before any device work
    lib.espo_create.restype = ctypes.c_int
    h = ctypes.c_void_p()
    assert lib.espo_create(None, None, 0, 1, 0, ctypes.byref(h)) == 1
    bad = Config()
    lib.espo_config_default(ctypes.byref(bad), 1)
    assert lib.espo_create(ctypes.byref(bad), None, 0, 1, 0, ctypes.byref(h)) == 1
    # NULL context is rejected everywhere
    lib.espo_loss_fwd.restype = ctypes.c_int
    assert lib.espo_loss_fwd(None, None, 0, None, None, None, 0, 0, 0, None) == 1
    lib.espo_launch_count.restype = ctypes.c_uint64
    assert lib.espo_launch_count(None) == 0


def test_binding_argument_checks():
    """The binding validates what the C ABI cannot see (it only gets addresses and pitches):
    dtype (int64 tokens would be read as interleaved int32 pairs), inner stride, row count,
    row width and device."""
    import torch
    from paper_2512_07710_b200.espo import check_tensor
    cpu = torch.device("cpu")
    check_tensor(torch.zeros(8, dtype=torch.int32), "tokens", torch.int32, cpu, 8)
    check_tensor(None, "mask", torch.uint8, cpu, 8, optional=True)
    with pytest.raises(TypeError):
        check_tensor(torch.zeros(8, dtype=torch.int64), "tokens", torch.int32, cpu, 8)
    with pytest.raises(ValueError):
        check_tensor(torch.zeros(7, dtype=torch.int32), "tokens", torch.int32, cpu, 8)
    with pytest.raises(ValueError):
        check_tensor(torch.zeros(16, dtype=torch.int32)[::2], "tokens", torch.int32, cpu, 8)
    with pytest.raises(ValueError):
        check_tensor(None, "tokens", torch.int32, cpu, 8)
    z = torch.zeros((4, 10), dtype=torch.bfloat16)
    check_tensor(z, "logits", torch.bfloat16, cpu, 4, 10)
    with pytest.raises(ValueError):
        check_tensor(z, "logits", torch.bfloat16, cpu, 4, 11)          # row narrower than vocab
    with pytest.raises(ValueError):
        check_tensor(z.t(), "logits", torch.bfloat16, cpu)             # inner stride != 1
    with pytest.raises(TypeError):
        check_tensor(z, "dlogits", torch.float32, cpu, 4, 10)
    with pytest.raises(ValueError):
        check_tensor(z, "logits", torch.bfloat16, torch.device("cuda", 0), 4, 10)
