"""The C ABI library loads on a CPU-only host and exports every entry point include/*.h declares;
calls that need no GPU behave (status codes, dry-run control plane)."""
import ctypes as C
import os
import re
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
LIB = os.path.join(ROOT, "paper_2404_18322_b200", "libblockexec.so")


def declared_functions():
    names = set()
    for h in ("blockexec.h", "blockhost.h", "blockpolicy.h"):
        text = open(os.path.join(ROOT, "include", h)).read()
        text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
        for m in re.finditer(r"\b((?:be|bh)_[a-z0-9_]+)\s*\(", text):
            names.add(m.group(1))
    return names


def test_header_declares_the_abi():
    names = declared_functions()
    assert {"be_exec_batch", "be_exec_batch_dev", "be_cosine", "be_gather_rows",
            "be_scatter_rows", "bh_pool_pop_batch", "bh_kv_append_tokens",
            "bh_runner_decode_step", "bh_policy_choose_binding", "bh_policy_speculation_marks",
            "bh_policy_choose_device", "bh_policy_placement_moves"} <= names
    assert len(names) > 50


def test_library_exports_every_declared_symbol():
    assert os.path.exists(LIB), "build first: __graft_entry__.build()"
    out = subprocess.run(["nm", "-D", "--defined-only", LIB], capture_output=True, text=True,
                         check=True).stdout
    exported = {line.split()[-1] for line in out.splitlines() if " T " in line}
    missing = declared_functions() - exported
    assert not missing, sorted(missing)


def test_library_loads_and_reports_errors_without_gpu():
    from paper_2404_18322_b200._lib import lib
    L = lib()
    h = C.c_void_p()
    # no context pointer: invalid argument, never a crash
    assert L.be_ctx_create(0, None) == 1
    assert L.be_exec_batch(None, None, None, None, 1, 0, None, 0, 1, None, None, None, None) == 1
    assert L.be_cosine(None, None, None, 1, 8, 0.95, None, None, None) == 1
    assert L.bh_runner_create(None, None, C.byref(h)) == 1


def test_sm100a_code_present():
    out = subprocess.run(["cuobjdump", "-lelf", LIB], capture_output=True, text=True).stdout
    assert "sm_100a" in out
    sass = subprocess.run(["cuobjdump", "-sass", LIB], capture_output=True, text=True).stdout
    # tcgen05 MMA, TMA and TMEM loads are in the product kernels
    for mnemonic in ("UTCHMMA", "UTMALDG", "UBLKCP", "LDTM"):
        assert mnemonic in sass, mnemonic


def test_dry_run_runner_on_cpu():
    from paper_2404_18322_b200.runner import Runner
    from paper_2404_18322_b200.workloads import c2_llama7b
    wl = c2_llama7b(prompt=64, output=4)
    run = Runner(None, wl, mode=1, dry_run=True)
    run.run()
    assert run.live == 64
    n = run.decode_step()
    assert n == 14  # 6 shared blocks at 64 rows + 2 private blocks x 4 tenants
    tr = run.trace()
    assert [len(t[3]) for t in tr[-14:]] == [64] * 6 + [16] * 8
    st = run.step_stats()
    # 22.7 GB of weights per decode step (9.71 shared + 12.95 private)
    assert abs(st["weight_bytes"] - 22.66e9) / 22.66e9 < 0.01
