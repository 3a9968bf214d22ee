"""The C-ABI library: it is built, loads, exports every symbol that
include/snpb200.h declares, its struct layouts match the ctypes mirror, and
without a GPU it refuses to run (no CPU fallback).  CPU only -- no compute
calls."""

import ctypes
import re
import subprocess

import pytest

from conftest import ROOT
from paper_2408_04343_b200 import _native as nat

HEADER = ROOT / "include" / "snpb200.h"


def declared_functions() -> list[str]:
    text = HEADER.read_text()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(snp_[a-z_]+)\s*\(", text)))


def test_library_exports_every_declared_symbol():
    lib = nat.load()
    names = declared_functions()
    assert len(names) >= 14
    for name in names:
        assert hasattr(lib, name), f"{name} missing from {nat.LIB_PATH}"
    assert {n for n, _, _ in nat.SIGNATURES} == set(names)
    assert lib.snp_abi_version() == 6


def test_struct_layouts_match_header(tmp_path):
    """Compile a probe against the header with gcc and compare sizeof/offsetof."""
    src = tmp_path / "probe.c"
    src.write_text(f"""
#include <stdio.h>
#include <stddef.h>
#include "{HEADER}"
int main(void) {{
  printf("%zu %zu %zu %zu %zu %zu\\n", sizeof(snp_system_desc), sizeof(snp_run_opts),
         sizeof(snp_trace_out), sizeof(snp_result), sizeof(snp_engine_info), sizeof(snp_exchange));
  printf("%zu %zu %zu\\n", offsetof(snp_system_desc, sparse_data), offsetof(snp_result, stats),
         offsetof(snp_run_opts, collect_stats));
  return 0;
}}
""")
    exe = tmp_path / "probe"
    subprocess.run(["gcc", "-std=c11", "-o", str(exe), str(src)], check=True)
    out = subprocess.run([str(exe)], check=True, capture_output=True, text=True).stdout.split()
    sizes = [ctypes.sizeof(c) for c in (nat.SystemDesc, nat.RunOpts, nat.TraceOut, nat.Result, nat.EngineInfo,
                                        nat.Exchange)]
    offs = [nat.SystemDesc.sparse_data.offset, nat.Result.stats.offset, nat.RunOpts.collect_stats.offset]
    assert [int(x) for x in out] == sizes + offs


def test_sm100a_code_in_library():
    out = subprocess.run(["cuobjdump", "--list-elf", str(nat.LIB_PATH)], capture_output=True, text=True)
    assert "sm_100a" in out.stdout


def test_no_gpu_means_loud_failure():
    import torch
    if torch.cuda.is_available():
        pytest.skip("a GPU is present")
    import paper_2408_04343_b200 as snp
    with pytest.raises(RuntimeError, match="no CPU fallback"):
        snp.prepare(snp.gen_sort(snp.SortInstance(3)), snp.Format.COMPRESSED)
