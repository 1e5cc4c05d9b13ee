"""The C-ABI library loads without a GPU and exports every symbol the header
declares; host-only entry points work on CPU; formats round-trip."""
import ctypes
import re
from pathlib import Path

import numpy as np
import pytest

from paper_2105_05821_b200 import _lib, build
from paper_2105_05821_b200.errors import IlsimError
from paper_2105_05821_b200.formats import CnnConfig, read_model, read_trace, write_model, write_trace

ROOT = Path(__file__).resolve().parents[1]
GOLD = ROOT / "tests" / "golden"


@pytest.fixture(scope="module")
def L():
    build.build()
    return _lib.lib()


def header_symbols():
    text = (ROOT / "include" / "ilsim_gpu.h").read_text()
    return sorted(set(re.findall(r"\b(ilsim_gpu_\w+)\s*\(", text)))


def test_exports_every_header_symbol(L):
    syms = header_symbols()
    assert set(syms) == set(_lib.EXPORTS)
    for s in syms:
        assert hasattr(L, s), s
    assert L.ilsim_gpu_abi_version() == _lib.ABI_VERSION == 2


STRUCTS = {"ilsim_gpu_options": _lib.Options, "ilsim_trace_view": _lib.TraceView, "ilsim_cnn_config": _lib.CnnCfg,
           "ilsim_sim_config": _lib.SimCfg, "ilsim_sub_result": _lib.SubResult, "ilsim_totals": _lib.Totals}


def test_struct_layouts_match_header(tmp_path):
    """ctypes mirrors vs the C compiler's sizeof/offsetof of every field."""
    import shutil
    import subprocess

    if not shutil.which("gcc"):
        pytest.skip("gcc unavailable")
    lines = ['#include <stdio.h>', '#include <stddef.h>', '#include "ilsim_gpu.h"', "int main(void){"]
    for cname, py in STRUCTS.items():
        lines.append(f'printf("{cname} %zu\\n", sizeof({cname}));')
        for f, _ in py._fields_:
            lines.append(f'printf("{cname}.{f} %zu\\n", offsetof({cname}, {f}));')
    lines.append("return 0;}")
    src = tmp_path / "layout.c"
    src.write_text("\n".join(lines))
    exe = tmp_path / "layout"
    subprocess.run(["gcc", "-I", str(ROOT / "include"), str(src), "-o", str(exe)], check=True)
    got = dict(l.split() for l in subprocess.run([str(exe)], capture_output=True, text=True).stdout.splitlines())
    for cname, py in STRUCTS.items():
        assert int(got[cname]) == ctypes.sizeof(py), cname
        for f, _ in py._fields_:
            assert int(got[f"{cname}.{f}"]) == getattr(py, f).offset, (cname, f)


def test_precision_enum_matches_header(tmp_path):
    """_lib.PREC (the Python names) mirrors the header's ILSIM_PREC_* values."""
    import shutil
    import subprocess

    from paper_2105_05821_b200._lib import PREC

    if not shutil.which("gcc"):
        pytest.skip("gcc unavailable")
    names = {"fp32": "ILSIM_PREC_FP32", "tf32x3": "ILSIM_PREC_TF32X3", "tf32": "ILSIM_PREC_TF32",
             "bf16": "ILSIM_PREC_BF16", "fp8": "ILSIM_PREC_FP8"}
    assert set(PREC) == set(names)
    src = tmp_path / "prec.c"
    src.write_text('#include <stdio.h>\n#include "ilsim_gpu.h"\nint main(void){' +
                   "".join(f'printf("{k} %d\\n", {v});' for k, v in names.items()) + "return 0;}")
    exe = tmp_path / "prec"
    subprocess.run(["gcc", "-I", str(ROOT / "include"), str(src), "-o", str(exe)], check=True)
    got = dict(l.split() for l in subprocess.run([str(exe)], capture_output=True, text=True).stdout.splitlines())
    assert {k: int(v) for k, v in got.items()} == PREC


def test_host_helpers_without_gpu(L, port):
    from paper_2105_05821_b200 import api

    assert api.partition_starts(10, 3) == [0, 4, 7]
    with pytest.raises(IlsimError, match="out of range"):
        api.partition_starts(10, 11)
    assert api.model_flops("c3") == 1_073_408  # cnn.cpp:319-333 for preset_c3
    cfg = CnnConfig.preset_c3()
    m = api.init_weights(cfg, np.zeros(106), 1)
    assert np.array_equal(m.params, port.init_params(cfg, 1))


def test_create_without_gpu_fails_loudly():
    import torch

    if torch.cuda.is_available():
        pytest.skip("GPU present")
    from paper_2105_05821_b200 import GpuSimulator

    with pytest.raises(IlsimError):
        GpuSimulator(0, "fp32")


def test_trace_roundtrip(tmp_path):
    t = read_trace(GOLD / "mix_3000_s4.trace")
    p = tmp_path / "x.trace"
    write_trace(p, t)
    assert p.read_bytes() == (GOLD / "mix_3000_s4.trace").read_bytes()


def test_model_roundtrip(tmp_path):
    m = read_model(GOLD / "small_dataset.model")
    p = tmp_path / "x.model"
    write_model(p, m)
    assert p.read_bytes() == (GOLD / "small_dataset.model").read_bytes()
    assert m.config.hash() == CnnConfig(conv_channels=[16, 16, 16], fc_hidden=32).hash()


def test_format_errors(tmp_path):
    p = tmp_path / "bad"
    p.write_bytes(b"XXXX" + bytes(40))
    with pytest.raises(IlsimError, match="bad trace magic"):
        read_trace(p)
    with pytest.raises(IlsimError, match="bad model magic"):
        read_model(p)
    raw = (GOLD / "mix_3000_s4.trace").read_bytes()
    p.write_bytes(raw[:-5])
    with pytest.raises(IlsimError, match="trace truncated"):
        read_trace(p)


def test_cpp_adapter_compiles_against_reference_headers(tmp_path, L):
    """include/ilsim_gpu.hpp adapts the reference's own C++ types onto the
    C-ABI; build a caller against /root/reference headers and run it (no GPU
    here: the adapter must surface the library error as ilsim::Error)."""
    import shutil
    import subprocess

    ref_inc = Path("/root/reference/proj/include")
    if not ref_inc.exists() or not shutil.which("g++"):
        pytest.skip("reference headers or g++ unavailable")
    src = tmp_path / "adapter.cpp"
    src.write_text(r'''
#include <cstdio>
#include "ilsim_gpu.hpp"
int main() {
  std::vector<ilsim::AnnotatedInstruction> trace(10);
  ilsim::ModelWeights w;
  w.params.assign(293857, 0.0f);  // default CnnConfig == preset_c3(110)
  ilsim::ParallelConfig pc;
  pc.k = 2;
  try {
    auto r = ilsim::gpu::simulate_parallel_gpu(trace, w, pc);
    std::printf("ok %llu\n", (unsigned long long)r.total_cycles);
  } catch (const ilsim::Error& e) {
    std::printf("error: %s\n", e.what());
  }
  return 0;
}
''')
    exe = tmp_path / "adapter"
    lib_dir = ROOT / "paper_2105_05821_b200"
    subprocess.run(["g++", "-std=c++20", "-I", str(ROOT / "include"), "-I", str(ref_inc), str(src), "-o", str(exe),
                    "-L", str(lib_dir), "-l:libilsim_gpu.so", f"-Wl,-rpath,{lib_dir}"], check=True)
    out = subprocess.run([str(exe)], capture_output=True, text=True, timeout=60).stdout
    import torch

    assert out.startswith("ok" if torch.cuda.is_available() else "error:"), out


def test_trace_records_header_checks(tmp_path):
    """The GPU-ingest reader applies read_trace's header checks (trace.cpp:102-124)."""
    import pytest as _pt

    from paper_2105_05821_b200 import IlsimError
    from paper_2105_05821_b200.formats import read_trace, trace_records

    gold = __import__("conftest").GOLDEN / "mix_3000_s4.trace"
    body, n, _ = trace_records(gold)
    assert n == read_trace(gold).n and body.size == n * 108
    raw = gold.read_bytes()
    (tmp_path / "bad.trace").write_bytes(b"XXXX" + raw[4:])
    with _pt.raises(IlsimError, match="bad trace magic"):
        trace_records(tmp_path / "bad.trace")
    (tmp_path / "short.trace").write_bytes(raw[:-5])
    with _pt.raises(IlsimError, match="trace truncated at record"):
        trace_records(tmp_path / "short.trace")


@pytest.mark.gpu
@pytest.mark.parametrize("precision,k,devices", [(1, 16, [0]), (0, 5, [0, 0]), (1, 7, [0, 0, 0])])
def test_cpp_dropin_on_gpu(precision, k, devices):
    """The C++ drop-in end to end on the GPU (tests/cpp/dropin_main.cpp, built
    by `make -C oracle dropin` against the reference's own libraries): the
    reference's simulate_parallel with CudaCnnPredictor plugged in, the
    whole-loop simulate_parallel_gpu and the multi-device group, against the
    reference's CPU CnnPredictor run (total cycles within 0.1%; group ==
    single-device bit-exactly) and OraclePredictor (bit-exact)."""
    import json
    import subprocess

    exe = ROOT / "oracle" / "_ref" / "ilsim_dropin"
    if not exe.exists():
        pytest.skip("oracle/_ref/ilsim_dropin not built (needs /root/reference at build time)")
    gold = __import__("conftest").GOLDEN
    out = subprocess.run([str(exe), str(gold / "mix_3000_s4.trace"), str(gold / "small_dataset.model"), str(k),
                          str(precision)] + [str(d) for d in devices], capture_output=True, text=True, timeout=600)
    assert out.returncode == 0, out.stdout + out.stderr
    r = json.loads(out.stdout)
    cpu = r["cpu"]
    for name in ("plugin", "gpu", "group"):
        assert r[name]["instructions"] == cpu["instructions"] == 3000
        assert abs(r[name]["total_cycles"] - cpu["total_cycles"]) <= 1e-3 * cpu["total_cycles"], (name, r)
    assert r["group"]["total_cycles"] == r["gpu"]["total_cycles"]
    assert r["group"]["same_subs"] == r["group"]["subs"] == k and r["group"]["same_fetch"] == 3000
    o = r["oracle_gpu"]
    assert o["total_cycles"] == r["oracle_cpu"]["total_cycles"] and o["same_subs"] == k and o["same_fetch"] == 3000


def test_sub_results_sequence_over_the_abi_array():
    """ParallelResult.sub_results (api.SubResults) over an ilsim_sub_result
    array, as GpuSimulator._collect builds it: sequence behaviour, per-sub-trace
    fetch slices in trace order, edits that stick, vectorised totals."""
    import numpy as np

    from paper_2105_05821_b200 import _lib
    from paper_2105_05821_b200.api import GpuSimulator
    from paper_2105_05821_b200.dist import Totals

    subs = (_lib.SubResult * 4)()
    for j, (n, c) in enumerate([(3, 10), (0, 0), (2, 9), (4, 7)]):
        subs[j].instructions, subs[j].total_cycles, subs[j].sum_fetch = n, c, c - 1
        subs[j].empty = int(n == 0)
    pf = np.arange(9, dtype=np.uint32)

    class Tot:
        device_ms, kernel_ms, launches, rounds = 1.5, (0.0, 0.0, 0.0, 0.0), 3, 4

    r = GpuSimulator._collect(subs, 4, pf, 9, Tot, None, 0, None)
    s = r.sub_results
    assert (r.total_cycles, r.instructions, len(s)) == (26, 9, 4)
    assert s[1].empty and s[1].cpi == 0.0 and s[-1] is s[3] and s[0].cpi == 10 / 3
    assert [x.predicted_fetch.tolist() for x in s] == [[0, 1, 2], [], [3, 4], [5, 6, 7, 8]]
    assert [x.total_cycles for x in s[1:3]] == [0, 9] and [x.instructions for x in s] == [3, 0, 2, 4]
    with pytest.raises(IndexError):
        s[4]
    t = Totals.of(s)
    assert (t.total_cycles, t.instructions, t.sum_fetch) == (26, 9, 22)
    s[2].total_cycles += 5  # edits stick on the cached object
    assert s[2].total_cycles == 14
