# HEAD check after the persistent kernels: GPU tests, smoke, c1 config, sanitizers on seq_c3
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/r02s_pytest.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/r02s_pytest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
timeout 900 python tools/configs.py --only c1 > gpurun_out/r02s_configs_c1.jsonl 2>&1; tail -c 600 gpurun_out/r02s_configs_c1.jsonl
cat > /tmp/c3_seq.py <<'PY'
import sys; sys.path.insert(0, ".")
from paper_2105_05821_b200 import GpuSimulator, ParallelConfig, SimConfig, read_model, read_trace
m = read_model("tests/golden/c3_trained.model"); t = read_trace("tests/golden/mix_3000_s4.trace").slice(0, int(sys.argv[1]))
g = GpuSimulator(0, "fp32"); g.load_model(m)
pc = ParallelConfig(k=1, sim=SimConfig(max_context=110)); g.load_trace(t, pc); r = g.run(pc)
print(f"seq_c3: {t.n} instructions, {r.launches} launch(es), total cycles {r.total_cycles}")
PY
for T in memcheck racecheck synccheck; do
  timeout 900 compute-sanitizer --tool $T python /tmp/c3_seq.py 300 2>&1 | tail -2 | sed "s/^/seq_c3 $T: /"
done
