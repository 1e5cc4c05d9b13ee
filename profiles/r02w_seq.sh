# simulate_trace with the C3 on the 10M c2 trace (persistent kernel) vs the reference's own K = 1 run
mkdir -p gpurun_out
timeout 1500 python tools/configs.py --only seq > gpurun_out/r02w_configs_seq.jsonl 2>&1; cat gpurun_out/r02w_configs_seq.jsonl
cat > /tmp/c3_seq.py <<'PY'
import sys; sys.path.insert(0, ".")
from paper_2105_05821_b200 import GpuSimulator, ParallelConfig, SimConfig, read_model, read_trace
m = read_model("tests/golden/c3_trained.model"); t = read_trace("tests/golden/mix_3000_s4.trace")
g = GpuSimulator(0, "fp32"); g.load_model(m)
pc = ParallelConfig(k=1, sim=SimConfig(max_context=110)); g.load_trace(t, pc); r = g.run(pc)
print(f"seq_c3: {t.n} instructions, {r.launches} launch(es), {1e3 * r.device_ms / t.n:.2f} us per instruction")
PY
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r02w_seq_c3_launches.csv \
   python /tmp/c3_seq.py > gpurun_out/r02w_seq_c3_short.txt 2>&1
python profiles/summarize_launches.py gpurun_out/r02w_seq_c3_launches.csv > gpurun_out/r02w_seq_c3_launches.txt 2>&1
cat gpurun_out/r02w_seq_c3_short.txt gpurun_out/r02w_seq_c3_launches.txt
