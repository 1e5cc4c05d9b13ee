# bench --config c3 (one global 100M-instruction trace, 65,536 sub-traces) on one GPU and under torchrun (1 proc)
timeout 1500 python bench.py --config c3 --steps 2 --warmup 1 --no-cpu-baseline > gpurun_out/r02g_bench_c3.jsonl 2> gpurun_out/r02g_bench_c3.err; echo "c3 rc=$?"
tail -c 2500 gpurun_out/r02g_bench_c3.jsonl
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29533 bench.py --gpus 1 --steps 2 --warmup 1 --no-cpu-baseline > gpurun_out/r02g_bench_torchrun.jsonl 2> gpurun_out/r02g_bench_torchrun.err; echo "torchrun rc=$?"
tail -c 600 gpurun_out/r02g_bench_torchrun.jsonl
timeout 600 python bench.py --impl reference --config c3 --steps 2 --warmup 0 > gpurun_out/r02g_bench_c3_reference.jsonl 2>&1; echo "c3 ref rc=$?"; tail -c 800 gpurun_out/r02g_bench_c3_reference.jsonl
