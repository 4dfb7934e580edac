timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/k1_gputest.log 2>&1
timeout 400 python bench.py --steps 50 --warmup 5 --no-cpu-baseline --sorted-k 0 --no-backward > gpurun_out/k1_bench.json 2> gpurun_out/k1_bench.err
bash tools/ncu_src.sh capture "project_kernel" k1src2
