timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/fuse_gputest.log 2>&1
timeout 600 python tools/ab_compare.py > gpurun_out/ab_fuse.txt 2> gpurun_out/ab_fuse.err
timeout 400 python bench.py --steps 50 --warmup 5 --no-cpu-baseline --sorted-k 0 --no-backward > gpurun_out/fuse_bench.json 2> gpurun_out/fuse_bench.err
