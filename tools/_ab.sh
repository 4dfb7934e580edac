timeout 600 python tools/ab_compare.py > gpurun_out/ab_emit.txt 2> gpurun_out/ab_emit.err
timeout 400 python bench.py --steps 50 --warmup 5 --no-cpu-baseline --sorted-k 0 --no-backward > gpurun_out/emit_bench.json 2> gpurun_out/emit_bench.err
ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"emit" --csv python tools/render_view.py 1 2 > gpurun_out/emit_launch.csv 2>&1
