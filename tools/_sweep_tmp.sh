cd /root/repo
for v in base win4 win16 t256i16 i9; do GUT_LIB=build_var/libgut_$v.so python tools/stage_bench.py 8 $v; done > gpurun_out/r2_sortsweep.txt 2>&1
GUT_BLEND_TRACE=1 python tools/blend_trace.py 0 1 > gpurun_out/r2_trace.txt 2>&1
