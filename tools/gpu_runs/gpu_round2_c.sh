set -x
python bench.py --workload c5 --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/bench_c5_r02c.json 2>&1
LORENZ_LIB=tools/variants/liblorenz_trace.so python tools/seg_trace.py --kib 65536 --integrator rk4fma > gpurun_out/seg_trace_fma.jsonl 2>&1
LORENZ_LIB=tools/variants/liblorenz_trace.so python tools/seg_trace.py --kib 65536 --integrator rk4 >> gpurun_out/seg_trace_fma.jsonl 2>&1
python tools/tune.py --integrator rk4fma --kib 65536 100000 131072 262144 > gpurun_out/tune_fma.jsonl 2>&1
python tools/tune.py --integrator rk4fma --kib 65536 --skew 0 --tag skew0 >> gpurun_out/tune_fma.jsonl 2>&1
python tools/tune.py --integrator rk4fma --kib 65536 --skew 30 --tag skew30 >> gpurun_out/tune_fma.jsonl 2>&1
python tools/tune.py --integrator rk4fma --kib 65536 --sched wave --tag wave >> gpurun_out/tune_fma.jsonl 2>&1
python tools/tune.py --integrator rk4fma --kib 65536 --reps 1 > gpurun_out/plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:lorenz_chain_seg_kernel -s 1 -c 1 -o gpurun_out/fma_c3_full_r02 python tools/tune.py --integrator rk4fma --kib 65536 --reps 1 > gpurun_out/ncu_fma.log 2>&1
echo done
