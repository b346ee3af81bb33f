set -x
python -m pytest tests -m gpu -q -x --deselect tests/test_gpu_fullsize.py > gpurun_out/pytest_gpu_r02j.log 2>&1
python tools/tune.py --tag imm --integrator rk4 --kib 37888 56832 65536 100000 131072 262144 524288 1048576 > gpurun_out/tune_imm.jsonl 2>&1
python tools/tune.py --tag imm-wave --integrator rk4 --kib 75776 262144 1048576 --sched wave >> gpurun_out/tune_imm.jsonl 2>&1
python tools/tune.py --tag imm --integrator euler --kib 65536 262144 1048576 >> gpurun_out/tune_imm.jsonl 2>&1
python tools/tune.py --tag imm-seg --integrator euler --kib 262144 1048576 --sched seg >> gpurun_out/tune_imm.jsonl 2>&1
python tools/tune.py --tag imm --integrator rk4 --kib 65536 --n-it 3000 --reps 2 >> gpurun_out/tune_imm.jsonl 2>&1
python bench.py > gpurun_out/bench_c4_r02c.json 2>&1
python bench.py --workload c3 --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/bench_c3_r02c.json 2>&1
python bench.py --integrator euler --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/bench_c4euler_r02c.json 2>&1
python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -c 60 --csv --log-file gpurun_out/launches_r02c.csv python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/ncu1.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:lorenz_chain_seg_kernel -s 1 -c 1 -o gpurun_out/chain_full_r02c python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/ncu2.log 2>&1 && \
ncu --set full --import-source on -k regex:lorenz_chain_seg_kernel -s 1 -c 1 -o gpurun_out/chain_full_baseclock_r02c python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/ncu3.log 2>&1
echo done
