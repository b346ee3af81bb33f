set -x
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_r02b.log 2>&1
python -m pytest tests -m gpu -q -x --durations=10 > gpurun_out/pytest_gpu_r02f.log 2>&1
python bench.py > gpurun_out/bench_c4_r02b.json 2> gpurun_out/bench_c4_r02b.err
python bench.py --workload c3 --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/bench_c3_r02b.json 2>&1
python bench.py --workload c3 --integrator rk4fma --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/bench_c3fma_r02b.json 2>&1
python bench.py --workload c5 --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/bench_c5_r02e.json 2>&1
python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/bench_ref_r02.json 2>&1
echo done
