set -x
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_final2.log 2>&1
python -m pytest tests -m gpu -q -x --durations=10 > gpurun_out/pytest_gpu_final2.log 2>&1
python bench.py --steps 20 --warmup 5 > gpurun_out/bench_final2_c4.json 2> gpurun_out/bench_final2_c4.err
python bench.py --workload c3 --steps 10 --warmup 3 > gpurun_out/bench_final2_c3.json 2>&1
python bench.py --workload c5 --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/bench_final2_c5.json 2>&1
python bench.py --integrator rk4fma --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/bench_final2_c4fma.json 2>&1
python bench.py --impl reference --steps 20 --warmup 5 > gpurun_out/bench_final2_ref.json 2>&1
python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29561 bench.py --gpus 1 --steps 5 --warmup 3 > gpurun_out/bench_final2_torchrun1.json 2>&1
echo done
