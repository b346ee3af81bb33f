set -x
python -m pytest tests/test_gpu_parity.py tests/test_gpu_multirank.py -q -x -k "host or torchrun or two_ranks" > gpurun_out/pytest_l.log 2>&1
echo done
