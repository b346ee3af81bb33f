set -x
for rep in 1 2; do
for v in default h1 h2; do
  lib=""; [ $v != default ] && lib=tools/variants/liblorenz_$v.so
  echo "{\"lib\": \"$v\"}" >> gpurun_out/fig1_h.jsonl
  LORENZ_LIB=$lib python tools/fig1.py >> gpurun_out/fig1_h.jsonl 2>&1
  LORENZ_LIB=$lib python tools/fig1.py --lanes 340992 >> gpurun_out/fig1_h.jsonl 2>&1
done
done
LORENZ_LIB=tools/variants/liblorenz_h1.so python -m pytest tests/test_gpu_fig1.py -q > gpurun_out/pytest_h1.log 2>&1
echo done
