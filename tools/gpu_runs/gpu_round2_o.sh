set -x
for sk in 8 0 4 12 16 24 8; do
  python tools/tune.py --tag skew$sk --integrator rk4 --kib 131072 1048576 --skew $sk >> gpurun_out/tune_skew.jsonl 2>&1
done
python tools/tune.py --tag slots1776 --integrator rk4 --kib 1048576 --slots 1776 >> gpurun_out/tune_skew.jsonl 2>&1
echo done
