set -x
python tools/fig1.py > gpurun_out/fig1_r02.jsonl 2>&1
python tools/fig1.py --lanes 170496 >> gpurun_out/fig1_r02.jsonl 2>&1
python tools/fig1.py --lanes 340992 >> gpurun_out/fig1_r02.jsonl 2>&1
python tools/fig1.py --lanes 65536 --samples 20 > gpurun_out/plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:digit_hist -s 1 -c 1 -o gpurun_out/fig1_full_r02 python tools/fig1.py --lanes 262144 > gpurun_out/ncu_f.log 2>&1
echo done
