# 3D quick check: parity tests, frozen / training split timing at 512^2, and
# the kernel launch list of an 8-wpp run (usage: bash tools/gpu_quick3.sh TAG)
T=${1:-x}
python -m pytest tests/test_gpu_parity3.py -x -q 2>&1 | tail -5 > gpurun_out/q3_${T}_tests.log
python tools/profile3.py --grid 512 --wpp 256 --train-until 0 --modes learnable_mis > gpurun_out/q3_${T}_split.log 2>&1
python tools/profile3.py --grid 512 --wpp 64 --train-until 64 --modes learnable_mis >> gpurun_out/q3_${T}_split.log 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/q3_${T}_launches.csv python tools/profile3.py --grid 512 --wpp 8 --train-until 8 --modes learnable_mis > /dev/null 2>&1
cat gpurun_out/q3_${T}_tests.log; grep "^{" gpurun_out/q3_${T}_split.log
