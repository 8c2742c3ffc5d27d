set -x
python -m pytest tests/test_gpu_parity3.py tests/test_gpu_values_train.py -x -q 2>&1 | tail -25 > gpurun_out/r2_c3_tests.log
for a in "--wpp 256 --train-until 256 --modes learnable_mis" "--wpp 256 --train-until 0 --modes learnable_mis uniform"; do
  python tools/profile3.py --grid 512 $a >> gpurun_out/r2_c3_split.log 2>&1
done
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"wave_(geom|dir)_kernel" --launch-skip 40 --launch-count 4 -o gpurun_out/r2_ncu_wave3 python tools/profile3.py --grid 512 --wpp 8 --train-until 0 --modes learnable_mis > gpurun_out/r2_c3_ncu.log 2>&1
tail -3 gpurun_out/r2_c3_ncu.log
