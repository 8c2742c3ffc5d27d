# ncu --set full captures of the final build's 3D kernels (one launch each):
# the geometry / direction pair in bench.py's own cfg-4 command (a training
# round), the same pair at a full pool (frozen rounds), and the drain kernel.
# Graph-body kernels are visible only with WOSTGPU_PROFILE_LOOP=1.
T=${1:-x}
export WOSTGPU_PROFILE_LOOP=1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"wave_(geom|dir)_kernel" --launch-skip 600 --launch-count 2 --kill 1 -o gpurun_out/${T}_ncu_bench_cfg4 python bench.py --steps 1 --warmup 0 --no-cfg2 --no-cpu-baseline > gpurun_out/${T}_ncu_bench.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"wave_(geom|dir)_kernel" --launch-skip 40 --launch-count 2 -o gpurun_out/${T}_ncu_frozen_cfg4 python tools/profile3.py --grid 512 --wpp 16 --train-until 0 --modes learnable_mis > gpurun_out/${T}_ncu_frozen.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"wave_tail_kernel" --launch-skip 2 --launch-count 1 -o gpurun_out/${T}_ncu_tail python tools/profile3.py --grid 512 --wpp 4 --train-until 4 --modes learnable_mis > gpurun_out/${T}_ncu_tail.log 2>&1
ls gpurun_out/ | grep "^${T}_"
