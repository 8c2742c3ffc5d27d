# Round-end style evidence: the default bench line, then ncu captures of the
# 3D kernels at the bench configuration (cfg 4: bench.py's own command,
# training rounds) and in frozen rounds (profile3.py, same scene and slice),
# plus the cfg 2 launch list. Usage: bash tools/gpu_bench_profile.sh TAG
T=${1:-x}
python bench.py > gpurun_out/${T}_bench.json 2> gpurun_out/${T}_bench.err || exit 1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"wave_(geom|dir)_kernel" --launch-skip 600 --launch-count 2 --kill 1 -o gpurun_out/${T}_ncu_bench_cfg4 python bench.py --steps 1 --warmup 0 --no-cfg2 --no-cpu-baseline > gpurun_out/${T}_ncu_bench.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"wave_(geom|dir)_kernel" --launch-skip 20 --launch-count 2 -o gpurun_out/${T}_ncu_frozen_cfg4 python tools/profile3.py --grid 512 --wpp 16 --train-until 0 --modes learnable_mis > gpurun_out/${T}_ncu_frozen.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/${T}_launches_cfg2.csv python bench.py --workload cfg2 --steps 1 --warmup 1 --no-cpu-baseline > /dev/null 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/${T}_launches_cfg4_w16.csv python tools/profile3.py --grid 512 --wpp 16 --train-until 4 --modes learnable_mis > /dev/null 2>&1
ls gpurun_out/ | grep "^${T}_"
