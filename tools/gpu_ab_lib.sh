# A/B two builds of the library on the 3D cfg-4 shape: usage bash tools/gpu_ab_lib.sh LIB_A LIB_B
for lib in "$@"; do
  WOSTGPU_LIB=$lib python tools/profile3.py --grid 512 --wpp 256 --train-until 0 --modes learnable_mis uniform 2>&1 | grep "^{" | cut -c1-130 | sed "s|^|$(basename $lib) |"
  WOSTGPU_LIB=$lib python tools/profile3.py --grid 512 --wpp 32 --train-until 32 --modes learnable_mis 2>&1 | grep "^{" | cut -c1-130 | sed "s|^|$(basename $lib) |"
done
