# A/B an experiment environment variable on the 3D cfg-4 shape: bash tools/gpu_ab_env.sh VAR v1 v2 ...
V=$1; shift
for e in "$@"; do
  env $V=$e python tools/profile3.py --grid 512 --wpp 256 --train-until 0 --modes learnable_mis 2>&1 | grep "^{" | cut -c1-110 | sed "s/^/$V=$e /"
  env $V=$e python tools/profile3.py --grid 512 --wpp 32 --train-until 32 --modes learnable_mis 2>&1 | grep "^{" | cut -c1-110 | sed "s/^/$V=$e /"
done
