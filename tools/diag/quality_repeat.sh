# repeated 8-seed cfg-2 quality runs: tensor walks + tensor training, tensor
# walks + CUDA-core training, exact path (diagnostic)
for r in 1 2; do
  python tools/quality_cfg2.py --seeds 1 2 3 4 5 6 7 8 2>/dev/null | grep -v '^{"grid' > gpurun_out/qr_tc_$r.log
  WOSTGPU_GRAD=cuda python tools/quality_cfg2.py --seeds 1 2 3 4 5 6 7 8 2>/dev/null | grep -v '^{"grid' > gpurun_out/qr_tcw_cudagrad_$r.log
done
