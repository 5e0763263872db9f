#!/bin/bash
# ncu evidence for the config-4 step (run on the GPU box from the repo root):
#   launch list of the whole --ncu run (last step = after the last k_sigma)
#   and one --set full capture per hot kernel from the last timed step.
# usage: tools/profile_r02.sh TAG
set -u
TAG=${1:-r02}
B="python bench.py --ncu --steps 2 --warmup 1"
mkdir -p gpurun_out
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_$TAG.csv $B > gpurun_out/ncu_$TAG.log 2>&1
echo "launch list rc=$?"
# guard + 1 warm-up + 2 timed = 4 steps: skip 3 instances of a once-per-step kernel
for K in k_basis_tc k_basis_bwd k_grad_block k_edge_weights_tile k_skel_lines k_points_restrict_w; do
  ncu --set full --clock-control none --import-source on -k regex:"$K" --launch-skip 3 -c 1 \
      -o gpurun_out/${TAG}_$K $B >> gpurun_out/ncu_$TAG.log 2>&1
  echo "$K rc=$?"
done
# coarse kernels launch several times per step
ncu --set full --clock-control none -k regex:"k_mf_solve_coop" --launch-skip 6 -c 2 -o gpurun_out/${TAG}_k_mf_solve_coop $B >> gpurun_out/ncu_$TAG.log 2>&1
ncu --set full --clock-control none -k regex:"k_mf_factor|k_mf_inv" --launch-skip 60 -c 20 -o gpurun_out/${TAG}_k_mf_factor $B >> gpurun_out/ncu_$TAG.log 2>&1
# summaries on the box (reports are large); keep the basis-kernel report only
python tools/ncu_summary.py gpurun_out/launches_$TAG.csv $(ls gpurun_out/${TAG}_*.ncu-rep | paste -sd,) gpurun_out/$TAG >> gpurun_out/ncu_$TAG.log 2>&1
for f in gpurun_out/${TAG}_*.ncu-rep; do
  case $f in *k_basis_tc*) ;; *) rm -f $f ;; esac
done
echo done
