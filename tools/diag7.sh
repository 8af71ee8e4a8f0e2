#!/bin/bash
mkdir -p gpurun_out
for k in bnd_resid bnd_solve bnd_assemble kr_gemm bnd_update bnd_panel; do
  bash tools/ncu_kernel.sh $k 8 4 2048 r2_$k > /dev/null 2>&1
  echo "$k done"
done
