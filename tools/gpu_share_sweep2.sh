#!/bin/bash
# dW share / aux weight re-sweep under the epilogue-aware partition (c2 and c4, alternating, 2 reps)
mkdir -p gpurun_out
: > gpurun_out/share2.txt
for rep in 1 2; do for v in "ZTP_DW_SHARE=1.2 ZTP_AUX_WEIGHT=1.0" "ZTP_DW_SHARE=1.0 ZTP_AUX_WEIGHT=1.0" "ZTP_DW_SHARE=1.4 ZTP_AUX_WEIGHT=1.0" "ZTP_DW_SHARE=1.2 ZTP_AUX_WEIGHT=1.3" "ZTP_DW_SHARE=1.0 ZTP_AUX_WEIGHT=1.3"; do
  env $v CONFIGS="c2 c4" bash tools/gpu_configs.sh > /dev/null 2>&1
  sed "s/^/$v rep$rep | /" gpurun_out/configs.txt | cut -c1-150 >> gpurun_out/share2.txt
done; done
cat gpurun_out/share2.txt
