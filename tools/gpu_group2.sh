#!/bin/bash
mkdir -p gpurun_out
rm -f gpurun_out/group_tl2.txt
for cfg in "ZTP_GROUP=1 ZTP_GROUP_DROP=0" "ZTP_GROUP=1 ZTP_GROUP_DROP=1" "ZTP_GROUP=1 ZTP_GROUP_DROP=2" "ZTP_CONC=0 ZTP_GROUP=0"; do
  echo "== $cfg" >> gpurun_out/group_tl2.txt
  env $cfg timeout -s KILL 300 python tools/graph_timeline.py >> gpurun_out/group_tl2.txt 2>&1
done
