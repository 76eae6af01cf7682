#!/bin/bash
# Round profiling on one B200 (run under gpurun from the repo root):
#   bench line per config, ncu launch list of the same command, and one
#   `ncu --set full` capture of the J^T J p kernel the bench chose.
# Results land in gpurun_out/; profiles/summarize.py turns them into profiles/.
R=${ROUND:-r01}
mkdir -p gpurun_out
variant() { case "$1" in *jtj7_*) echo tma4;; *jtj6_*) echo gprog;; *jtj5_*) echo warp;; *jtj4_*) echo tma;; *jtj3_*) echo stream;; *jtj2_*) echo twophase;; *) echo gather;; esac; }
while read -r tag args; do
  [ -z "$tag" ] && continue
  timeout 900 python bench.py $args --steps 5 --warmup 3 ${CPU:---no-cpu-baseline} > gpurun_out/${R}_${tag}_bench.json 2> gpurun_out/${R}_${tag}_bench.err
  k=$(python -c "import json,sys; d=json.loads(open('gpurun_out/${R}_${tag}_bench.json').read().strip().splitlines()[-1]); print(d['roofline']['kernel'].split('(')[1].split(',')[0])")
  v=$(variant "$k"); echo "$tag kernel=$k variant=$v"
  MO_B200_JTJ=$v timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -s 300 -c 400 --csv \
    --log-file gpurun_out/${R}_${tag}_launches.csv python bench.py $args --steps 1 --warmup 1 --no-cpu-baseline > /dev/null 2>&1
  MO_B200_JTJ=$v timeout 900 ncu --set full --clock-control none --import-source on -k regex:"$k" -s 6 -c 1 \
    -o gpurun_out/${R}_${tag}_jtj python bench.py $args --steps 1 --warmup 1 --no-cpu-baseline > gpurun_out/${R}_${tag}_ncu.log 2>&1
  tail -1 gpurun_out/${R}_${tag}_ncu.log
done <<CFG
${CONFIGS:-arap_warp
arap_warp_8192 --size 8192
poisson --config poisson
poisson_8192 --config poisson --size 8192
sfs --config sfs
arap_mesh --config arap_mesh}
CFG
