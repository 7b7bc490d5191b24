#!/bin/bash
# On the GPU box: plain run, then the ncu launch list, then one full capture
# of the two stage kernels.  Outputs under gpurun_out/.
#   tools/profile.sh <tag> <bench args...>
set -u
TAG=$1; shift
ARGS="$@"
mkdir -p gpurun_out
python bench.py $ARGS > gpurun_out/${TAG}_plain.log 2>&1 || { echo "plain run failed"; tail -5 gpurun_out/${TAG}_plain.log; exit 1; }
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/${TAG}_launches.csv \
    python bench.py $ARGS > gpurun_out/${TAG}_ncu_launches.log 2>&1
echo "launch list rc=$?"
ncu --set full --clock-control none --import-source on -k regex:"elem_stage|face_flux" -s 20 -c 2 \
    -o gpurun_out/${TAG}_full python bench.py $ARGS > gpurun_out/${TAG}_ncu_full.log 2>&1
echo "full capture rc=$?"
