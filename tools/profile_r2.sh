# On the GPU box: launch list of the bench step, then one --set full capture
# per stage kernel (FP64 and mixed).  Outputs gpurun_out/${PFX}_*.
set -u
PFX=${PFX:-r2p}
ARGS="--no-cpu --no-sub --steps 5 --warmup 3"
python bench.py $ARGS > gpurun_out/${PFX}_plain.log 2>&1 || { echo "plain failed"; exit 1; }
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/${PFX}_launches.csv \
    python bench.py $ARGS > gpurun_out/${PFX}_launches.log 2>&1
echo "launches rc=$?"
ncu --set full --clock-control none --import-source on -k regex:"elem_stage|face_flux" -s 60 -c 2 \
    -o gpurun_out/${PFX}_fp64 -f python bench.py $ARGS > gpurun_out/${PFX}_fp64.log 2>&1
echo "fp64 rc=$?"
python bench.py $ARGS --prec 32 > gpurun_out/${PFX}_plain32.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"elem_stage|face_flux" -s 60 -c 2 \
    -o gpurun_out/${PFX}_mixed -f python bench.py $ARGS --prec 32 > gpurun_out/${PFX}_mixed.log 2>&1
echo "mixed rc=$?"
# warm-cache DRAM traffic per launch (no cache flush between replays)
ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum,lts__t_sector_hit_rate.pct \
    --cache-control none --clock-control none -k regex:"elem_stage|face_flux" -s 60 -c 12 --csv \
    --log-file gpurun_out/${PFX}_warm_traffic.csv python bench.py $ARGS > gpurun_out/${PFX}_warm.log 2>&1
echo "warm rc=$?"
