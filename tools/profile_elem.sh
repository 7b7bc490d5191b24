# On the GPU box: one --set full capture of the element kernel, FP64 and mixed
ARGS="--no-cpu --no-sub --steps 5 --warmup 3"
PFX=${PFX:-r2q}
python bench.py $ARGS > gpurun_out/${PFX}_plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:elem_stage -s 20 -c 1 \
    -o gpurun_out/${PFX}_elem64 -f python bench.py $ARGS > gpurun_out/${PFX}_elem64.log 2>&1
echo "fp64 rc=$?"
python bench.py $ARGS --prec 32 > gpurun_out/${PFX}_plain32.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:elem_stage -s 20 -c 1 \
    -o gpurun_out/${PFX}_elem32 -f python bench.py $ARGS --prec 32 > gpurun_out/${PFX}_elem32.log 2>&1
echo "mixed rc=$?"
