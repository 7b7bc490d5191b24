# On the GPU box: --set full of the P3 FP64 stage kernels (n = 40 cube)
ARGS="--no-cpu --no-sub --steps 5 --warmup 3 --order 3 --n 40"
python bench.py $ARGS > gpurun_out/r2p3_plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"elem_stage|face_flux_kernel<double, false" -s 20 -c 2 \
    -o gpurun_out/r2p3_fp64 -f python bench.py $ARGS > gpurun_out/r2p3_fp64.log 2>&1
echo "p3 rc=$?"
