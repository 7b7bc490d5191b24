# on the box: plain run then one `ncu --set full` capture of a kernel
# usage: bash tools/ncu_box.sh OUTNAME KERNEL_REGEX "<bench args>" [skip]
OUT=$1; K=$2; ARGS=$3; SKIP=${4:-6}
python bench.py --no-cpu --steps 2 --warmup 3 $ARGS > gpurun_out/${OUT}_plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:$K -s $SKIP -c 1 -o gpurun_out/$OUT -f \
    python bench.py --no-cpu --steps 2 --warmup 3 $ARGS > gpurun_out/${OUT}_ncu.log 2>&1
echo "ncu rc=$?"
