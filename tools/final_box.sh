# On the box: the whole GPU suite, the default bench line, smoke(), and the ncu
# evidence (launch list + --set full of the stage kernels + warm traffic)
timeout 2400 python -m pytest tests -m gpu -q > gpurun_out/r2z_gputests.log 2>&1; echo "tests rc=$?"
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2z_smoke.log 2>&1; echo "smoke rc=$?"
python bench.py --roofline-csv gpurun_out/r2z_roofline.csv > gpurun_out/r2z_bench.json 2> gpurun_out/r2z_bench.err; echo "bench rc=$?"
python bench.py --impl reference > gpurun_out/r2z_ref.json 2> gpurun_out/r2z_ref.err; echo "ref rc=$?"
bash tools/profile_r2.sh
bash tools/profile_elem.sh
