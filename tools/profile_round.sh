# Round-end measurement recipe (run on the GPU box from the repo root):
# GPU tests, the default bench, the ncu launch list of a bench run, and one
# full ncu capture of the hot kernels (LR train step kernels and the 256^3
# render's binning + whole-brick forward, via kbench).  Outputs land in
# gpurun_out/; summaries go to profiles/ (tools/ncu_summary.py).
set -x
python -m pytest tests -m gpu -x -q 2>&1 | tail -4 > gpurun_out/final_gpu_tests.log
python bench.py > gpurun_out/final_bench.log 2>&1
echo bench rc=$?
ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv --log-file gpurun_out/final_launches.csv python bench.py --steps 3 --warmup 3 --no-render512 --no-cpu --no-count --no-e2e > gpurun_out/final_launch_run.log 2>&1
echo launches rc=$?
timeout 900 ncu --set full --import-source on --clock-control none -k regex:"forward32_kernel|backward32m|tail_tma|emit_warp|preprocess_kernel|forward32w|Onesweep" -c 14 -o gpurun_out/r01_final5 python tools/kbench.py --iters 1 --hr > gpurun_out/ncu_final5.log 2>&1
echo ncu rc=$?
cat gpurun_out/final_gpu_tests.log
