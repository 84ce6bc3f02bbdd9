# One GPU-box pass: GPU suite, smoke, config 2/3 bench lines, ncu captures of the
# hot kernels per level (read back with tools/ncu_traffic.py / ncu_summary.py).
mkdir -p gpurun_out
set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/gpu.txt
timeout 1500 python -m pytest tests -m gpu -x -q -p no:cacheprovider --durations=15 > gpurun_out/gpu_tests.log 2>&1; echo tests_rc=$? >> gpurun_out/gpu_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo rc=$? >> gpurun_out/smoke.log
timeout 600 python bench.py --steps 20 --warmup 5 > gpurun_out/bench_c2.json 2> gpurun_out/bench_c2.err
timeout 600 python bench.py --config 3 --steps 20 --warmup 5 --no-cpu > gpurun_out/bench_c3.json 2> gpurun_out/bench_c3.err
for spec in "2 K0" "3 K0" "3 ISO0" "2 ISO0"; do set -- $spec
 timeout 600 ncu --set full --import-source on --clock-control none -k regex:"spmv_kernel|vanka_patch_kernel|vanka_subwarp_kernel|vanka_gather" -o gpurun_out/prof_c$1_$2 python tools/prof_once.py --config $1 --level $2 > gpurun_out/prof_c$1_$2.log 2>&1
done
