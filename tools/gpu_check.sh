# One GPU-box pass: GPU suite, smoke, config 2/3 bench lines, ncu captures of the
# hot kernels per level, summarised on the box (gpurun_out/ must stay < 64 MiB).
mkdir -p gpurun_out
set -x
R=${R:-r02}
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/gpu.txt
timeout 1800 python -m pytest tests -m gpu -q -p no:cacheprovider --durations=25 ${PYTEST_ARGS} > gpurun_out/gpu_tests.log 2>&1; echo tests_rc=$? >> gpurun_out/gpu_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo rc=$? >> gpurun_out/smoke.log
[ -n "$NO_BENCH" ] && exit 0
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/bench_c2.json 2> gpurun_out/bench_c2.err
timeout 900 python bench.py --config 3 --steps 20 --warmup 5 --no-cpu > gpurun_out/bench_c3.json 2> gpurun_out/bench_c3.err
timeout 900 python bench.py --config 4 --steps 20 --warmup 5 --no-cpu > gpurun_out/bench_c4.json 2> gpurun_out/bench_c4.err
timeout 900 python bench.py --dist --steps 20 --warmup 5 --no-cpu > gpurun_out/bench_dist1.json 2> gpurun_out/bench_dist1.err
[ -n "$NO_NCU" ] && exit 0
# launch list of the bench command (cold-cache, serialised: shares, not absolutes)
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv --log-file gpurun_out/launches.csv python bench.py --steps 4 --warmup 3 --no-cpu --no-setup --no-solve > gpurun_out/launches_bench.log 2>&1
python tools/launch_summary.py gpurun_out/launches.csv > gpurun_out/launches_summary.txt 2>&1
gzip -f gpurun_out/launches.csv
for spec in "2 K0" "3 K0" "3 ISO0" "2 ISO0"; do set -- $spec
 rep=gpurun_out/prof_c$1_$2
 timeout 900 ncu --set full --import-source on --clock-control none -k regex:"spmv_kernel|vanka_patch_kernel|vanka_subwarp_kernel|vanka_fixed_kernel|vanka_gather" -o $rep python tools/prof_once.py --config $1 --level $2 > $rep.log 2>&1
 wl=$(python -c "import bench;print(bench.CONFIGS[$1]['workload'])")
 key=$wl; [ "$2" != "K0" ] && key="$wl/$2"
 python tools/ncu_traffic.py $rep.ncu-rep gpurun_out/ncu_traffic.json "$key" "ncu --set full --clock-control none, tools/prof_once.py --config $1 --level $2, second round" > $rep.traffic.txt 2>&1
 python tools/ncu_summary.py $rep.ncu-rep > $rep.summary.txt 2>&1
 ncu -i $rep.ncu-rep --page source --csv > $rep.source.csv 2>/dev/null; gzip -f $rep.source.csv
 rm -f $rep.ncu-rep
done
du -sh gpurun_out
