# Targeted GPU pass: selected test files ($TESTS), bench lines ($BENCH_CONFIGS),
# one ncu capture ($NCU_SPEC, e.g. "3 K0"), extra commands ($EXTRA).
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/gpu.txt
if [ "$TESTS" != "none" ]; then
  timeout 1500 python -m pytest ${TESTS:-tests} -m gpu -q -p no:cacheprovider --durations=10 > gpurun_out/gpu_tests.log 2>&1; echo tests_rc=$? >> gpurun_out/gpu_tests.log
fi
for c in ${BENCH_CONFIGS:-2 3}; do
  timeout 900 python bench.py --config $c --steps 20 --warmup 5 --no-cpu --no-setup > gpurun_out/bench_c$c.json 2> gpurun_out/bench_c$c.err
done
if [ -n "$EXTRA" ]; then bash -c "$EXTRA" > gpurun_out/extra.log 2>&1; fi
if [ -n "$NCU_SPEC" ]; then set -- $NCU_SPEC
 rep=gpurun_out/prof_c$1_$2
 timeout 900 ncu --set full --import-source on --clock-control none -k regex:"spmv_kernel|vanka_patch_kernel|vanka_subwarp_kernel|vanka_fixed_kernel|vanka_gather" -o $rep python tools/prof_once.py --config $1 --level $2 > $rep.log 2>&1
 wl=$(python -c "import bench;print(bench.CONFIGS[$1]['workload'])")
 key=$wl; [ "$2" != "K0" ] && key="$wl/$2"
 python tools/ncu_traffic.py $rep.ncu-rep gpurun_out/ncu_traffic.json "$key" "ncu --set full --clock-control none, tools/prof_once.py --config $1 --level $2, second round" > $rep.traffic.txt 2>&1
 python tools/ncu_summary.py $rep.ncu-rep > $rep.summary.txt 2>&1
 ncu -i $rep.ncu-rep --page source --csv > $rep.source.csv 2>/dev/null; gzip -f $rep.source.csv
 rm -f $rep.ncu-rep
fi
du -sh gpurun_out
