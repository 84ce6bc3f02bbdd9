# compute-sanitizer memcheck / racecheck / synccheck over smoke() and the
# n <= 64 GPU tests that exercise the bulk-copy rings (Vanka patch and
# sub-warp kernels), the dof-ordered gather, the cluster-launch scalar tail
# (DSMEM), the whole-solve graph, the FEM sort, and the two-rank IPC
# reverse halo (vanka_gather_push_kernel). Logs: gpurun_out/sanitize_*.log
mkdir -p gpurun_out
CS="compute-sanitizer --target-processes all --print-limit 50 --error-exitcode 9"
SEL="tests/test_gpu_parity.py::test_apply_vanka_parity tests/test_gpu_parity.py::test_apply_vanka_subwarp_classes tests/test_gpu_parity.py::test_apply_vanka_sv_subwarp tests/test_gpu_parity.py::test_vanka_spmv_step tests/test_gpu_parity.py::test_dc_apply_parity tests/test_gpu_parity.py::test_sv_scalar_tail tests/test_gpu_parity.py::test_factor_payload_bitwise tests/test_gpu_fem.py::test_sort_permutation_is_std_sort tests/test_gpu_fem.py::test_assembly_bitwise"
DIST="tests/test_gpu_dist.py"
for tool in memcheck racecheck synccheck; do
  log=gpurun_out/sanitize_${tool}.log
  echo "== smoke" > $log
  timeout 1200 $CS --tool $tool python -c "import __graft_entry__ as g; g.smoke()" >> $log 2>&1; echo "smoke rc=$?" >> $log
  echo "== tests" >> $log
  timeout 2400 $CS --tool $tool python -m pytest -q -p no:cacheprovider -m gpu -k "not 64 or scalar_tail" $SEL >> $log 2>&1; echo "tests rc=$?" >> $log
  if [ "$tool" = memcheck ]; then
    echo "== dist (two ranks on one GPU: IPC peer halo)" >> $log
    timeout 1800 $CS --tool $tool python -m pytest -q -p no:cacheprovider -m gpu -k "gloo" $DIST >> $log 2>&1; echo "dist rc=$?" >> $log
  fi
  grep -E "ERROR SUMMARY|rc=" $log
done
