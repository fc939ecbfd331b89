#!/bin/bash
# compute-sanitizer evidence (memcheck / racecheck / synccheck) on representative GPU tests:
# strip operators (2D/3D), the persistent damage PCG and coarse V-cycle, Newton (device MINRES),
# the element-list path.  Logs -> gpurun_out/sanitize/, summary -> gpurun_out/sanitize/summary.txt
mkdir -p gpurun_out/sanitize
S=/usr/local/cuda/bin/compute-sanitizer
run() {  # tool tag pytest-args...
  local tool=$1 tag=$2; shift 2
  timeout 900 $S --tool $tool --error-exitcode 99 --print-limit 50 --log-file gpurun_out/sanitize/${tool}_${tag}.log \
    python -m pytest -x -q -p no:cacheprovider "$@" > gpurun_out/sanitize/${tool}_${tag}.pytest.log 2>&1
  local rc=$?
  echo "$tool $tag rc=$rc $(tail -n 1 gpurun_out/sanitize/${tool}_${tag}.pytest.log)" >> gpurun_out/sanitize/summary.txt
}
: > gpurun_out/sanitize/summary.txt
run memcheck ops2d "tests/test_gpu_ops.py::test_operator_parity"
run memcheck ops3d tests/test_gpu_ops3d.py -k "3x4x5 or 1x1x1"
run memcheck solvers tests/test_gpu_solvers.py -k "persistent_damage_pcg and 20 or persistent_coarse_cycle and 57 or damage_step_matches or coupled_newton_matches or device_minres"
run memcheck umesh tests/test_umesh.py -m gpu -k "parity_vs_oracle or damage"
run racecheck ops2d "tests/test_gpu_ops.py::test_operator_parity" -k "crossed"
run racecheck solvers tests/test_gpu_solvers.py -k "persistent_damage_pcg and 20 and crossed or persistent_coarse_cycle and 57 and crossed"
run racecheck ops3d tests/test_gpu_ops3d.py -k "3x4x5"
run synccheck ops2d "tests/test_gpu_ops.py::test_operator_parity" -k "crossed"
run synccheck solvers tests/test_gpu_solvers.py -k "persistent_damage_pcg and 20 and crossed or persistent_coarse_cycle and 57 and crossed"
run synccheck umesh tests/test_umesh.py -m gpu -k "parity_vs_oracle"
cat gpurun_out/sanitize/summary.txt
