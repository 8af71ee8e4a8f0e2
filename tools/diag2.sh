#!/bin/bash
mkdir -p gpurun_out
timeout 600 python -m pytest -q -p no:cacheprovider tests/test_gpu_ordering.py "tests/test_gpu_parity.py::test_ragged_shapes" "tests/test_gpu_parity.py::test_standard_arm_config3_ablation" "tests/test_gpu_parity.py::test_standard_arm_backward_matches_oracle" "tests/test_gpu_parity.py::test_initialization_point_matches_oracle" -s > gpurun_out/diag2_pytest.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/diag2_pytest.log
QPB200_PHASE_PROFILE=1 timeout 300 python tools/run_cfg.py 4 1184 > gpurun_out/diag_prof4.log 2>&1; echo "p4 rc=$?"
QPB200_PHASE_PROFILE=1 timeout 300 python tools/run_cfg.py 2 1024 > gpurun_out/diag_prof2.log 2>&1; echo "p2 rc=$?"
TOOLS="memcheck racecheck synccheck initcheck" timeout 1800 bash tools/sanitize.sh > gpurun_out/sanitize_r2.log 2>&1; echo "san rc=$?"
