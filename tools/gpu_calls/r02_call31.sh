# round 2, call 31: sanitizers on the launch-overlap path (programmatic dependent launch, first-wave
# L2 bulk prefetch, late trigger) and the dist world-1 path under the new default
set -x
T="tests/test_gpu_parity.py::test_launch_overlap_dependent_chain"
timeout 1500 compute-sanitizer --tool memcheck --error-exitcode 9 python -m pytest "$T" tests/test_gpu_dist_world1.py -x -q > gpurun_out/r02c31_memcheck.txt 2>&1; echo "rc=$?" >> gpurun_out/r02c31_memcheck.txt
timeout 1500 compute-sanitizer --tool racecheck --error-exitcode 9 python -m pytest "$T" -x -q > gpurun_out/r02c31_racecheck.txt 2>&1; echo "rc=$?" >> gpurun_out/r02c31_racecheck.txt
timeout 1500 compute-sanitizer --tool synccheck --error-exitcode 9 python -m pytest "$T" -x -q > gpurun_out/r02c31_synccheck.txt 2>&1; echo "rc=$?" >> gpurun_out/r02c31_synccheck.txt
