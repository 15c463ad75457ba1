# compute-sanitizer over the GPU tests of the kernels added or changed in
# round 2, at sizes the tools finish quickly (usage: bash tools/gpu_sanitize.sh;
# output: gpurun_out/sanitize.txt)
cd ${GRAFT_REPO_ROOT:-.}
mkdir -p gpurun_out
SEL="tests/test_univ_f64.py tests/test_gen_kernel.py
     tests/test_sharding.py::test_sharded_stop_criteria_match_single_engine
     tests/test_univ_sliced.py::test_truth_table_equals_adder_and_lane_per_solution
     tests/test_replay_full.py::test_replay_full_size_matches_reference"
for tool in memcheck synccheck initcheck racecheck; do
  echo "== $tool" >> gpurun_out/sanitize.txt
  timeout 2400 compute-sanitizer --tool $tool --print-limit 10 python -m pytest $SEL -q -p no:cacheprovider \
    -k "not c3_full and not c5_n1024" >> gpurun_out/sanitize.txt 2>&1
  echo "rc=$?" >> gpurun_out/sanitize.txt
done
