# Round 2 (fourth session: ring history, zero start, result-download overlap) ncu evidence:
# run on the GPU box from the repo root, after pytest -m gpu and the bench have exited 0 without ncu.
set -x
mkdir -p gpurun_out/ncu
python -c "import sys; sys.path.insert(0,'.'); from paper_2508_08062_b200 import problems; problems.cached_config(4)"
# 1. the launch list of the bench command (configs[4]; kernels inside conditional graph nodes are invisible to ncu)
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/ncu/launches_bench_r02d.csv python bench.py --steps 2 --warmup 1 --no-config1 --no-ttt --no-cpu > gpurun_out/ncu/launches_bench.log 2>&1
# 2. configs[4], 2 eager AA-PDHG iterations: every column pass (K' x2, K x4) and row-order epilogue
#    (k_dual_epi x4, k_primal_epi) of both iterations, then the final lambda's K' passes
ncu --set full --clock-control none --import-source on -k regex:"k_spmv_pass|k_dual_epi|k_primal_epi" -c 26 -o gpurun_out/ncu/cfg4_r02d python profiles/profile_cfg.py 4 1.0 2 > gpurun_out/ncu/cfg4.log 2>&1
ncu -i gpurun_out/ncu/cfg4_r02d.ncu-rep --page raw --csv > gpurun_out/ncu/cfg4_r02d_raw.csv 2>&1
# 3. k_plain_loop (configs[1]), one launch: 8 plain iterations + the dropped speculative K1
ncu --set full --clock-control none --import-source on -k regex:k_plain_loop --launch-skip ${PLAIN_SKIP:-360} -c 1 -o gpurun_out/ncu/plain_r02d python profiles/profile_plain.py 24 ${PLAIN_WARM:-3} > gpurun_out/ncu/plain.log 2>&1
ncu -i gpurun_out/ncu/plain_r02d.ncu-rep --page raw --csv > gpurun_out/ncu/plain_r02d_raw.csv 2>&1
ncu -i gpurun_out/ncu/plain_r02d.ncu-rep --page details --csv > gpurun_out/ncu/plain_r02d_details.csv 2>&1
rm -f gpurun_out/ncu/*.ncu-rep gpurun_out/ncu/*.tmp; ls -la gpurun_out/ncu
