set -x
mkdir -p gpurun_out/ncu
# 1. the launch list of the bench command (graph kernels with conditional nodes are invisible to ncu)
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/ncu/launches_bench_r02.csv python bench.py --steps 2 --warmup 1 --no-config4 --no-ttt --no-cpu > gpurun_out/ncu/launches_bench.log 2>&1
# 2. k_plain_loop, one launch (8 plain iterations + the dropped speculative K1)
ncu --set full --clock-control none --import-source on -k regex:k_plain_loop -c 1 -o gpurun_out/ncu/plain_r02 python profiles/profile_plain.py 24 > gpurun_out/ncu/plain.log 2>&1
ncu -i gpurun_out/ncu/plain_r02.ncu-rep --page details --csv > gpurun_out/ncu/plain_r02_details.csv 2>&1
ncu -i gpurun_out/ncu/plain_r02.ncu-rep --page raw --csv > gpurun_out/ncu/plain_r02_raw.csv 2>&1
# 3. configs[4]: the K' / K column passes and the fused last blocks
python -c "import sys; sys.path.insert(0,'.'); from paper_2508_08062_b200 import problems; problems.cached_config(4)"
ncu --set full --clock-control none -k regex:"k_spmv_pass|k_dual_side|k_primal_side" -c 8 -o gpurun_out/ncu/cfg4_r02 python profiles/profile_cfg.py 4 1.0 2 > gpurun_out/ncu/cfg4.log 2>&1
ncu -i gpurun_out/ncu/cfg4_r02.ncu-rep --page raw --csv > gpurun_out/ncu/cfg4_r02_raw.csv 2>&1
# 4. configs[2] FAA: the double-double Gram
ncu --set full --clock-control none -k regex:"k_gram_dots_dd|k_aa_solve" -c 4 -o gpurun_out/ncu/cfg2_faa_r02 python profiles/profile_cfg.py 2 1.0 40 > gpurun_out/ncu/cfg2.log 2>&1
ncu -i gpurun_out/ncu/cfg2_faa_r02.ncu-rep --page raw --csv > gpurun_out/ncu/cfg2_faa_r02_raw.csv 2>&1
ls -la gpurun_out/ncu
