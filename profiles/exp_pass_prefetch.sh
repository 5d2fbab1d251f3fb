mkdir -p gpurun_out/r02d
python -c "import sys; sys.path.insert(0,'.'); from paper_2508_08062_b200 import problems; problems.cached_config(4)"
for rep in 1 2; do
for pf in 0 1; do
for blk in "81920 81920" "81920 55000" "65536 55000" "49152 40960" "40960 40960"; do
set -- $blk
echo "PASS_PREFETCH=$pf K=$1 KT=$2" 
AAPDHG_PASS_PREFETCH=$pf AAPDHG_L2_BLOCK_KB_K=$1 AAPDHG_L2_BLOCK_KB_KT=$2 python profiles/exp_cfg4_l2.py 81920,0
done; done; done > gpurun_out/r02d/pass_prefetch.txt 2>&1
