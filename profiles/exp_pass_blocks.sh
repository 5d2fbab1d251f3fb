# configs[4] block sizes (KB of x per K pass / of y per K' pass) with the partial preload on:
# per-iteration device timestamps of the bench's solves (exp_cfg4_iters.py)
mkdir -p gpurun_out/r02d
for blk in "109300 81920" "81920 81920" "109300 109300" "160000 81920"; do
  set -- $blk
  echo "=== K blocks $1 KB, K' blocks $2 KB"
  AAPDHG_L2_BLOCK_KB_K=$1 AAPDHG_L2_BLOCK_KB_KT=$2 python profiles/exp_cfg4_iters.py 2>/dev/null | python -c "
import sys, statistics
plain = []
for l in sys.stdin:
    if l.startswith('---'): print(l.strip())
    elif ' aa=0 ' in l and '+' in l:
        k = int(l.split('k=')[1].split()[0]); d = float(l.rsplit('+', 1)[1])
        if k >= 2: plain.append(d)
print('plain iterations: median %.3f ms, min %.3f, n %d' % (statistics.median(plain), min(plain), len(plain)))
"
done > gpurun_out/r02d/pass_blocks2.txt 2>&1
