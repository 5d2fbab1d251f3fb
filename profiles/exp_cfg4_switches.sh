# configs[4]: the split-epilogue switches re-measured on the final code (partial preload on):
# per-iteration device timestamps of the bench's solves (exp_cfg4_iters.py)
mkdir -p gpurun_out/r02d
for rep in 1 2; do for sw in "AAPDHG_EPI_PIPE=1" "AAPDHG_EPI_PIPE=0" "AAPDHG_SPLIT_EPI=0" "AAPDHG_PDL=0"; do
  echo "=== $sw (rep $rep)"
  env $sw python profiles/exp_cfg4_iters.py 2>/dev/null | python -c "
import sys, statistics
plain = []
for l in sys.stdin:
    if l.startswith('---'): print(l.strip())
    elif ' aa=0 ' in l and '+' in l:
        k = int(l.split('k=')[1].split()[0]); d = float(l.rsplit('+', 1)[1])
        if k >= 2: plain.append(d)
print('plain iterations: median %.3f ms, min %.3f, n %d' % (statistics.median(plain), min(plain), len(plain)))
"
done; done > gpurun_out/r02d/cfg4_switches.txt 2>&1
