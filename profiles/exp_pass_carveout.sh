# configs[4]: shared-memory carve-out of the column-pass kernels (AAPDHG_CARVEOUT: -1 = driver default,
# 0 / 10 = % of the maximum, the rest is L1): per-iteration device timestamps (exp_cfg4_iters.py)
mkdir -p gpurun_out/r02d
for rep in 1; do for cv in -1 0 10 25 50; do
  echo "=== AAPDHG_CARVEOUT_PASS=$cv (passes and epilogues alike) (rep $rep)"
  AAPDHG_CARVEOUT_PASS=$cv python profiles/exp_cfg4_iters.py 2>/dev/null | python -c "
import sys, statistics
plain = []
for l in sys.stdin:
    if l.startswith('---'): print(l.strip())
    elif ' aa=0 ' in l and '+' in l:
        k = int(l.split('k=')[1].split()[0]); d = float(l.rsplit('+', 1)[1])
        if k >= 2: plain.append(d)
print('plain iterations: median %.3f ms, min %.3f, n %d' % (statistics.median(plain), min(plain), len(plain)))
"
done; done > gpurun_out/r02d/pass_carveout_all.txt 2>&1
