# A/B of AAPDHG_PASS_PREFETCH (0 off, 2 L2 prefetch, 3 register preload of a later column pass's row
# partial; 3 is the default) on configs[4]: per-iteration device timestamps of the bench's solves
# (exp_cfg4_iters.py). Results: profiles/r02d/pass_prefetch_modes.txt. (The unroll-8 variant of
# profiles/r02d/pass_unroll8.txt was an experiment build of k_spmv_pass, since removed.)
mkdir -p gpurun_out/r02d
for rep in 1 2; do for pf in 0 2 3; do
  echo "=== AAPDHG_PASS_PREFETCH=$pf (rep $rep)"
  AAPDHG_PASS_PREFETCH=$pf python profiles/exp_cfg4_iters.py 2>/dev/null | python -c "
import sys, statistics
plain = []
for l in sys.stdin:
    if l.startswith('---'): print(l.strip())
    elif ' aa=0 ' in l and '+' in l:
        k = int(l.split('k=')[1].split()[0]); d = float(l.rsplit('+', 1)[1])
        if k >= 2: plain.append(d)
print('plain iterations: median %.3f ms, min %.3f, n %d' % (statistics.median(plain), min(plain), len(plain)))
"
done; done > gpurun_out/r02d/pass_prefetch_modes.txt 2>&1
