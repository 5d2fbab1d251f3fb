# configs[4]: shared-memory carve-out of the column-pass kernels (an experiment build that set
# cudaFuncAttributePreferredSharedMemoryCarveout on k_spmv_pass / k_spmv (and, for pass_carveout_all.txt,
# on the row-order epilogues) from this variable; the shipped code leaves them at the driver default):
# per-iteration device timestamps (exp_cfg4_iters.py). Results: profiles/r02d/pass_carveout*.txt
mkdir -p gpurun_out/r02d
for rep in 1; do for cv in -1 0 10 25; do
  echo "=== AAPDHG_CARVEOUT=$cv (rep $rep)"
  AAPDHG_CARVEOUT=$cv python profiles/exp_cfg4_iters.py 2>/dev/null | python -c "
import sys, statistics
plain = []
for l in sys.stdin:
    if l.startswith('---'): print(l.strip())
    elif ' aa=0 ' in l and '+' in l:
        k = int(l.split('k=')[1].split()[0]); d = float(l.rsplit('+', 1)[1])
        if k >= 2: plain.append(d)
print('plain iterations: median %.3f ms, min %.3f, n %d' % (statistics.median(plain), min(plain), len(plain)))
"
done; done > gpurun_out/r02d/pass_carveout.txt 2>&1
