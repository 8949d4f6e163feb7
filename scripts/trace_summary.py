"""Summarise the SAND_T4_TRACE per-job timelines written by scripts/gpu_trace.sh."""
import sys
import numpy as np

for name in sys.argv[1:] or ["d1", "d8", "c2"]:
    t = np.loadtxt(f"gpurun_out/t4trace_{name}.txt", dtype=np.int64)
    n = int((t[:, 7] > 0).sum())
    T = t[n // 4: 3 * n // 4]
    per_step = (T[-1, 7] - T[0, 7]) / (len(T) - 1)
    med = lambda x: float(np.median(x))
    print(f"{name}: per step {per_step:.0f} clk | epi wait {med(T[:,5]-T[:,4]):.0f} | epi compute {med(T[:,6]-T[:,5]):.0f} | "
          f"publish->end {med(T[:,7]-T[:,6]):.0f} | end->next wait {med(T[1:,4]-T[:-1,7]):.0f} | "
          f"MMA issue->acc ready {med(T[:,5]-T[:,3]):.0f} | publish->MMA afull(next same slot) {med(T[2:,1]-T[:-2,6]):.0f} | "
          f"MMA afull->weights {med(T[:,2]-T[:,1]):.0f} | MMA weights->issued {med(T[:,3]-T[:,2]):.0f}")
