"""Structure of the sequential greedy on a bench queue (design input for greedy.cu):
where in the descending key order the picks land, and how many keys a scan sees
if keys blocked at the start of each window of the sorted order are dropped.
usage: python tools/greedy_stats.py C4 5000"""
import ctypes
import os
import subprocess
import sys
import time

import numpy as np
import torch

sys.path.insert(0, '.')
import paper_2405_03838_b200 as cs  # noqa: E402
from synth import bench_config  # noqa: E402

SRC = r'''
#include <stdint.h>
#include <string.h>
#include <stdlib.h>
// order: set ids in greedy (key) order; pairs decoded by colex
static void unrank2(int64_t id, int64_t* a, int64_t* b) {
  int64_t j = (int64_t)((1.0 + __builtin_sqrt(1.0 + 8.0 * (double)id)) * 0.5);
  while (j * (j - 1) / 2 > id) j--;
  while ((j + 1) * j / 2 <= id) j++;
  *b = j; *a = id - j * (j - 1) / 2;
}
// returns number of picks; pos[t] = index of pick t in the order; free_at[w] = keys with both jobs
// free at the start of window w (window = wsize keys) within window w
int64_t run(const int64_t* order, int64_t n, int64_t n_jobs, int64_t k, int64_t* pos, int64_t wsize, int64_t* free_in_win, int64_t nwin) {
  char* taken = calloc(n_jobs, 1);
  int64_t np = 0;
  for (int64_t w = 0; w < nwin && np < k; w++) {
    int64_t lo = w * wsize, hi = lo + wsize < n ? lo + wsize : n;
    int64_t f = 0;
    for (int64_t i = lo; i < hi; i++) { int64_t a, b; unrank2(order[i], &a, &b); if (!taken[a] && !taken[b]) f++; }
    free_in_win[w] = f;
    for (int64_t i = lo; i < hi && np < k; i++) {
      int64_t a, b; unrank2(order[i], &a, &b);
      if (!taken[a] && !taken[b]) { taken[a] = taken[b] = 1; pos[np++] = i; }
    }
  }
  free(taken);
  return np;
}
'''
so = '/tmp/greedy_stats.so'
open('/tmp/greedy_stats.c', 'w').write(SRC)
subprocess.check_call(['gcc', '-O2', '-shared', '-fPIC', '/tmp/greedy_stats.c', '-o', so, '-lm'])
L = ctypes.CDLL(so)
L.run.restype = ctypes.c_int64
P = ctypes.c_void_p
I64 = ctypes.c_int64
L.run.argtypes = [P, I64, I64, I64, P, I64, P, I64]

name = sys.argv[1] if len(sys.argv) > 1 else "C4"
k = int(sys.argv[2]) if len(sys.argv) > 2 else 5000
pb, F = bench_config(name)
s = cs.Scheduler(pb)
obj, cfg = s.score_all(torch.from_numpy(F).cuda())
torch.cuda.synchronize()
ids = torch.arange(obj.numel(), device='cuda', dtype=torch.int64)
feas = obj > -float('inf')
o, i = obj[feas], ids[feas]
# descending obj, ascending id: sort by id first then stable sort by -obj
t0 = time.time()
order = i[torch.sort(-o, stable=True).indices].cpu().numpy().astype(np.int64)
n = len(order)
wsize = 4096
nwin = (n + wsize - 1) // wsize
pos = np.zeros(k, np.int64)
fw = np.zeros(nwin, np.int64)
npk = L.run(order.ctypes.data, ctypes.c_int64(n), ctypes.c_int64(F.shape[0]), ctypes.c_int64(k), pos.ctypes.data,
            ctypes.c_int64(wsize), fw.ctypes.data, ctypes.c_int64(nwin))
last = pos[npk - 1]
used = fw[: last // wsize + 1]
print(f"{name}: feasible keys {n}, picks {npk}, last pick at sorted position {last} ({last / n:.3f} of keys)")
for q in (0.1, 0.25, 0.5, 0.75, 0.9, 0.99, 1.0):
    t = int(q * npk) - 1
    print(f"  pick {t + 1:5d} at position {pos[t]:10d}")
print(f"  keys free at their window's start (windows of {wsize}) up to the last pick: {used.sum()} "
      f"({used.sum() / max(last, 1):.4f} of the keys scanned); windows {len(used)}")
