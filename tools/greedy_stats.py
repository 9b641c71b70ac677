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
// pipeline model: batches of `batch0` keys growing x2 (keys compacted if free at
// batch start), windows of `win` keys of the compacted list (select: free at window
// start), the scan sees the survivors. Returns picks; out[0] = sorted keys,
// out[1] = selected (input to select) keys, out[2] = scan input keys, out[3] = batches
int64_t model(const int64_t* order, int64_t n, int64_t n_jobs, int64_t k, int64_t batch0, int64_t win, int64_t* out) {
  char* taken = calloc(n_jobs, 1);
  int64_t* lst = malloc(sizeof(int64_t) * n);
  int64_t np = 0, pos = 0, b = batch0;
  out[0] = out[1] = out[2] = out[3] = 0;
  while (pos < n && np < k) {
    int64_t hi = pos + b < n ? pos + b : n, m = 0;
    for (int64_t i = pos; i < hi; i++) { int64_t a, c; unrank2(order[i], &a, &c); if (!taken[a] && !taken[c]) lst[m++] = order[i]; }
    out[0] += m; out[3]++;
    for (int64_t w0 = 0; w0 < m && np < k; w0 += win) {
      int64_t w1 = w0 + win < m ? w0 + win : m;
      int64_t surv = 0;
      if (w0 > 0) out[1] += w1 - w0;
      for (int64_t i = w0; i < w1; i++) { int64_t a, c; unrank2(lst[i], &a, &c); if (w0 == 0 || (!taken[a] && !taken[c])) lst[w0 + surv++] = lst[i]; }
      out[2] += surv;
      for (int64_t i = w0; i < w0 + surv && np < k; i++) { int64_t a, c; unrank2(lst[i], &a, &c); if (!taken[a] && !taken[c]) { taken[a] = taken[c] = 1; np++; } }
    }
    pos = hi; b *= 2;
  }
  free(taken); free(lst);
  return np;
}
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
L.model.restype = I64
L.model.argtypes = [P, I64, I64, I64, I64, I64, P]

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

out = np.zeros(4, np.int64)
for b0 in (1 << 20, 1 << 21, 1 << 23):
    for win in (1 << 16, 1 << 18, 1 << 20):
        L.model(order.ctypes.data, n, F.shape[0], k, b0, win, out.ctypes.data)
        print(f"  model batch0 {b0 >> 20}M win {win >> 10}K: sorted {out[0]/1e6:.2f}M selected {out[1]/1e6:.2f}M "
              f"scanned {out[2]/1e6:.3f}M batches {out[3]} windows~{out[0] // win}")
