"""Mismatch pattern of one forward vs the oracle (development aid).
usage: python tools/probe_parity.py M N K P mode(fast|exact) [token_tile] [ksplit]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "oracle"))
import numpy as np
import torch

import oracle_py as O
import paper_2412_14590_b200 as mq
from paper_2412_14590_b200 import capi

M, N, K = (int(x) for x in sys.argv[1:4])
P = float(sys.argv[4])
mode = capi.MQ_EXACT if sys.argv[5] == "exact" else capi.MQ_FAST
tt = int(sys.argv[6]) if len(sys.argv) > 6 else 0
ks = int(sys.argv[7]) if len(sys.argv) > 7 else 0
W, A, prom = mq.bench_inputs(M, N, K, P, 9)
L = mq.partition_and_quantize(W, prom)
dl = mq.DeviceLayer(L)
Y = dl.forward(torch.from_numpy(A).cuda(), opts=mq.exec_opts(mode, 128, token_tile=tt, ksplit=ks)).cpu().numpy()
sub8 = O.QTensor(8, True, 128, L.sub8.rows, L.sub8.cols, L.sub8.payload, L.sub8.scales, None)
sub4 = O.QTensor(4, False, 128, L.sub4.rows, L.sub4.cols, L.sub4.payload, L.sub4.scales, L.sub4.zero_points)
ref, _, _ = O.mixed_linear(O.Layer(N, K, 128, L.index_map8, L.index_map4, sub8, sub4), A)
err = np.abs(Y - ref) > 1e-3 * np.abs(ref).max()
rel = float(np.abs(Y - ref).max() / np.abs(ref).max())
bad_m = np.where(err.any(axis=1))[0]
bad_n = np.where(err.any(axis=0))[0]
inv = np.empty(N, np.int64)
inv[L.index_map8] = np.arange(L.sub8.rows)
inv[L.index_map4] = L.sub8.rows + np.arange(L.sub4.rows)  # engine row order: sub8 then sub4
rows = np.sort(inv[bad_n])
print(f"M={M} N={N} K={K} P={P} mode={sys.argv[5]} tt={tt} ks={ks}: rel={rel:.3g} bad={int(err.sum())} "
      f"tokens={bad_m[:20].tolist()}{'...' if len(bad_m) > 20 else ''} n_bad_tok={len(bad_m)} "
      f"engine_rows={rows[:12].tolist()}.. n_bad_rows={len(rows)}")
