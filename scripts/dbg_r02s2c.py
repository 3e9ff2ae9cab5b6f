"""Which kernel of the wide pipeline goes wrong on a repeated call?  Checks KMW's
range histograms R and KR's totals in the workspace against host counts."""
import os, sys, json
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np, torch
import oracle, paper_1701_01189_b200 as ms
from paper_1701_01189_b200 import _lib
if os.environ.get('DBG_LIB'): _lib.LIB_PATH = os.environ['DBG_LIB']
from gen import device as gdev, inputs as gen
ms.device_init(0)
h = lambda t: t.cpu().numpy().view(np.uint32)
mode = sys.argv[1]
n = int(sys.argv[2]); m = int(sys.argv[3]); pairs = sys.argv[4] == "1"
sms = torch.cuda.get_device_properties(0).multi_processor_count
T = 4096 if pairs else 8192
LW = (n + T - 1) // T
K = -(-LW // min(sms * 2, 4096))
if pairs and K & 1: K += 1
G = -(-LW // K)
NB = 1 if m <= 32 else 2 if m <= 64 else (4 if m <= 128 else 8)
mP = 32 * NB
k = torch.empty(n, dtype=torch.int32, device="cuda")
gdev.keys_(k, 0x5EED + m, kind=gen.IDENTITY, m=m)
v = torch.empty(n, dtype=torch.int32, device="cuda")
gdev.values_(v, 0x5EED + m, parity=True)
kh, vh = h(k), h(v)
ek, ev, eo = oracle.multisplit(kh, oracle.identity(m), vh if pairs else None)
Rexp = np.zeros((G, mP), np.uint32)
for c in range(G):
    seg = kh[c * K * T:(c + 1) * K * T]
    Rexp[c, :m] = np.bincount(seg, minlength=m)[:m]
Texp = Rexp.sum(0)
ws_keep = torch.empty(ms.workspace_size(n, m, pairs), dtype=torch.uint8, device="cuda")
ko_keep = torch.empty_like(k); vo_keep = torch.empty_like(v)
for rep in range(4):
    if mode == "fresh":
        ko, vo, off = ms.multisplit(k, v if pairs else None, bucket=ms.Identity(m))
        ws = ms.multisplit.last_workspace
    elif mode == "keep":
        ko, vo, off = ms.multisplit(k, v if pairs else None, bucket=ms.Identity(m), out_keys=ko_keep,
                                    out_values=vo_keep if pairs else None, workspace=ws_keep)
        ws = ws_keep
    elif mode == "sync":
        torch.cuda.synchronize()
        ko, vo, off = ms.multisplit(k, v if pairs else None, bucket=ms.Identity(m))
        torch.cuda.synchronize()
        ws = ms.multisplit.last_workspace
    elif mode == "zero":  # fresh but zeroed workspace
        ws = torch.zeros(ms.workspace_size(n, m, pairs), dtype=torch.uint8, device="cuda")
        ko, vo, off = ms.multisplit(k, v if pairs else None, bucket=ms.Identity(m), workspace=ws)
    torch.cuda.synchronize()
    w = ws.view(torch.int32) if ws.numel() % 4 == 0 else ws[: ws.numel() // 4 * 4].view(torch.int32)
    wh = h(w)
    R = wh[(256 + 1280) // 4:(256 + 1280) // 4 + G * mP].reshape(G, mP)
    Tot = wh[256 // 4:256 // 4 + mP]
    res = dict(mode=mode, rep=rep, ws_ptr=ws.data_ptr() % (1 << 40), ko_ptr=ko.data_ptr() % (1 << 40),
               keys_ok=bool(np.array_equal(h(ko), ek)), off_ok=bool(np.array_equal(h(off), eo)),
               R_ok=bool(np.array_equal(R, Rexp)), R_bad_rows=int((R != Rexp).any(1).sum()),
               Tot_ok=bool(np.array_equal(Tot, Texp)))
    if pairs: res["vals_ok"] = bool(np.array_equal(h(vo), ev))
    print(json.dumps(res), flush=True)
    del ko, vo, off, ws, w
