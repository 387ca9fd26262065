"""Probe the attention kernel on tiny cases, each in its own subprocess with a short timeout."""
import subprocess
import sys

CASE = r'''
import sys, numpy as np, torch
sys.path.insert(0, ".")
from paper_2505_10951_b200 import host
ctx = host.Context(0)
ctx.set_option("attn_db", int(sys.argv[1]))
rows, pfx, hd, heads = int(sys.argv[2]), int(sys.argv[3]), int(sys.argv[4]), int(sys.argv[5])
d = hd * heads
g = torch.Generator(device="cuda").manual_seed(1)
q = torch.randn(rows, d, device="cuda", generator=g).bfloat16()
kp = torch.randn(max(pfx, 1), d, device="cuda", generator=g).bfloat16()
vp = torch.randn(max(pfx, 1), d, device="cuda", generator=g).bfloat16()
kl = torch.randn(rows, d, device="cuda", generator=g).bfloat16()
vl = torch.randn(rows, d, device="cuda", generator=g).bfloat16()
seg = torch.zeros(rows, dtype=torch.int32, device="cuda")
out = torch.zeros(rows, d, device="cuda", dtype=torch.bfloat16)
work = np.array([[r0, min(256, rows - r0), 0, pfx] for r0 in range(0, rows, 256)], np.int32)
torch.cuda.synchronize()
ctx.attention(q.data_ptr(), kp.data_ptr(), vp.data_ptr(), max(pfx, 1), kl.data_ptr(), vl.data_ptr(), seg.data_ptr(), work, rows, d, heads, out.data_ptr())
torch.cuda.synchronize()
# reference
qf, kk, vv = q.float(), torch.cat([kp[:pfx], kl]).float(), torch.cat([vp[:pfx], vl]).float()
ref = torch.zeros(rows, d, device="cuda")
for h in range(heads):
    s = qf[:, h*hd:(h+1)*hd] @ kk[:, h*hd:(h+1)*hd].t() / hd ** 0.5
    mask = torch.ones(rows, pfx + rows, dtype=torch.bool, device="cuda")
    mask[:, pfx:] = torch.tril(torch.ones(rows, rows, dtype=torch.bool, device="cuda"))
    s = s.masked_fill(~mask, float("-inf"))
    ref[:, h*hd:(h+1)*hd] = torch.softmax(s, -1) @ vv[:, h*hd:(h+1)*hd]
print("ok max err", float((out.float() - ref).abs().max()))
'''

cases = ((64, 0, 128, 1), (128, 0, 128, 1), (200, 0, 128, 1), (256, 64, 128, 1),
         (300, 200, 128, 2), (64, 0, 64, 1), (512, 700, 128, 4))
if len(sys.argv) > 1:
    cases = [tuple(int(v) for v in c.split(",")) for c in sys.argv[1:]]
for db in (1, 0):
    for rows, pfx, hd, heads in cases:
        try:
            r = subprocess.run([sys.executable, "-c", CASE, str(db), str(rows), str(pfx), str(hd), str(heads)],
                               capture_output=True, text=True, timeout=60)
            msg = " | ".join((r.stdout.strip().splitlines() or [""])[-3:] + (r.stderr.strip().splitlines() or [""])[-2:])
        except subprocess.TimeoutExpired:
            msg = "TIMEOUT (hang)"
        print(f"db={db} rows={rows} pfx={pfx} hd={hd} heads={heads}: {msg}", flush=True)
