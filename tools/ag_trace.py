"""Summarise an RV_AG_TRACE event dump of attn_tcg_kernel (CTA 0): per-pair timeline of the
loader (pair start / chunk issue), the MMA issuer (S / P V issue) and the softmax groups."""
import sys
from collections import defaultdict

lines = [l.split() for l in open(sys.argv[1]) if l.startswith("AG ")]
ev = [(int(a, 16), int(b)) for _, a, b in lines]
blocks, cur = [], [ev[0]]
for e in ev[1:]:
    if abs(e[1] - cur[-1][1]) > 2_000_000:
        blocks.append(cur)
        cur = []
    cur.append(e)
blocks.append(cur)
b = sorted(blocks[-1], key=lambda x: x[1])
t0 = b[0][1]
names = {(1, 0): "L pair-wait", (1, 1): "L pair-go", (1, 2): "L chunk-issue", (1, 3): "L chunk-done",
         (2, 0): "I S", (2, 1): "I PV", (3, 0): "X s_full", (3, 1): "X p_arrive", (3, 2): "X o_full", (3, 3): "X epi-done"}
limit = int(sys.argv[2]) if len(sys.argv) > 2 else 200
for code, t in b[:limit]:
    role, e, a, c = code >> 24, (code >> 16) & 255, (code >> 8) & 255, code & 255
    print(f"{(t - t0) / 1000:9.3f} us  {names.get((role, e), '?'):14s} a={a:3d} b={c:3d}")
# aggregates
tot = (b[-1][1] - t0) / 1000
print(f"total {tot:.1f} us, events {len(b)}")
iss = [t for code, t in b if code >> 24 == 1 and (code >> 16) & 255 == 2]
don = [t for code, t in b if code >> 24 == 1 and (code >> 16) & 255 == 3]
if iss:
    d = [(y - x) / 1000 for x, y in zip(iss, don)]
    print(f"loader chunk issue time: mean {sum(d) / len(d):.3f} us over {len(d)} chunks; chunk starts every "
          f"{(iss[-1] - iss[0]) / 1000 / max(1, len(iss) - 1):.3f} us")
