"""Compare two attn_dump.py outputs bitwise."""
import sys
import torch
a, b = torch.load(sys.argv[1]), torch.load(sys.argv[2])
for shp in a:
    for k in a[shp]:
        x, y = a[shp][k], b[shp][k]
        eq = torch.equal(x, y)
        d = (x.float() - y.float()).abs().max().item()
        print(shp, k, "bitwise" if eq else f"DIFF max {d:.3e}")
