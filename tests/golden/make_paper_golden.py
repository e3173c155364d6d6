"""Regenerates tests/golden/paper_convergence.json from the reference's PAPER.md.

The reference implementation cannot be compiled in this environment (Eigen3 /
doctest / CLI11 absent), so its published accuracy numbers are the golden
values: the pgfplots coordinates of the convergence figures (DG curves) and the
rate table.  Run in the build container where /root/reference exists.
"""
import json
import re
import sys

src = sys.argv[1] if len(sys.argv) > 1 else "/root/reference/PAPER.md"
text = open(src).read()
blocks = re.findall(r"coordinates\{([^}]*)\}", text)


def parse(b):
    return [float(y) for _, y in re.findall(r"\(([^,]+),([^)]+)\)", b)]


# figure order in PAPER.md: structured (DG N1..3, LSC N1..3), unstructured (same), arnold (same)
curves = [parse(b) for b in blocks]
out = json.load(open("tests/golden/paper_convergence.json"))
for name, base in (("structured_errors", 0), ("unstructured_errors", 6), ("arnold_errors", 12)):
    out[name] = {str(n + 1): curves[base + n] for n in range(3)}
json.dump(out, open("tests/golden/paper_convergence.json", "w"), indent=2)
print("ok", {k: out[k]["1"][:2] for k in ("structured_errors", "unstructured_errors", "arnold_errors")})
