"""Build step (TEST INFRASTRUCTURE): writes the Eigen-free first part of the
reference's verify.cpp -- the SAO filter and its Bowyer-Watson Delaunay,
verify.cpp:1-341 -- to oracle/_ref/verify_sao.cpp so the unmodified code can
be compiled here (the RANSAC part below it needs Eigen, which is absent).
usage: python3 cut_sao.py SRC/verify.cpp OUT.cpp"""
import re
import sys

src, out = sys.argv[1], sys.argv[2]
text = open(src).read()
head = text.split("// --- fundamental-matrix estimation", 1)[0]
head = "\n".join(ln for ln in head.splitlines() if "Eigen/Dense" not in ln).rstrip()
head = re.sub(r"namespace \{\s*$", "", head).rstrip()  # the RANSAC helpers' anonymous namespace
open(out, "w").write(head + "\n\n}  // namespace bandmatch\n")
