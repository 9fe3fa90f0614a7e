"""Write the column streams the bench's SpMM gathers (Reddit-shaped R-MAT, m = 1: every arc of the CSR, in CSR
order) and run build/gather_ceiling on them: the ceiling of exactly this access pattern without the SpMM's arithmetic,
segments or fixup.  Widths: 256 bf16 (512 B rows; the transform-first layer-1 Y rows sit at a 1024 B stride) and 48 bf16
(96 B rows, the last layer).  Run on the GPU box:  python scripts/ceiling_rmat.py > gpurun_out/.../ceiling_rmat.jsonl"""
import os
import subprocess
import sys
import tempfile

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    from paper_2203_10983_b200 import inputs as I
    name = sys.argv[1] if len(sys.argv) > 1 else "reddit"
    sh = I.SHAPES[name]
    indptr, indices = I.rmat(sh.N, sh.nnz)
    exe = os.path.join(ROOT, "build", "gather_ceiling")
    with tempfile.TemporaryDirectory() as d:
        f = os.path.join(d, "col.bin")
        np.ascontiguousarray(indices, np.int32).tofile(f)
        w = (sh.hidden + 7) // 8 * 8 * 2
        c = (sh.C + 7) // 8 * 8 * 2
        for rb, stride, tag in [(w, w, f"{name} R-MAT CSR order, {w} B rows (hidden layers)"),
                                (w, 2 * w, f"{name} R-MAT CSR order, {w} B rows at {2 * w} B stride (TF layer-1 Y)"),
                                (c, 2 * c, f"{name} R-MAT CSR order, {c} B rows at {2 * c} B stride (last layer TF)")]:
            subprocess.run([exe, "10", f, str(rb), str(stride), tag], check=True)


if __name__ == "__main__":
    main()
