"""Full-size config-2 parity fixture from the pinned CPU oracle.

    python tests/golden/make_oracle_c2.py

Runs the oracle port (tests/test_oracle_golden.py pins it to the reference)
on BASELINE config 2 at 64^3 -- static prototype A, IC(0)/ILU(0), GMRES(50)
to 1e-8 -- and stores the iteration count, the residual history, the true
relative residual and every 97th entry of the solution with its norm, so the
GPU parity test can gate the full-size workload without the two CPU minutes.
"""

import pathlib
import sys

import numpy as np

HERE = pathlib.Path(__file__).resolve().parent
sys.path.insert(0, str(HERE.parent.parent))

from oracle import edfa_oracle as O                     # noqa: E402
from paper_2009_13916_b200 import configs                # noqa: E402


def main():
    s = configs.config2(n=64).system
    A, b = s.full_matrix(), s.rhs()
    o1 = O.build_stage1(s.A_ff, s.A_fc, s.A_cf, sets=O.static_sets(s.grid, s.face_index, "A"), no_fill=True)
    o2 = O.build_stage2(s.A_cc, o1, no_fill=True)
    x, r = O.gmres(lambda v: A @ v, lambda v: O.apply(o1, o2, s.A_fc, s.A_cf, v), b, tol=1e-8, restart=50)
    np.savez_compressed(HERE / "oracle_config2_n64.npz", n_it=r.n_it, hist=np.array(r.relres_history),
                        final_relres=r.final_relres, x_sub=x[::97], x_norm=np.linalg.norm(x),
                        nnz_H=o1.H.nnz, nnz_S=o2.S.nnz)
    print(r.n_it, r.final_relres)


if __name__ == "__main__":
    main()
