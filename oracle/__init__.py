"""CPU oracle (test infrastructure; see gft_oracle.py header). Never imported by the product."""
from .gft_oracle import *  # noqa: F401,F403
from .approx_oracle import (delta_error, epsilon_error, givens_matrix, haar_approx_basis,  # noqa: F401
                            off2, truncated_jacobi)
