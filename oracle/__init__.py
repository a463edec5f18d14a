"""CPU oracle (test infrastructure; see gft_oracle.py header). Never imported by the product."""
from .gft_oracle import *  # noqa: F401,F403
