"""CPU oracle for the MASQuant hot path — TEST INFRASTRUCTURE ONLY (see masq_oracle.py header)."""
from .masq_oracle import *  # noqa: F401,F403
