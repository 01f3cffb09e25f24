"""CPU oracle — TEST INFRASTRUCTURE ONLY (see espo_oracle.py header).

Importable only from tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
--impl reference legs. Never imported by the product package.
"""
from .espo_oracle import *  # noqa: F401,F403
from .espo_oracle import OracleConfig, OracleResult, OracleInputError  # noqa: F401
