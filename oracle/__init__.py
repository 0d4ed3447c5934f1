"""ORACLE package — TEST INFRASTRUCTURE ONLY (see oracle/oracle.py header).

Importable only from tests/, __graft_entry__.smoke() and bench.py's CPU
baseline / reference legs.  Shares no code with paper_1610_01265_b200/.
"""
from .oracle import *  # noqa: F401,F403
from . import oracle as core  # noqa: F401
