"""ORACLE — TEST INFRASTRUCTURE ONLY (see fpbem_oracle.cpp header)."""
from .oracle import *  # noqa: F401,F403
