"""Float64 CPU oracle (TEST INFRASTRUCTURE ONLY; never imported by the product path).

See oracle/ptycho.py for the header: citations, pins and the parity-unpinned note.
"""
from . import ptycho, partition  # noqa: F401
