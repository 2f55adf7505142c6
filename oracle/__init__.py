"""TEST INFRASTRUCTURE — CPU oracles for the flow+blend path.

Only tests/, __graft_entry__.smoke() and bench.py's CPU legs may import this
package.  It is the checker, never the thing measured or shipped.
"""
from .binding import Oracle, ref_available, restatement, reference  # noqa: F401
