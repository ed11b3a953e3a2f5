"""Error type of the file layer.

The reference raises ``SimError`` for bad configuration and broken
invariants (gpuiosim/simcore.py:13) and its CLI maps it to exit status 2
(gpuiosim/cli.py:88-90).  The B200 layer keeps that contract: every
configuration error, native-library failure or parity/invariant violation
surfaces as ``GfsError``; ``SimError`` is the same class under the
reference's name so callers' ``except SimError`` keeps working.
"""


class GfsError(Exception):
    """Fatal file-layer error (bad config, native failure, broken invariant)."""


SimError = GfsError
