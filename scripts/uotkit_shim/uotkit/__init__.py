# Test-only shim (scripts/reference_suite.sh): routes the reference test-suite's `uotkit`
# imports to paper_2201_00730_b200.  Not part of the product.
# test-only shim: the reference's tests import `uotkit`; route them to the B200 package
from paper_2201_00730_b200 import *  # noqa
from .certify import double_star_norm, hilbert_norm, scalar_max_oracle  # noqa
from . import barycenter, certify, cli, duality, entropies, exceptions, fw, measures, ot1d, sinkhorn  # noqa
