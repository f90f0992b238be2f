# Test-only shim (scripts/reference_suite.sh): routes the reference test-suite's `uotkit`
# imports to paper_2201_00730_b200.  Not part of the product.
#
# The certificate itself is the package's (src/certify.py:31-66, row B7).  The host-side
# norm / scalar-oracle helpers (src/certify.py:69-177) are out of the hot-path scope and
# not in the package; for the suite they come from the REFERENCE's own module, staged
# git-ignored by scripts/reference_suite.sh as _reftests/_ref_certify.py.
from paper_2201_00730_b200.certify import *  # noqa
from paper_2201_00730_b200.certify import WEAK_DUALITY_SLACK  # noqa

try:
    from _ref_certify import (  # noqa: F401
        double_star_norm,
        double_star_norm_grid,
        grid_max_scalar,
        hilbert_norm,
        hilbert_norm_grid,
        scalar_max_oracle,
    )
except ImportError:  # suite not staged
    pass
