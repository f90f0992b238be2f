from paper_2201_00730_b200.fw import *  # noqa
from paper_2201_00730_b200.fw import _h0_value as _h0  # noqa
