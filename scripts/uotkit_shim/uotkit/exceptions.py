from paper_2201_00730_b200.exceptions import *  # noqa
