from paper_2201_00730_b200.ot1d import *  # noqa
