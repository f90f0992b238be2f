"""``python -m paper_2201_00730_b200 <command>``: the uotkit-compatible CLI."""

from .cli import entry

entry()
