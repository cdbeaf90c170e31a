"""pytest plugin: run the reference's OWN CLI tests (test_cli.py) against
this package's CLI (paper_2001_04179_b200.cli: every solve on the B200,
generators with the device oracle, the native MatrixMarket reader).
Test infrastructure only.

    PYTHONPATH=baseline/_ref:. python -m pytest -p tools.ref_cli_plugin \
        baseline/_ref/kaczmarz_tests/test_cli.py

The reference's test module binds `main` and `derive_seed` from
kaczmarz.cli at import; the plugin rebinds them before collection."""

import kaczmarz.cli as ref_cli

from paper_2001_04179_b200 import cli as dev_cli

ref_cli.main = dev_cli.main
ref_cli.derive_seed = dev_cli.derive_seed
