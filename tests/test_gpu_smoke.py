"""The driver's round-end entry point: __graft_entry__.smoke() (one tiny update on cuda:0 against the oracle)."""
import pytest

pytestmark = pytest.mark.gpu


def test_graft_entry_smoke():
    import __graft_entry__
    __graft_entry__.smoke()
