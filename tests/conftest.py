import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (sm_100a) and the built libwlfuse.so")


@pytest.fixture
def b200():
    from paper_2404_03617_b200.core import DeviceSpec

    return DeviceSpec("b200-datasheet", 2.25e15, 8.0e12, l2_bytes=126 * 2**20)
