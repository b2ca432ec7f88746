"""Host-side (no GPU) unit test of the device cache state machines: the LRU
and LFU code in csrc/cache_sim.cu is compiled __host__ __device__ and run on
the CPU against the C oracle (tests/native/lru_host_test.cu)."""
import os
import subprocess

import pytest

HERE = os.path.join(os.path.dirname(os.path.abspath(__file__)), "native")


@pytest.mark.timeout(600)
def test_cache_state_machines_on_host():
    subprocess.run(["make", "-s", "-C", HERE, "lru_host_test"], check=True)
    res = subprocess.run([os.path.join(HERE, "lru_host_test")], capture_output=True, text=True,
                         timeout=300)
    assert res.returncode == 0, res.stdout[-3000:]
    assert "ok (0 failures)" in res.stdout
