"""Multi-tenancy on green-context SM partitions: at MT level
k the SMs are split into k groups, instance i runs on group i with the
persistent kernels' grids sized to it. Tile math does not depend on the grid,
so every instance's logits equal the stream mode's bit for bit; the A/B of
throughput is printed (the bench's config 4 reports both sweeps)."""
import numpy as np
import pytest

from paper_2308_13803_b200 import Config, GpuBackend
from paper_2308_13803_b200 import serving as S

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("model", ["mobilenet_v1", "inception_v3"])
def test_green_partitions_bit_identical_to_streams(model):
    k = 4
    outs = {}
    with GpuBackend(model, Config(abs_max_bs=4, max_mtl=8)) as be:
        for mode in ("streams", "green"):
            be.set_mt_mode(mode)
            assert be.mt_mode() == mode
            be.set_mtl(k)
            be.run_mt_requests(4 * k)
            outs[mode] = [be.last_output(i) for i in range(k)]
            be.set_mtl(1)
    for (a, fa), (b, fb) in zip(outs["streams"], outs["green"]):
        assert fa == fb
        assert np.array_equal(a, b)


def test_green_mt_sweep_and_level_changes():
    with GpuBackend("mobilenet_v1", Config(abs_max_bs=8, max_mtl=10)) as be:
        streams = S.mt_sweep(be, [1, 2, 4, 8, 10], calls_per_instance=10)
        be.set_mt_mode("green")
        green = S.mt_sweep(be, [1, 2, 4, 8, 10], calls_per_instance=10)
        # batching still runs on the whole device in green mode
        lat = be.run_batches(8, 5)
    print("streams", [(c["mtl"], round(c["measured_throughput"])) for c in streams])
    print("green  ", [(c["mtl"], round(c["measured_throughput"])) for c in green])
    assert all(c["measured_throughput"] > 0 for c in green)
    assert green[-1]["measured_throughput"] > 2 * green[0]["measured_throughput"]
    assert np.all(lat > 0)
