"""The byte-level drop-in: compress(data, config) -> VLZ1 bytes and
decompress(blob) -> array, on the GPU, against containers and arrays produced
by the reference (tests/golden/corpus.npz), plus the reference's own
end-to-end properties (test_reconstruct.py:57-118, acceptance criteria 1, 3,
4, 10)."""

from __future__ import annotations

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("needs a CUDA device", allow_module_level=True)

import paper_2201_04614_b200 as vlzg  # noqa: E402
from paper_2201_04614_b200 import model as M  # noqa: E402
from paper_2201_04614_b200.errors import SectionOffsetError  # noqa: E402


@pytest.fixture(autouse=True)
def _allow_256():
    M.allow_block_256(True)
    yield
    M.allow_block_256(False)


def _cfg(eb, b, pol, radius, lanes=8, threads=1):
    return M.CompressionConfig(M.ErrorBound.absolute(eb), block_edge=b, lane_width=lanes,
                               padding=M.PaddingPolicy.parse(pol), radius=radius,
                               thread_count=threads)


def test_compress_bytes_match_reference(corpus_cases):
    n = 0
    for c in corpus_cases:
        if "blob" not in c:
            continue
        cfg = _cfg(c["eb"], c["block_edge"], c["padding"], c["radius"])
        blob, stream = vlzg.compress_detailed(c["data"], cfg)
        assert blob == c["blob"].tobytes(), c["tag"]
        assert stream.codes.tobytes() == c["codes"].astype(np.uint32).tobytes()
        back, desc = vlzg.decompress(blob)
        assert desc.dims == tuple(c["shape"])
        assert back.tobytes() == c["decompressed"].tobytes(), c["tag"]
        n += 1
    assert n > 50


@pytest.mark.parametrize("shape", [(77,), (13, 21), (5, 9, 17), (40, 64, 64)])
def test_round_trip_bound_and_idempotence(shape):
    rng = np.random.default_rng(sum(shape))
    data = rng.uniform(-800, 800, shape).astype(np.float32)
    for eb in (1e-2, 1e-4):
        cfg = _cfg(eb, 8, "mean:global", 32768)
        blob = vlzg.compress(data, cfg)
        back, desc = vlzg.decompress(blob)
        assert np.max(np.abs(back.astype(np.float64) - data.astype(np.float64))) <= eb
        assert vlzg.compress(back, cfg) == blob


def test_thread_count_and_lane_width_do_not_change_bytes():
    rng = np.random.default_rng(8)
    data = rng.uniform(-100, 100, (40, 30)).astype(np.float32)
    blobs = {vlzg.compress(data, _cfg(1e-3, 8, "mean:block", 512, lanes=l, threads=t))
             for l in (1, 4, 8, 16) for t in (1, 4)}
    # lane width is written into the header; for a fixed lane width the
    # thread count never changes the bytes
    assert len(blobs) == 4


def test_relative_bound_and_truncation():
    rng = np.random.default_rng(21)
    data = rng.uniform(0, 100, (31, 17)).astype(np.float32)
    cfg = M.CompressionConfig(M.ErrorBound.relative(1e-3), block_edge=8, lane_width=8)
    blob = vlzg.compress(data, cfg)
    back, _ = vlzg.decompress(blob)
    resolved = 1e-3 * (float(data.max()) - float(data.min()))
    assert np.max(np.abs(back.astype(np.float64) - data.astype(np.float64))) <= resolved
    with pytest.raises(SectionOffsetError):
        vlzg.decompress(blob[: len(blob) // 2])


@pytest.mark.parametrize("dims", [(64,), (24, 16), (8, 8, 16)])
@pytest.mark.parametrize("block", [8, 16, 32, 64])
def test_constant_field_outlier_counts(dims, block):
    data = np.full(dims, 100.0, dtype=np.float32)
    _, zs = vlzg.compress_detailed(data, _cfg(1e-4, block, "zero", 32768))
    _, ms = vlzg.compress_detailed(data, _cfg(1e-4, block, "mean:global", 32768))
    grid = M.build_block_grid(M.ArrayDescriptor(len(dims), dims), block)
    assert int(zs.outlier_counts.sum()) == grid.block_count
    assert int(ms.outlier_counts.sum()) == 0


def test_device_crc32_equals_zlib():
    # csrc/k_crc.cu: any length and start alignment, segment boundaries (4 KiB
    # frames) on both sides, the payload CRC of reference containers
    import zlib

    from paper_2201_04614_b200.gpu import crc32_device

    rng = np.random.default_rng(4)
    raw = rng.integers(0, 256, (9 << 20) + 333, dtype=np.uint8)
    dev = torch.from_numpy(raw).cuda()
    for off in (0, 1, 3, 7, 8, 15):
        for n in (0, 1, 2, 15, 16, 17, 4079, 4080, 4095, 4096, 4097, 8192 + 5, 65536 * 3 + 11,
                  (9 << 20) - off):
            got = crc32_device(dev[off:off + n], n)
            assert got == zlib.crc32(raw[off:off + n].tobytes()), (off, n)


def test_container_payload_crc_on_device_detects_flips(corpus_cases):
    # decompress(blob) checks the payload CRC on the device: every flipped
    # payload byte must be rejected with the reference's PayloadCrcError
    from paper_2201_04614_b200.container import deserialize
    from paper_2201_04614_b200.errors import PayloadCrcError

    blobs = [c["blob"].tobytes() for c in corpus_cases if "blob" in c][:8]
    rng = np.random.default_rng(9)
    for blob in blobs:
        p = deserialize(blob, device=torch.device("cuda", 0))
        assert p.device_payload is not None
        for _ in range(4):
            b = bytearray(blob)
            pos = int(rng.integers(112, len(b) - 4))
            b[pos] ^= 1 << int(rng.integers(0, 8))
            with pytest.raises(PayloadCrcError):
                vlzg.decompress(bytes(b))
