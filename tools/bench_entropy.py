"""Entropy stage on the GPU: histogram + device Huffman encode throughput on
the code stream of a BASELINE config, plus the end-to-end compress() /
decompress() container pipeline time.  For DESIGN.md / profiling, not the
driver's bench."""

from __future__ import annotations

import json
import os
import statistics
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import paper_2201_04614_b200 as vlzg  # noqa: E402
from paper_2201_04614_b200 import gpu, workloads  # noqa: E402
from paper_2201_04614_b200 import model as M  # noqa: E402
from paper_2201_04614_b200.huffman import build_codebook_from_freqs  # noqa: E402


def ev_time(fn, reps=7):
    flush = torch.empty(64 * 1024 * 1024, dtype=torch.float32, device="cuda")
    ts = []
    for _ in range(reps):
        flush.zero_()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        fn()
        b.record()
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b))
    return statistics.median(ts)


def case(name, data, rel, b, pol, radius):
    M.allow_block_256(True)
    x = torch.from_numpy(data).cuda()
    eb = workloads.value_range_eb(data, rel)
    cfg = M.CompressionConfig(M.ErrorBound.absolute(eb), block_edge=b, radius=radius,
                              padding=M.PaddingPolicy.parse(pol))
    dev = gpu.compress_device(x, cfg, eb=eb).check()
    n = data.size
    codes = dev.codes[:n]
    freqs = gpu.histogram_device(codes, radius)
    cb = build_codebook_from_freqs(freqs)
    nbits = int((freqs[cb.symbols] * cb.lengths.astype(np.uint64)).sum())
    lib = gpu._lib.load()
    tab = torch.empty(int(lib.vlz_huff_table_bytes()), dtype=torch.uint8, device="cuda")
    syms = np.ascontiguousarray(cb.symbols, dtype=np.uint16)
    lens = np.ascontiguousarray(cb.lengths, dtype=np.uint8)
    assert lib.vlz_huff_table(syms.ctypes.data, lens.ctypes.data, len(syms), tab.data_ptr(),
                              None) == 0
    cap = (nbits + 31) // 32 * 4 + 4
    out = torch.empty(cap, dtype=torch.uint8, device="cuda")
    ws = torch.empty(int(lib.vlz_huff_encode_ws_size(n)), dtype=torch.uint8, device="cuda")
    info = torch.empty(4, dtype=torch.int64, device="cuda")
    fr = torch.empty(65536, dtype=torch.int64, device="cuda")

    def enc():
        lib.vlz_huff_encode_device(codes.data_ptr(), n, tab.data_ptr(), int(syms.max()) + 1,
                                   int(lens.max()),
                                   out.data_ptr(), cap, info.data_ptr(), ws.data_ptr(),
                                   ws.numel(), None)

    def hist():
        lib.vlz_histogram(codes.data_ptr(), n, radius, fr.data_ptr(), None)

    enc()
    torch.cuda.synchronize()
    assert int(info[0].item()) == nbits
    t_enc = ev_time(enc)
    t_hist = ev_time(hist)
    # device decode of the same payload (includes its host-synchronised sync
    # passes: wall time around the call, payload already on the device)
    from paper_2201_04614_b200.huffman import decode_device

    payload = out[: (nbits + 7) // 8].cpu().numpy().tobytes()
    dec = decode_device(payload, nbits, cb, n)
    assert torch.equal(dec, codes), "device decode mismatch"
    dpay = torch.zeros((len(payload) + 3) // 4 * 4 + 16, dtype=torch.uint8, device="cuda")
    dpay[: len(payload)].copy_(torch.frombuffer(bytearray(payload), dtype=torch.uint8))
    dout = torch.empty(n, dtype=torch.int16, device="cuda")
    dws = torch.empty(int(lib.vlz_huff_decode_ws_size(len(payload))), dtype=torch.uint8,
                      device="cuda")
    consumed = gpu.ctypes.c_int64(0)

    def dec_call():
        rc = lib.vlz_huff_decode_device(dpay.data_ptr(), len(payload), nbits, syms.ctypes.data,
                                        lens.ctypes.data, len(syms), n, dout.data_ptr(),
                                        gpu.ctypes.byref(consumed), dws.data_ptr(), dws.numel(),
                                        None)
        assert rc == 0

    dec_call()
    tds = []
    for _ in range(5):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        dec_call()
        torch.cuda.synchronize()
        tds.append((time.perf_counter() - t0) * 1e3)
    t_dec = statistics.median(tds)
    # full container pipeline (host array in, bytes out; and back)
    blob = vlzg.compress(data, cfg)
    t0 = time.perf_counter()
    for _ in range(3):
        blob = vlzg.compress(data, cfg)
    t_c = (time.perf_counter() - t0) / 3
    back, _ = vlzg.decompress(blob)  # warm-up (pinned output block, tables)
    del back
    t0 = time.perf_counter()
    for _ in range(3):
        back, _ = vlzg.decompress(blob)
        del back
    t_d = (time.perf_counter() - t0) / 3
    alg = 2 * n + nbits / 8
    print(json.dumps(dict(
        case=name, n=n, bits_per_symbol=nbits / n, nsym=len(syms), maxlen=int(lens.max()),
        encode_ms=t_enc, encode_gbs_codes=2 * n / t_enc / 1e6,
        encode_algorithmic_tbs=alg / t_enc / 1e9, histogram_ms=t_hist,
        decode_ms=t_dec, decode_gbs_codes=2 * n / t_dec / 1e6,
        compress_pipeline_s=t_c, compress_pipeline_gbs=4 * n / t_c / 1e9,
        decompress_pipeline_s=t_d, decompress_pipeline_gbs=4 * n / t_d / 1e9,
        container_bytes=len(blob), ratio=4 * n / len(blob))), flush=True)


def main():
    which = sys.argv[1:] or ["C3", "C4"]
    if "C2" in which:
        case("C2 mean:block", workloads.gen_c2(), 1e-4, 16, "mean:block", 512)
    if "C3" in which:
        case("C3 mean:global", workloads.gen_c3(), 1e-3, 8, "mean:global", 512)
    if "C4" in which:
        case("C4 b=8 R=512", workloads.gen_c4(512), 1e-3, 8, "mean:global", 512)


if __name__ == "__main__":
    main()
