"""Run the native host Huffman decoder (csrc/huffman.cpp, built here with
-fsanitize=address) over every golden container that deserializes, including
the crafted over-subscribed codebooks of tests/golden/container_full.json.

    LD_PRELOAD=$(g++ -print-file-name=libasan.so) ASAN_OPTIONS=detect_leaks=0 \
        python tools/asan_huffman.py /tmp/libhuff_asan.so

Exits non-zero (AddressSanitizer report) on any out-of-bounds access.
Used by tests/test_container_full.py::test_host_decoder_asan."""

from __future__ import annotations

import ctypes
import json
import os
import sys

import numpy as np

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, REPO)

from paper_2201_04614_b200.container import deserialize  # noqa: E402


def main(so_path: str) -> int:
    lib = ctypes.CDLL(so_path)
    golden = os.path.join(REPO, "tests", "golden")
    cases = []
    for name in ("container_full.json", "container.json"):
        with open(os.path.join(golden, name)) as fh:
            cases += json.load(fh)
    n = 0
    for c in cases:
        try:
            p = deserialize(bytes.fromhex(c["blob"]))
        except Exception:  # noqa: BLE001 -- rejected before the decoder
            continue
        syms = np.ascontiguousarray(p.codebook.symbols, dtype=np.uint16)
        lens = np.ascontiguousarray(p.codebook.lengths, dtype=np.uint8)
        pay = bytes(p.code_bits)
        # exact-size copies so the sanitizer sees any overrun of the payload
        buf = (ctypes.c_uint8 * max(1, len(pay))).from_buffer_copy(pay or b"\0")
        count = p.descriptor.element_count
        out = (ctypes.c_uint16 * max(1, count))()
        consumed = ctypes.c_int64()
        lib.vlz_huff_decode(buf, ctypes.c_int64(len(pay)), ctypes.c_int64(p.code_bit_length),
                            ctypes.c_void_p(syms.ctypes.data), ctypes.c_void_p(lens.ctypes.data),
                            ctypes.c_int32(len(syms)), ctypes.c_int64(count), out,
                            ctypes.byref(consumed))
        n += 1
    print(f"asan: {n} decodes clean")
    return 0


if __name__ == "__main__":
    sys.exit(main(sys.argv[1]))
