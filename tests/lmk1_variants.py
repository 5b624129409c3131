"""Deterministic corruptions of an LMK1 file (TEST INFRASTRUCTURE).

Shared by tests/golden/make_lmk1.py (which records the REFERENCE's load_model
verdict on each variant, serialize.hpp:185-301) and tests/test_lmk1.py (which
checks the B200 loader gives the same verdict and message).
"""
from __future__ import annotations


def _split(b: bytes):
    hlen = int.from_bytes(b[4:8], "little")
    return b[8:8 + hlen].decode(), b[8 + hlen:]


def _with_header(b: bytes, h: str) -> bytes:
    hb = h.encode()
    return b"LMK1" + len(hb).to_bytes(4, "little") + hb + _split(b)[1]


def _sub(h: str, old: str, new: str) -> str:
    assert old in h, old
    return h.replace(old, new, 1)


def variants(b: bytes) -> dict[str, bytes]:
    h, _ = _split(b)
    hlen = len(h.encode())
    i = h.index('"bytes":') + len('"bytes":')
    j = i
    while h[j].isdigit():
        j += 1
    num = h[i:j]
    bumped = num[:-1] + str((int(num[-1]) + 1) % 10)
    last = h.rindex(',{"bytes"')
    manifest_short = h[:last] + h[h.index("]", h.index("}", last)):]
    return {
        "empty": b"",
        "bad_magic": b"LMK2" + b[4:],
        "trunc_len": b[:6],
        "trunc_header": b[:8 + hlen - 5],
        "bad_json": _with_header(b, h[:-1] + "!"),
        "bad_format": _with_header(b, _sub(h, '"format":"LMK1"', '"format":"LMK0"')),
        "bad_version": _with_header(b, _sub(h, '"version":1', '"version":2')),
        "bad_dtype": _with_header(b, _sub(h, '"dtype":"f64"', '"dtype":"f16"')),
        "unknown_block": _with_header(b, _sub(h, '"type":"lmkan"', '"type":"lmkax"')),
        "bad_mode": _with_header(b, _sub(h, '"mode":"none"', '"mode":"nonx"')),
        "bad_G": _with_header(b, _sub(h, '"G":8', '"G":2')),
        "missing_key": _with_header(b, _sub(h, '"n_in"', '"n_ix"')),
        "manifest_order": _with_header(b, _sub(h, '"name":"block1.P"', '"name":"block1.Q"')),
        "manifest_short": _with_header(b, manifest_short),
        "bytes_mismatch": _with_header(b, h[:i] + bumped + h[j:]),
        "trunc_payload": b[:-3],
        "trailing": b + b"\0",
    }
