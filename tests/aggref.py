"""Python restatement of the exact aggregate's digit conversion (agg_pieces,
paper_2602_05179_b200/csrc/common.cuh) -- test helper for CPU checks of the
host-side finalization and of the sharded all-reduce."""
import math
import struct

import numpy as np


def pieces(v):
    bits = struct.unpack("<Q", struct.pack("<d", v))[0]
    be = (bits >> 52) & 0x7FF
    M = bits & ((1 << 52) - 1)
    if be == 0:
        E = -1074
    else:
        M |= 1 << 52
        E = be - 1075
    pos = E + 192
    if pos + 53 > 384:
        return None
    if pos < 0:
        M = 0 if -pos >= 64 else M >> (-pos)
        pos = 0
    x = M << (pos & 31)
    return pos >> 5, [x & 0xFFFFFFFF, (x >> 32) & 0xFFFFFFFF, (x >> 64) & 0xFFFFFFFF]


def raw_of(values):
    """scendp_agg_raw of a list of costs."""
    from paper_2602_05179_b200 import _capi as A
    r = A.AggRaw()
    for v in values:
        if not math.isfinite(v):
            r.infeasible_count += 1
            continue
        li, ps = pieces(v)
        for j, p in enumerate(ps):
            if p:
                r.digits[li + j] += p
        r.finite_count += 1
    return r


def raw_words(totals_per_candidate):
    """[k][16] u64 words (the buffer the library all-reduces)."""
    out = []
    for vals in totals_per_candidate:
        r = raw_of(list(vals))
        out.append(list(r.digits) + [r.finite_count, r.infeasible_count, r.error_count,
                                     r.range_errors])
    return np.array(out, dtype=np.uint64)


def to_struct(words):
    from paper_2602_05179_b200 import _capi as A
    k = len(words)
    arr = (A.AggRaw * k)()
    for c, w in enumerate(words):
        for j in range(A.AGG_DIGITS):
            arr[c].digits[j] = int(w[j])
        arr[c].finite_count, arr[c].infeasible_count = int(w[12]), int(w[13])
        arr[c].error_count, arr[c].range_errors = int(w[14]), int(w[15])
    return arr
