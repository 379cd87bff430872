"""Wire codec and the frame-level oracle peer against the reference's own
bytes (tests/golden/wire.json / wire.npz, recorded by make_wire_golden.py). CPU only."""

from __future__ import annotations

import numpy as np
import pytest

from oracle import simplehash as osh
from oracle import wire_peer
from paper_2505_14065_b200 import wire
from tests.golden.gen import WIRE_CASES
from tests.wire_util import case_inputs, load_wire, replay, stale_prefix

META, NPZ = load_wire()
OPS = {"sum": 1, "avg": 2, "max": 3, "min": 4}


def test_codec_matches_reference_bytes():
    g = META["codec"]
    hdr = wire.ChunkHeader(tag=8, seq_nr=2, chunk_index=5, byte_offset=4096, byte_len=12)
    qm = wire.QuantMeta(8, 2, 1, -1.5, 0.25)
    assert hdr.pack().hex() == g["chunk_header"]
    assert qm.pack().hex() == g["quant_meta"]
    assert wire.encode_frame(wire.CHUNK_DATA, hdr.pack() + b"abcdefghijkl").hex() == g["frame_chunk"]
    assert wire.encode_frame(wire.QUANT_META, qm.pack()).hex() == g["frame_meta"]
    assert wire.encode_frame(wire.CHUNK_DATA).hex() == g["frame_empty"]
    assert (wire.CHUNK_DATA, wire.QUANT_META) == (g["chunk_data"], g["quant_meta_type"])
    assert wire.ChunkHeader.unpack_from(bytes.fromhex(g["chunk_header"])) == hdr
    assert wire.QuantMeta.unpack(bytes.fromhex(g["quant_meta"])) == qm


def test_vote_codecs_match_reference_bytes():
    g = META["codec"]
    v = wire.CollectiveInitVote(8, 1 << 20, 1, 2, True)
    assert v.pack().hex() == g["init_vote"] and wire.CollectiveInitVote.unpack(v.pack()) == v
    v = wire.CollectiveInitVote(2**63 + 5, 3, 2, 4, False)
    assert v.pack().hex() == g["init_vote_f64"] and wire.CollectiveInitVote.unpack(v.pack()) == v
    c = wire.CollectiveCompleteVote(8, 2, True, 100, 101)
    assert c.pack().hex() == g["complete_vote"] and wire.CollectiveCompleteVote.unpack(c.pack()) == c
    c = wire.CollectiveCompleteVote(9, 7, False)
    assert c.pack().hex() == g["complete_vote_fail"] and wire.CollectiveCompleteVote.unpack(c.pack()) == c
    assert (wire.COLLECTIVE_INIT_VOTE, wire.COLLECTIVE_COMPLETE_VOTE) == (g["init_vote_type"], g["complete_vote_type"])
    with pytest.raises(wire.ProtocolError):
        wire.CollectiveCompleteVote.unpack(b"\0" * 3)


def _frames(stream: bytes):
    off = 0
    while off < len(stream):
        length, typ = wire._FRAME.unpack_from(stream, off)
        yield typ, stream[off + 5 : off + 4 + length]
        off += 4 + length
    assert off == len(stream)


@pytest.mark.parametrize("i", range(len(WIRE_CASES)))
def test_transcripts_parse(i):
    """Every recorded stream is a sequence of well-formed frames of the
    attempt; payload counters equal the frame bytes (collective.py:296-313)."""
    c = META["cases"][i]
    for r in range(c["w"]):
        stream = NPZ[f"c{i}_tx{r}"].tobytes()
        total = 0
        for typ, body in _frames(stream):
            total += 5 + len(body)
            if typ == wire.CHUNK_DATA:
                h = wire.ChunkHeader.unpack_from(body)
                assert (h.tag, h.seq_nr) == (c["tag"], c["seq_nr"])
                assert h.byte_len == len(body) - wire.CHUNK_HEADER_LEN <= c["chunk_bytes"]
            else:
                assert typ == wire.QUANT_META and c["quantize"]
                assert wire.QuantMeta.unpack(body).seq_nr == c["seq_nr"]
        assert total == c["counters"][r][0]
        assert c["counters"][(r + 1) % c["w"]][1] == total


@pytest.mark.parametrize("i", range(len(WIRE_CASES)))
def test_oracle_peer_reproduces_reference_transcripts(i):
    c = META["cases"][i]
    bufs = case_inputs(c)
    w = c["w"]
    for r in range(w):
        buf = bufs[r].copy()
        rx = NPZ[f"c{i}_tx{(r - 1) % w}"].tobytes()
        counters = []

        def run(tx, rxs):
            counters.append(wire_peer.run_rank(tx, rxs, buf, OPS[c["op"]], c["quantize"], r, w,
                                               c["chunk_bytes"], c["tag"], c["seq_nr"]))

        prefix = stale_prefix(c["tag"], c["seq_nr"]) if r == 0 and w > 1 else b""
        out = replay(run, rx, prefix)
        assert out == NPZ[f"c{i}_tx{r}"].tobytes(), (i, r)
        assert list(counters[0]) == c["counters"][r]
        assert osh.simplehash_np(buf) == c["output_hash"]
