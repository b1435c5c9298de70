"""SEM blocks on the reference's framed wire (tag 0x07): round trip, framing
conventions shared with the reference (wire.py header struct), and malformed
frames raising ProtocolError."""
import struct

import numpy as np
import pytest

from paper_2312_09888_b200 import synth
from paper_2312_09888_b200.data_model import POINT, FieldArray, SemBlock
from paper_2312_09888_b200.sem_wire import HEADER, TAG_SEM_BLOCK, ProtocolError, decode_sem_frame, encode_sem_frame


def _block(aos=False):
    c = synth.box(3, 9, nel=(3, 2, 2))
    vel = c.fields["velocity"]
    fields = (FieldArray("velocity", POINT, 3, vel.T.ravel() if aos else vel.ravel(),
                         comp_stride=0 if aos else c.n_points),
              FieldArray("temperature", POINT, 1, c.fields["temperature"].ravel()))
    return c, SemBlock(c.n_elements, c.x, c.y, c.z, fields=fields, element_offset=3, n_elements_global=12)


@pytest.mark.parametrize("aos", [False, True])
def test_round_trip_bit_exact(aos):
    c, b = _block(aos)
    mv = encode_sem_frame(b)
    magic, ver, tag, n = HEADER.unpack_from(mv, 0)
    assert (magic, ver, tag, n) == (b"NKSS", 1, TAG_SEM_BLOCK, len(mv) - HEADER.size)
    r = decode_sem_frame(mv)
    assert (r.n_elements, r.element_offset, r.n_elements_global, r.order) == (6, 3, 12, 7)
    for a, e in ((r.x, c.x), (r.y, c.y), (r.z, c.z)):
        assert np.array_equal(a.view(np.uint64), e.view(np.uint64))
    v = r.fields[0]
    assert v.name == "velocity" and v.components == 3 and v.comp_stride == c.n_points
    assert np.array_equal(np.asarray(v.values).reshape(3, -1), c.fields["velocity"])
    assert np.array_equal(np.asarray(r.fields[1].values), c.fields["temperature"].ravel())


def test_malformed_frames():
    _, b = _block()
    raw = bytes(encode_sem_frame(b))
    with pytest.raises(ProtocolError, match="payload length"):
        decode_sem_frame(raw[:-8])
    bad = bytearray(raw)
    bad[:4] = b"XXXX"
    with pytest.raises(ProtocolError, match="magic"):
        decode_sem_frame(bad)
    other = HEADER.pack(b"NKSS", 1, 0x04, 0)
    with pytest.raises(ProtocolError, match="not a SEM"):
        decode_sem_frame(other)
    short = HEADER.pack(b"NKSS", 1, TAG_SEM_BLOCK, 30) + struct.pack("<qqqB", 0, 1, 1, 7) + b"\0" * 5
    with pytest.raises(ProtocolError, match="truncated"):
        decode_sem_frame(short)


@pytest.mark.gpu
def test_device_arrays_encode_like_host_arrays():
    """A partition living on the GPU (device x, y, z and SoA fields) frames to
    the same bytes as its host copy (D2H straight into the frame)."""
    import torch

    c, hb = _block()
    dev = lambda a: torch.from_numpy(np.ascontiguousarray(a)).cuda()  # noqa: E731
    fields = (FieldArray("velocity", POINT, 3, dev(c.fields["velocity"].ravel()), comp_stride=c.n_points),
              FieldArray("temperature", POINT, 1, dev(c.fields["temperature"].ravel())))
    db = SemBlock(c.n_elements, dev(c.x), dev(c.y), dev(c.z), fields=fields, element_offset=3, n_elements_global=12)
    assert bytes(encode_sem_frame(db)) == bytes(encode_sem_frame(hb))
