"""The reference-side registration of INTEGRATION.md, executed against the
reference itself: examples/nekmini_gpu_sink.py adds a `gpu_render` kind to
nekmini's closed registries (bridge.py:32-39, sinks.py:405-410), nekmini's
own parse_config / initialize / Bridge.update drive it, and a consume that
cannot reach a GPU is isolated into a SinkReport exactly as the reference
isolates any sink failure (bridge.py:164-176).

Needs the reference sources (/root/reference, present in the build
container, absent on the GPU box): skipped elsewhere."""
import importlib
import os
import sys

import numpy as np
import pytest

REF_SRC = "/root/reference/pkg/src"
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

pytestmark = pytest.mark.skipif(not os.path.isdir(os.path.join(REF_SRC, "nekmini")),
                                reason="reference sources not present")


@pytest.fixture
def nekmini(monkeypatch):
    monkeypatch.syspath_prepend(REF_SRC)
    monkeypatch.syspath_prepend(os.path.join(ROOT, "examples"))
    bridge = importlib.import_module("nekmini.bridge")
    sinks = importlib.import_module("nekmini.sinks")
    # the registries are module globals: restore them after the test
    monkeypatch.setattr(bridge, "KINDS", tuple(bridge.KINDS))
    monkeypatch.setattr(bridge, "_KNOWN_ATTRS", {k: set(v) for k, v in bridge._KNOWN_ATTRS.items()})
    monkeypatch.setattr(sinks, "_SINK_TYPES", dict(sinks._SINK_TYPES))
    stub = importlib.import_module("nekmini_gpu_sink")
    yield bridge, sinks, stub
    sys.modules.pop("nekmini_gpu_sink", None)


def _snapshot(dm, step):
    nx, ny = 9, 5
    t = np.linspace(0.0, 1.0, nx * ny)
    vel = np.stack([np.sin(3 * t), np.cos(2 * t), t], axis=1).ravel()
    blk = dm.Block((0.0, 0.0, 0.0), (1.0, 1.0, 1.0), (0, nx - 1, 0, ny - 1, 0, 0),
                   (dm.FieldArray("temperature", dm.POINT, 1, t), dm.FieldArray("velocity", dm.POINT, 3, vel)))
    return dm.Snapshot(0.1 * step, step, 0, (blk,))


def test_registration_parses_constructs_and_isolates(nekmini, tmp_path):
    bridge, sinks, stub = nekmini
    dm = importlib.import_module("nekmini.data_model")
    with pytest.raises(bridge.ConfigError, match="unknown analysis kind"):
        bridge.parse_config('<sensei><analysis type="gpu_render" frequency="1"/></sensei>')
    assert stub.register() == "gpu_render"
    cfg = bridge.parse_config(f'<sensei><analysis type="gpu_render" frequency="2" dir="{tmp_path}" '
                              f'width="32" height="16" field="velocity:mag" bogus="1"/>'
                              f'<analysis type="null" frequency="1"/></sensei>')
    spec = cfg.specs[0]
    assert spec.kind == "gpu_render" and spec.frequency == 2
    assert spec.params == {"dir": str(tmp_path), "width": "32", "height": "16", "field": "velocity:mag"}
    br = bridge.initialize(cfg)
    assert isinstance(br.sinks[0], stub.GpuRenderSink) and br.sinks[0].fields == ["velocity:mag"]
    reps = br.update(_snapshot(dm, 0))
    assert [r.kind for r in reps] == ["gpu_render", "null"]
    gpu = reps[0]
    if gpu.error is None:                      # a GPU is present: the reference's file name and size
        assert gpu.bytes_written == len(b"P6\n32 16\n255\n") + 32 * 16 * 3
        assert (tmp_path / "step000000_velocity_mag.ppm").exists()
    else:                                      # no GPU here: isolated, later sinks still ran
        assert reps[1].error is None
    summ = br.finalize()
    assert summ[0].kind == "gpu_render" and summ[0].invocations == 1


def test_unwritable_directory_fails_at_initialize(nekmini, tmp_path):
    bridge, sinks, stub = nekmini
    stub.register()
    f = tmp_path / "file"
    f.write_text("x")
    cfg = bridge.parse_config(f'<sensei><analysis type="gpu_render" frequency="1" dir="{f}/sub"/></sensei>')
    with pytest.raises(OSError):
        bridge.initialize(cfg)
