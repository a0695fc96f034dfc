"""Probe: where the end-to-end C4 build (host key blob -> serialized
descriptor) spends its time beyond the device build."""
import cProfile
import os
import pstats
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

from paper_2308_09561_b200 import device as dev, recsplit, workloads as W  # noqa: E402

k = W.build_keys(4)
blob = np.frombuffer(np.ascontiguousarray(k, dtype="<u8").tobytes(), dtype=np.uint8)
pin = dev.PinnedBuffer.from_array(blob)
d = dev.DeviceBuffer(blob.nbytes)
for name, src in (("pageable", blob), ("pinned", pin.array)):
    for _ in range(2):
        d.upload(src)
    dev.sync()
    t = time.perf_counter()
    for _ in range(5):
        d.upload(src)
    dev.sync()
    print(f"H2D {name}: {(time.perf_counter() - t) / 5 * 1e3:.2f} ms for {blob.nbytes / 1e6:.0f} MB", flush=True)
for name, src in (("pageable", blob), ("pinned", pin.array)):
    recsplit.build_blob(src, 8, 2000, 40, 1)
    t = time.perf_counter()
    for _ in range(3):
        desc = recsplit.build_blob(src, 8, 2000, 40, 1)
    t1 = time.perf_counter()
    for _ in range(3):
        out = desc.serialize()
    t2 = time.perf_counter()
    print(f"build_blob {name}: {(t1 - t) / 3 * 1e3:.2f} ms, serialize {(t2 - t1) / 3 * 1e3:.2f} ms "
          f"({len(out)} bytes), device phases {desc.device_profile['phase_ms']}", flush=True)
pr = cProfile.Profile()
pr.enable()
desc = recsplit.build_blob(pin.array, 8, 2000, 40, 1)
desc.serialize()
pr.disable()
pstats.Stats(pr).sort_stats("tottime").print_stats(15)
