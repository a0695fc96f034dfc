import sys, os
sys.path.insert(0, os.getcwd())
import numpy as np
from paper_2308_09561_b200 import device as dev, recsplit, workloads as W
k = W.build_keys(4)
blob = np.frombuffer(np.ascontiguousarray(k, dtype="<u8").tobytes(), dtype=np.uint8)
d = recsplit.build_blob(blob, 8, 2000, 40, 1)
print(d.build_stats, d.device_profile)
