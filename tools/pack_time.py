import sys, os, time
sys.path.insert(0, os.getcwd())
from paper_1212_2287_b200 import GpuModel, synth
import torch
torch.zeros(1, device="cuda")
for name, fn in [("cfg1", lambda: synth.config1(n=1)), ("cfg3", lambda: synth.config3(n=1)), ("cfg4b", lambda: synth.config4b(n=1))]:
    t0 = time.time(); w = fn(); t1 = time.time()
    m = GpuModel(w.flat, 0); torch.cuda.synchronize(); t2 = time.time()
    print(f"{name}: synth {t1-t0:.2f} s, pack+upload {t2-t1:.2f} s, device_bytes {m.info['device_bytes']/1e6:.1f} MB, segments {m.info['num_segments']}", flush=True)
