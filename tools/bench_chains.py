"""The chain timings of bench.py alone (bench.time_chains: tk_ncon and pairwise, CUDA graphs, L2 flushed):
python tools/bench_chains.py [CFG,CFG,...] -- one JSON line per chain. Peaks: MEASURED_PEAKS.json's HBM
figure and the sustained DMMA probe."""
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402

if __name__ == "__main__":
    if len(sys.argv) > 1:
        bench.CHAIN_CFGS = tuple(int(x) for x in sys.argv[1].split(","))
    dev = torch.device("cuda", 0)
    torch.cuda.set_device(dev)
    stream = torch.cuda.current_stream(dev)
    peak = bench.measure_fp64_peak(stream, dev)
    hbm = float(bench.load_peaks()["hbm_gbs"])
    res = bench.time_chains(dev, stream, peak["dmma_probe_sustained_tflops"] * 1e12, hbm * 1e9)
    for k, v in res.items():
        print(json.dumps({"cfg": k, **v}), flush=True)
