"""Experiment: a stream of independent fused convs (cfg4) with the next step's K3 + K0 on a
side stream, overlapping this step's K6 (its ragged tail leaves SMs idle), against the
serial ring graph bench.py times.  NSETS plan objects give each in-flight step its own
workspace and packed weights.

    python tools/overlap_probe.py [cfg4] [nsets]
"""
import ctypes
import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import numpy as np
import torch
from paper_2407_10730_b200 import _capi, algos
from paper_2407_10730_b200.configs import CONFIGS, conv_flops
from paper_2407_10730_b200.harness import RunConfig, make_inputs

name = sys.argv[1] if len(sys.argv) > 1 else "cfg4"
nsets = int(sys.argv[2]) if len(sys.argv) > 2 else 3
R = 12  # steps per graph
d = CONFIGS[name]
inp = make_inputs(d, RunConfig(seed=0))
NB = 4
xs = [torch.from_numpy(np.asarray(inp.input)).cuda() for _ in range(NB)]
ws = [torch.from_numpy(np.asarray(inp.weights)).cuda() for _ in range(NB)]
ys = [torch.empty((d.batch, d.out_channels) + algos.output_shape(d), device="cuda") for _ in range(NB)]
lib = _capi.load()


def time_graph(g, steps):
    for _ in range(3):
        g.replay()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(10):
        g.replay()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) * 1e3 / (10 * steps)


# serial: what bench.py does (one plan object, steps in sequence)
fc = algos.FusedConv(d, "tc3xbf16")
serial = fc.capture_steps([(xs[i % NB], ws[i % NB], ys[i % NB]) for i in range(R)])
t_serial = time_graph(serial, R)
ref = ys[(R - 1) % NB].clone()

# overlapped: packing of step i + 1 on a side stream while K6 of step i runs
fcs = [algos.FusedConv(d, "tc3xbf16") for _ in range(nsets)]
for f in fcs:
    f.run(xs[0], ys[0], weights=ws[0])
torch.cuda.synchronize()


def pack(f, i):
    st = torch.cuda.current_stream().cuda_stream
    f.pack_weights(ws[i % NB])
    _capi.check(lib.cb_fused_pack_input(f.vid, ctypes.byref(f._cd), xs[i % NB].data_ptr(),
                                        f.workspace.data_ptr(), f.ws_bytes, st))


def conv(f, i):
    st = torch.cuda.current_stream().cuda_stream
    ptr = lambda t: None if t is None else t.data_ptr()
    _capi.check(lib.cb_conv_fused_packed(f.vid, ctypes.byref(f._cd), xs[i % NB].data_ptr(),
                                         f.workspace.data_ptr(), f.ws_bytes, ptr(f.w_hi), ptr(f.w_lo),
                                         ptr(f.w_f32), None, ys[i % NB].data_ptr(), st))


side = torch.cuda.Stream()
g = torch.cuda.CUDAGraph()
with torch.cuda.graph(g):
    main = torch.cuda.current_stream()
    packed = [torch.cuda.Event() for _ in range(R)]
    done = [torch.cuda.Event() for _ in range(R)]
    side.wait_stream(main)
    for i in range(R):
        with torch.cuda.stream(side):
            if i >= nsets:
                side.wait_event(done[i - nsets])  # this set's previous K6 has read its operands
            pack(fcs[i % nsets], i)
            packed[i].record(side)
        main.wait_event(packed[i])
        conv(fcs[i % nsets], i)
        done[i].record(main)
    main.wait_stream(side)
t_over = time_graph(g, R)
ok = torch.equal(ys[(R - 1) % NB], ref)
fl = conv_flops(d)
print(f"{name}: serial {t_serial:.1f} us/step ({fl / t_serial / 1e6:.1f} TFLOP/s), overlapped x{nsets} sets "
      f"{t_over:.1f} us/step ({fl / t_over / 1e6:.1f} TFLOP/s), identical output: {ok}")
