"""Soak test: runs the decode chain (32 Llama-3-8B blocks, d=2, C=256, B=1)
back to back for ~SECS seconds and prints ms/token per window next to
nvidia-smi samples (SM clock, power, temperatures, throttle reasons) --
shows whether a sustained decode is power- or thermal-limited.
usage: python tools/chain_soak.py [secs]"""
import os
import subprocess
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import paper_2605_04084_b200 as F
import synth

NAMES = [("q_proj", "k_proj", "v_proj"), ("o_proj",), ("gate_proj", "up_proj"), ("down_proj",)]
secs = float(sys.argv[1]) if len(sys.argv) > 1 else 6.0
blocks = []
for b in range(32):
    Ls = {}
    for li, (name, fo, fi) in enumerate(synth.LLAMA3_8B_LAYERS):
        cb, idx = synth.torch_random_layer(fo, fi, 2, 256, seed=b * 7 + li)
        Ls[name] = F.import_layer(cb, idx, fi)
    blocks.append(Ls)
steps = []
for b in range(32):
    for i in range(4):
        steps.append(([blocks[b][n] for n in NAMES[i]], None if not steps else (len(steps) - 1, 0)))
ch = F.Chain(steps, B=1)
x = synth.torch_activation(1, 4096)
q = ("timestamp,clocks.sm,clocks.mem,power.draw,temperature.gpu,temperature.memory,"
     "clocks_event_reasons.sw_power_cap,clocks_event_reasons.hw_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
     "clocks_event_reasons.hw_power_brake_slowdown")
smi = subprocess.Popen(["nvidia-smi", "--query-gpu=" + q, "--format=csv,noheader", "-lms", "200"],
                       stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
time.sleep(0.5)
t_end = time.time() + secs
win = 200
while time.time() < t_end:
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(win):
        ch.run(x)
    e1.record()
    torch.cuda.synchronize()
    print("t=%.2fs  %.4f ms/token" % (secs - (t_end - time.time()), e0.elapsed_time(e1) / win), flush=True)
time.sleep(0.3)
smi.terminate()
print(smi.communicate()[0])
