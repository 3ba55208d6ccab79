"""Host<->device copy bandwidth from pinned buffers, with the process (and so
the pinned pages' first touch) on each NUMA node in turn: shows whether the
GPU's own node matters on this box.  python tools/h2d_probe.py"""
import glob
import os

import torch


def gpu_numa_node(dev=0):
    p = torch.cuda.get_device_properties(dev)
    bus = f"{p.pci_domain_id:04x}:{p.pci_bus_id:02x}:{p.pci_device_id:02x}.0"
    try:
        return int(open(f"/sys/bus/pci/devices/{bus}/numa_node").read()), bus
    except OSError:
        return -1, bus


def node_cpus(n):
    out = set()
    for part in open(f"/sys/devices/system/node/node{n}/cpulist").read().strip().split(","):
        a, _, b = part.partition("-")
        out.update(range(int(a), int(b or a) + 1))
    return out


node, bus = gpu_numa_node()
nodes = sorted(int(p.split("node")[-1]) for p in glob.glob("/sys/devices/system/node/node[0-9]*"))
print("gpu", bus, "numa node", node, "nodes", nodes, "cpus", os.cpu_count(), "affinity", len(os.sched_getaffinity(0)))
torch.cuda.init()
n = 16 << 20
d = torch.empty(n, dtype=torch.uint8, device="cuda")
full = os.sched_getaffinity(0)
for nd in nodes + [None]:
    cpus = node_cpus(nd) & full if nd is not None else full
    if not cpus:
        continue
    os.sched_setaffinity(0, cpus)
    h = torch.empty(n, dtype=torch.uint8).pin_memory()
    h.fill_(1)
    for _ in range(3):
        d.copy_(h, non_blocking=True)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(20):
        d.copy_(h, non_blocking=True)
    e1.record()
    torch.cuda.synchronize()
    h2d = 20 * n / (e0.elapsed_time(e1) * 1e-3) / 1e9
    e0.record()
    for _ in range(20):
        h.copy_(d, non_blocking=True)
    e1.record()
    torch.cuda.synchronize()
    d2h = 20 * n / (e0.elapsed_time(e1) * 1e-3) / 1e9
    print(f"node {nd}: H2D {h2d:.1f} GB/s  D2H {d2h:.1f} GB/s")
    del h
os.sched_setaffinity(0, full)
