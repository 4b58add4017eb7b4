#!/bin/bash
# One-shot hardware probe of the GPU box: host cores/RAM/NUMA, PCIe link of the GPU, IOMMU.
out=gpurun_out/probe.txt
{
echo "== nproc"; nproc
echo "== lscpu"; lscpu | head -30
echo "== free -g"; free -g
echo "== numa"; ls /sys/devices/system/node/ | grep node; cat /sys/devices/system/node/node*/meminfo 2>/dev/null | grep MemTotal
echo "== hugepages"; cat /proc/meminfo | grep -i huge
echo "== thp"; cat /sys/kernel/mm/transparent_hugepage/enabled
echo "== ulimit -l"; ulimit -l
echo "== nvidia-smi"; nvidia-smi
echo "== topo"; nvidia-smi topo -m
echo "== pcie"; nvidia-smi --query-gpu=pci.bus_id,pcie.link.gen.current,pcie.link.gen.max,pcie.link.width.current,pcie.link.width.max --format=csv
bus=$(nvidia-smi --query-gpu=pci.bus_id --format=csv,noheader | head -1 | tr 'A-F' 'a-f' | sed 's/^0000//; s/^00000000/0000/')
echo "bus=$bus"
for d in /sys/bus/pci/devices/*; do
  if [ -f $d/vendor ] && grep -q 0x10de $d/vendor && grep -q 0x030 $d/class; then
     echo "$d speed=$(cat $d/current_link_speed) width=$(cat $d/current_link_width) numa=$(cat $d/numa_node) iommu_group=$(readlink $d/iommu_group)"
  fi
done
echo "== iommu"; ls /sys/class/iommu 2>/dev/null; cat /proc/cmdline
echo "== lspci -tv"; lspci -tv 2>/dev/null | head -80
echo "== cuda-samples?"; ls /usr/local/cuda/extras/demo_suite 2>/dev/null
} > $out 2>&1
python - >> $out 2>&1 <<'PY'
import torch, time
print("torch", torch.__version__, torch.cuda.get_device_name(0))
p = torch.cuda.get_device_properties(0)
print(p)
# pinned H2D / D2H
for sz in (1<<26, 1<<30):
    h = torch.empty(sz, dtype=torch.uint8).pin_memory()
    d = torch.empty(sz, dtype=torch.uint8, device="cuda")
    for _ in range(2): d.copy_(h, non_blocking=True)
    torch.cuda.synchronize()
    s=torch.cuda.Event(enable_timing=True); e=torch.cuda.Event(enable_timing=True)
    s.record(); 
    for _ in range(5): d.copy_(h, non_blocking=True)
    e.record(); torch.cuda.synchronize()
    print(f"H2D pinned {sz>>20} MiB: {5*sz/s.elapsed_time(e)/1e6:.2f} GB/s")
    s.record(); 
    for _ in range(5): h.copy_(d, non_blocking=True)
    e.record(); torch.cuda.synchronize()
    print(f"D2H pinned {sz>>20} MiB: {5*sz/s.elapsed_time(e)/1e6:.2f} GB/s")
t=time.time(); h = torch.empty(8<<30, dtype=torch.uint8).pin_memory(); print("pin 8GiB s", time.time()-t)
PY
