free -g; nproc; lscpu | grep -E "Model name|Socket|NUMA"; lsblk -o NAME,SIZE,TYPE,MOUNTPOINT,ROTA,MODEL 2>/dev/null | head -30; df -h / /tmp /root 2>/dev/null; mount | grep -E " / | /tmp " ; nvidia-smi topo -m 2>/dev/null | head; 
python - <<'PY'
import torch, time
n = 4<<30
h = torch.empty(n, dtype=torch.uint8, pin_memory=True)
d = torch.empty(n, dtype=torch.uint8, device="cuda")
for it in range(3):
    s=torch.cuda.Event(enable_timing=True); e=torch.cuda.Event(enable_timing=True)
    s.record(); d.copy_(h, non_blocking=True); e.record(); torch.cuda.synchronize()
    t1=s.elapsed_time(e)
    s.record(); h.copy_(d, non_blocking=True); e.record(); torch.cuda.synchronize()
    t2=s.elapsed_time(e)
    print("H2D GB/s", n/t1/1e6, "D2H GB/s", n/t2/1e6)
PY
dd if=/dev/zero of=/tmp/ddtest bs=16M count=256 oflag=direct 2>&1 | tail -1
dd if=/tmp/ddtest of=/dev/null bs=16M iflag=direct 2>&1 | tail -1
rm -f /tmp/ddtest
