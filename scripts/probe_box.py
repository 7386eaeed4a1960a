"""Box facts for the memory plans: GPU memory, host RAM, /dev/shm, cores."""
import json, os, shutil, subprocess
import torch
free, total = torch.cuda.mem_get_info()
mem = {}
for line in open("/proc/meminfo"):
    k, v = line.split(":")
    if k in ("MemTotal", "MemAvailable", "Shmem", "HugePages_Total"):
        mem[k] = v.strip()
shm = shutil.disk_usage("/dev/shm") if os.path.exists("/dev/shm") else None
print(json.dumps({"gpu_total": total, "gpu_free": free, "meminfo": mem, "dev_shm_total": shm.total if shm else None,
                  "nproc": os.cpu_count(), "ulimit_l": subprocess.run("ulimit -l", shell=True, capture_output=True,
                                                                       text=True).stdout.strip()}))
