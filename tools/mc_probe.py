"""Multicast (NVLS) capability probe on the GPU box (dev tool)."""
import ctypes

cu = ctypes.CDLL("libcuda.so.1")
cu.cuInit(0)
dev = ctypes.c_int()
cu.cuDeviceGet(ctypes.byref(dev), 0)
for name, attr in (("MULTICAST_SUPPORTED", 132), ("HANDLE_TYPE_FABRIC_SUPPORTED", 128),
                   ("IPC_EVENT_SUPPORTED", 125), ("VIRTUAL_MEMORY_MANAGEMENT_SUPPORTED", 102)):
    v = ctypes.c_int(-1)
    rc = cu.cuDeviceGetAttribute(ctypes.byref(v), attr, dev)
    print(name, attr, "rc", rc, "value", v.value)
import subprocess
print(subprocess.run(["nvidia-smi", "topo", "-m"], capture_output=True, text=True).stdout)
print(subprocess.run(["nvidia-smi", "-q", "-d", "FABRIC"], capture_output=True, text=True).stdout[-1500:])
