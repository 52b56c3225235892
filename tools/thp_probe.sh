# Transparent-huge-page / hugetlb probe of the GPU box (backs the host-tier allocation choice in engine.cu alloc_host_tier).
mkdir -p gpurun_out
{ cat /sys/kernel/mm/transparent_hugepage/enabled; cat /sys/kernel/mm/transparent_hugepage/defrag; 
python - <<'PY'
import mmap, ctypes, os, time
libc = ctypes.CDLL("libc.so.6")
n = 1 << 30
m = mmap.mmap(-1, n, flags=mmap.MAP_PRIVATE | mmap.MAP_ANONYMOUS)
addr = ctypes.addressof(ctypes.c_char.from_buffer(m))
print("madvise", libc.madvise(ctypes.c_void_p(addr), ctypes.c_size_t(n), 14))
m.write(b"\0" * n)
for l in open("/proc/meminfo"):
    if "AnonHuge" in l: print(l.strip())
for l in open("/proc/self/smaps_rollup"):
    if "AnonHuge" in l: print("self", l.strip())
PY
} > gpurun_out/thp.txt 2>&1
