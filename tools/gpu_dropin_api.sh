# the reference C++ API (fmoe::forward / backward through libfmoe_dropin.so, FMOE_F64) at cfg1:
# default glibc malloc vs large freed blocks kept in the heap (no page faults on the next step's matrices)
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
B=paper_2103_13262_b200/fmoe_bench
A="bench-local --api reference --n-b 8192 --d-m 1024 --d-h 4096 --k 2 --n-e 16 --reps 3 --warmup 1"
timeout 600 $B $A > gpurun_out/refapi_default.csv 2>&1
MALLOC_MMAP_THRESHOLD_=17179869184 MALLOC_TRIM_THRESHOLD_=68719476736 timeout 600 $B $A > gpurun_out/refapi_heap.csv 2>&1
MALLOC_MMAP_THRESHOLD_=17179869184 MALLOC_TRIM_THRESHOLD_=68719476736 MALLOC_TOP_PAD_=4294967296 timeout 600 $B $A > gpurun_out/refapi_heap_pad.csv 2>&1
