for m in kernel fixup; do echo "DFX_SPLITK=$m"; DFX_SPLITK=$m python scripts/gpu_zoo_timing.py 2>&1 | grep "ms/query"; done
