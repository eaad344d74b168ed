# quick GPU check: division probe, bitwise parity across G, timings
./tools/probe/divtest
timeout 120 python tools/gpu/lz.py 2>&1 | grep -v "Exception\|Trace\|close\|TypeError" | awk '{print $5, $6}' | sort | uniq -c
timeout 300 python tools/gpu/kscale.py 1 | awk '{print $NF}' | sort | uniq -c
timeout 300 python tools/gpu/diag.py --reps 3 --groups ${PSP_G:-2,4,8}
