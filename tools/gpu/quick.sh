# quick GPU check: division probe, bitwise parity across G, timings
./tools/probe/divtest
timeout 120 python tools/gpu/lz.py 2>&1 | grep -v "Exception\|Trace\|close\|TypeError" | awk '{print $5, $6}' | sort | uniq -c
timeout 300 python tools/gpu/kscale.py ${PSP_KS:-1:1,2:2} | awk '{print $1, $2, $NF}' | sort | uniq -c
timeout 300 python tools/gpu/diag.py --reps 3 --groups ${PSP_G:-1:1,2:2,2:1}
