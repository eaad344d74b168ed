# quick GPU check: division probe, bitwise parity across G, timings
./tools/probe/divtest
timeout 120 python tools/gpu/lz.py 2>&1 | grep -v "Exception\|Trace\|close\|TypeError" | awk '{print $1,$2,$3,$4,$NF}' | sort | uniq -c | head -20
timeout 300 python tools/gpu/diag.py --reps 3 --groups ${PSP_G:-2,4,8}
