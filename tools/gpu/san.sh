timeout 300 compute-sanitizer --tool memcheck python tools/gpu/lz1.py 8 > gpurun_out/san_mem.log 2>&1; echo mem=$?
timeout 300 compute-sanitizer --tool racecheck --racecheck-report hazard python tools/gpu/lz1.py 8 > gpurun_out/san_race.log 2>&1; echo race=$?
timeout 300 compute-sanitizer --tool synccheck python tools/gpu/lz1.py 8 > gpurun_out/san_sync.log 2>&1; echo sync=$?
tail -5 gpurun_out/san_mem.log; grep -m5 -A5 "Error\|Hazard" gpurun_out/san_race.log | head -40; tail -5 gpurun_out/san_race.log; tail -5 gpurun_out/san_sync.log
