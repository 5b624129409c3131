set -x
O=gpurun_out/s3q; mkdir -p $O
timeout 900 compute-sanitizer --tool memcheck python tools/sanitize_smoke.py > $O/memcheck.txt 2>&1; tail -3 $O/memcheck.txt
timeout 900 compute-sanitizer --tool synccheck python tools/sanitize_smoke.py > $O/synccheck.txt 2>&1; tail -3 $O/synccheck.txt
timeout 1200 compute-sanitizer --tool racecheck python tools/sanitize_smoke.py > $O/racecheck.txt 2>&1; grep "Race reported" $O/racecheck.txt | sed 's/0x[0-9a-f]*//g' | sort | uniq -c | sort -rn | head -20; tail -3 $O/racecheck.txt
