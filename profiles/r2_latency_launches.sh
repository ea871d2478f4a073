# per-kernel durations (ncu launch list, serialised) of the latency configs C1 and C3 after run_graph + cluster split-K
mkdir -p gpurun_out
for c in C1 C3; do
  d=1; [ $c = C3 ] && d=9
  ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r2_launches_$c.csv python profiles/one_config.py $c 3 3 $d > /dev/null 2>&1
  python profiles/summarize_launches.py gpurun_out/r2_launches_$c.csv > gpurun_out/r2_launches_$c.txt 2>&1
done
