#!/bin/bash
# One gpurun session.  Usage: bash scripts/gpu_session.sh TAG [parts...]
#   tests      full -m gpu suite                  quick     -m gpu without the C4 full-size tests
#   bench      short C3 bench line                fullbench the default bench line with variants
#   variants   queue-variant sweep (C2/C3/C4)     bounded   bounded-kind parity tests (no C4)
#   adm        bounded / overflow / log-growth / C4 / FIFO parity tests
#   nosmem     the -m gpu suite with the neuron state kept in HBM (EQ_NO_SMEM_STATE=1)
#   partition  partition tests                    c5 / c5c  C5 peer + host-routed / concurrent peer (+ graph)
#   ncu        launch list + ncu --set full of the headline kernels
#   ncuadm     ncu --set full of the admission kernel at C4 heap[16]
#   timeline   phase timelines (EQ_TIMELINE) of C3 x 24 and of the admission kinds at C4 / C3 / C2
#   abadm      admission vs HBM structures on C2 / C3 / C4
# Library A/Bs: scripts/ab_args.sh (bench arguments x libraries) and scripts/ab_env.sh
# (libraries x environment settings) on one box.
TAG=${1:-r2}; shift
PARTS=${@:-tests bench}
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
for p in $PARTS; do
  case $p in
    tests)
      timeout 2400 python -m pytest tests -m gpu -q --durations=15 > gpurun_out/${TAG}_gpu_tests.log 2>&1
      echo "tests rc=$?"; tail -25 gpurun_out/${TAG}_gpu_tests.log ;;
    quick)
      timeout 1200 python -m pytest tests -m gpu -q -x --durations=10 \
        --deselect tests/test_gpu_parity_r2.py::test_c4_full_size_bounded_with_drops_bitwise > gpurun_out/${TAG}_gpu_quick.log 2>&1
      echo "quick rc=$?"; tail -25 gpurun_out/${TAG}_gpu_quick.log ;;
    nosmem)
      EQ_NO_SMEM_STATE=1 timeout 1500 python -m pytest tests -m gpu -q -x \
        --deselect tests/test_gpu_parity_r2.py::test_c4_full_size_bounded_with_drops_bitwise > gpurun_out/${TAG}_nosmem_tests.log 2>&1
      echo "nosmem tests rc=$?"; tail -2 gpurun_out/${TAG}_nosmem_tests.log ;;
    bench)
      timeout 900 python bench.py --steps 5 --warmup 3 --no-cpu > gpurun_out/${TAG}_bench.log 2>&1
      echo "bench rc=$?"; tail -1 gpurun_out/${TAG}_bench.log ;;
    fullbench)
      timeout 1500 python bench.py --steps 10 --warmup 3 > gpurun_out/${TAG}_fullbench.log 2>&1
      echo "fullbench rc=$?"; tail -1 gpurun_out/${TAG}_fullbench.log ;;
    variants)
      C4=1 timeout 2400 bash scripts/variant_sweep.sh gpurun_out/${TAG}_variants.jsonl 3 3
      echo "variants rc=$?"
      python -c "
import json
for l in open('gpurun_out/${TAG}_variants.jsonl'):
    d=json.loads(l); r=d['roofline']; c=d['config']
    print(c['workload'][:70], '%.3e'%d['value'], 'fwd %.1f bwd %.1f frac %.3f drops %d'%(r['fwd_ms'], r['bwd_ms'], r['frac'], c['drops_per_gpu']))
" ;;
    bounded)
      timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_parity_r2.py -m gpu -q -x \
        -k "(bounded or fifo or log_grows) and not c4" > gpurun_out/${TAG}_bounded.log 2>&1
      echo "bounded rc=$?"; tail -15 gpurun_out/${TAG}_bounded.log ;;
    adm)
      timeout 2400 python -m pytest tests/test_gpu_parity.py tests/test_gpu_parity_r2.py -m gpu -x -q \
        -k "bounded or overflow or grows or c4 or admission or fifo" > gpurun_out/${TAG}_adm_tests.log 2>&1
      tail -3 gpurun_out/${TAG}_adm_tests.log ;;
    partition)
      timeout 900 python -m pytest tests/test_gpu_partition.py -m gpu -q > gpurun_out/${TAG}_partition.log 2>&1
      echo "partition rc=$?"; tail -5 gpurun_out/${TAG}_partition.log ;;
    c5)
      timeout 900 python scripts/c5_partitioned.py --parts 8 --exchange peer --check > gpurun_out/${TAG}_c5_peer.json 2> gpurun_out/${TAG}_c5_peer.err
      echo "c5 peer rc=$?"; tail -1 gpurun_out/${TAG}_c5_peer.json; tail -3 gpurun_out/${TAG}_c5_peer.err
      timeout 900 python scripts/c5_partitioned.py --parts 8 --exchange host > gpurun_out/${TAG}_c5_host.json 2> gpurun_out/${TAG}_c5_host.err
      echo "c5 host rc=$?"; tail -1 gpurun_out/${TAG}_c5_host.json ;;
    c5c)
      timeout 900 python scripts/c5_partitioned.py --parts 8 --exchange peer --concurrent --check > gpurun_out/${TAG}_c5_conc.json 2> gpurun_out/${TAG}_c5_conc.err
      echo "c5 concurrent rc=$?"; tail -1 gpurun_out/${TAG}_c5_conc.json; tail -3 gpurun_out/${TAG}_c5_conc.err
      timeout 900 python scripts/c5_partitioned.py --parts 8 --exchange peer --concurrent --graph > gpurun_out/${TAG}_c5_graph.json 2> gpurun_out/${TAG}_c5_graph.err
      echo "c5 graph rc=$?"; tail -1 gpurun_out/${TAG}_c5_graph.json; tail -1 gpurun_out/${TAG}_c5_graph.err ;;
    ncu)
      timeout 900 /usr/local/cuda/bin/ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
        --log-file gpurun_out/${TAG}_launches.csv python bench.py --steps 2 --warmup 1 --no-cpu --no-variants > gpurun_out/${TAG}_ncu_launch.log 2>&1
      echo "ncu launches rc=$?"
      timeout 1500 /usr/local/cuda/bin/ncu --set full --import-source on --clock-control none -k regex:"k_forward|k_backward" -s 2 -c 2 \
        -o gpurun_out/${TAG}_c3x24 -f python bench.py --steps 2 --warmup 1 --no-cpu --no-variants > gpurun_out/${TAG}_ncu_full.log 2>&1
      echo "ncu full rc=$?"; tail -3 gpurun_out/${TAG}_ncu_full.log ;;
    ncuadm)
      timeout 1200 /usr/local/cuda/bin/ncu --set full --import-source on --clock-control none -k regex:"k_forward" -s 1 -c 1 \
        -o gpurun_out/${TAG}_adm -f python bench.py --config C4 --trials 4 --kind binaryheap --capacity 16 --steps 1 --warmup 3 --no-cpu --no-variants > gpurun_out/${TAG}_ncu_adm.log 2>&1
      echo "ncu adm rc=$?" ;;
    timeline)
      for cfg in "--config C3 --trials 24 --steps 1000" \
                 "--config C4 --trials 4 --steps 300 --kind binaryheap --capacity 16" "--config C4 --trials 4 --steps 300 --kind ring" \
                 "--config C3 --trials 16 --steps 300 --kind binaryheap --capacity 64" "--config C2 --trials 32 --steps 300 --kind binaryheap --capacity 64"; do
        echo "== $cfg"; EQ_TIMELINE=1 timeout 600 python scripts/timeline.py $cfg 2>&1 | tail -17
      done 2>&1 | tee gpurun_out/${TAG}_timeline.txt ;;
    abadm)
      for cfg in "--config C2 --trials 32 --kind binaryheap --capacity 64" "--config C2 --trials 32 --kind sortedarray --capacity 64" \
                 "--config C3 --trials 16 --kind binaryheap --capacity 64" "--config C4 --trials 4 --kind binaryheap --capacity 16" \
                 "--config C4 --trials 4 --kind sortedarray --capacity 32" "--config C2 --trials 32 --kind ring"; do
        for impl in admission hbm; do
          bash scripts/ab_args.sh "$cfg --queue-impl $impl" $impl=paper_2512_05906_b200/lib/libeventq_b200.so
        done
      done 2>&1 | tee gpurun_out/${TAG}_abadm.txt ;;
    sanitize)
      bash scripts/sanitize.sh gpurun_out/${TAG}_sanitize ;;
    *)
      echo "unknown part $p" ;;
  esac
done
