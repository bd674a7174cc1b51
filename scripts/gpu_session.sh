#!/bin/bash
# One gpurun session.  Usage: bash scripts/gpu_session.sh TAG [parts...]
#   parts: tests (full -m gpu suite), bench (short C3 bench line), variants (C2 + C4 sweep)
TAG=${1:-r2}; shift
PARTS=${@:-tests bench}
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
for p in $PARTS; do
  case $p in
    tests)
      timeout 2400 python -m pytest tests -m gpu -q --durations=15 > gpurun_out/${TAG}_gpu_tests.log 2>&1
      echo "tests rc=$?"; tail -25 gpurun_out/${TAG}_gpu_tests.log ;;
    quick)
      timeout 1200 python -m pytest tests -m gpu -q -x --durations=10 --deselect tests/test_gpu_parity_r2.py::test_c4_full_size_bounded_with_drops_bitwise > gpurun_out/${TAG}_gpu_quick.log 2>&1
      echo "quick rc=$?"; tail -25 gpurun_out/${TAG}_gpu_quick.log ;;
    bench)
      timeout 900 python bench.py --steps 5 --warmup 3 --no-cpu > gpurun_out/${TAG}_bench.log 2>&1
      echo "bench rc=$?"; tail -1 gpurun_out/${TAG}_bench.log ;;
    variants)
      C4=1 timeout 2400 bash scripts/variant_sweep.sh gpurun_out/${TAG}_variants.jsonl 3 3
      echo "variants rc=$?"
      python -c "
import json
for l in open('gpurun_out/${TAG}_variants.jsonl'):
    d=json.loads(l); r=d['roofline']; c=d['config']
    print(c['workload'][:70], '%.3e'%d['value'], 'fwd %.1f bwd %.1f frac %.3f drops %d'%(r['fwd_ms'], r['bwd_ms'], r['frac'], c['drops_per_gpu']))
" ;;
  esac
done
for p in $PARTS; do
  case $p in
    partition)
      timeout 900 python -m pytest tests/test_gpu_partition.py -m gpu -q > gpurun_out/${TAG}_partition.log 2>&1
      echo "partition rc=$?"; tail -5 gpurun_out/${TAG}_partition.log ;;
    c5)
      timeout 900 python scripts/c5_partitioned.py --parts 8 --exchange peer --check > gpurun_out/${TAG}_c5_peer.json 2> gpurun_out/${TAG}_c5_peer.err
      echo "c5 peer rc=$?"; tail -1 gpurun_out/${TAG}_c5_peer.json; tail -3 gpurun_out/${TAG}_c5_peer.err
      timeout 900 python scripts/c5_partitioned.py --parts 8 --exchange host > gpurun_out/${TAG}_c5_host.json 2> gpurun_out/${TAG}_c5_host.err
      echo "c5 host rc=$?"; tail -1 gpurun_out/${TAG}_c5_host.json ;;
  esac
done
for p in $PARTS; do
  case $p in
    c5c)
      timeout 900 python scripts/c5_partitioned.py --parts 8 --exchange peer --concurrent --check > gpurun_out/${TAG}_c5_conc.json 2> gpurun_out/${TAG}_c5_conc.err
      echo "c5 concurrent rc=$?"; tail -1 gpurun_out/${TAG}_c5_conc.json; tail -3 gpurun_out/${TAG}_c5_conc.err ;;
  esac
done
for p in $PARTS; do
  case $p in
    bounded)
      timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_parity_r2.py -m gpu -q -x -k "(bounded or fifo or log_grows) and not c4" > gpurun_out/${TAG}_bounded.log 2>&1
      echo "bounded rc=$?"; tail -15 gpurun_out/${TAG}_bounded.log ;;
    bvariants)
      OUT=gpurun_out/${TAG}_bvariants.jsonl; : > $OUT
      for spec in "C2 32 binaryheap 64" "C2 32 sortedarray 64" "C2 32 fiforing 64 32,32" "C4 4 binaryheap 16" "C4 4 sortedarray 32"; do
        set -- $spec
        extra=""; [ -n "$5" ] && extra="--delays $5"
        timeout 600 python bench.py --steps 3 --warmup 3 --no-cpu --no-variants --config $1 --trials $2 --kind $3 --capacity $4 $extra 2>>${OUT%.jsonl}.err | tail -1 >> $OUT
      done
      python -c "
import json
for l in open('$OUT'):
    d=json.loads(l); r=d['roofline']; c=d['config']
    print(c['workload'][:70], '%.3e'%d['value'], 'fwd %.1f bwd %.1f frac %.3f drops %d'%(r['fwd_ms'], r['bwd_ms'], r['frac'], c['drops_per_gpu']))
" ;;
  esac
done
for p in $PARTS; do
  case $p in
    sanitize)
      bash scripts/sanitize.sh gpurun_out/${TAG}_sanitize ;;
    fullbench)
      timeout 1500 python bench.py --steps 10 --warmup 3 > gpurun_out/${TAG}_fullbench.log 2>&1
      echo "fullbench rc=$?"; tail -1 gpurun_out/${TAG}_fullbench.log ;;
  esac
done
for p in $PARTS; do
  case $p in
    abfwd)
      for r in 1 2; do
        bash scripts/ab_args.sh "" head=scratch_lib/head.so new=paper_2512_05906_b200/lib/libeventq_b200.so
      done
      bash scripts/ab_args.sh "--precision 64" head=scratch_lib/head.so new=paper_2512_05906_b200/lib/libeventq_b200.so ;;
  esac
done
for p in $PARTS; do
  case $p in
    tlfwd)
      for lib in scratch_lib/head.so paper_2512_05906_b200/lib/libeventq_b200.so; do
        echo "== $lib"
        EQ_LIB_PATH=$lib timeout 600 python scripts/timeline.py --config C3 --trials 24 --steps 1000 2>&1 | tail -16
      done ;;
  esac
done
for p in $PARTS; do
  case $p in
    ncu)
      timeout 900 /usr/local/cuda/bin/ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
        --log-file gpurun_out/${TAG}_launches.csv python bench.py --steps 2 --warmup 1 --no-cpu --no-variants > gpurun_out/${TAG}_ncu_launch.log 2>&1
      echo "ncu launches rc=$?"
      timeout 1500 /usr/local/cuda/bin/ncu --set full --import-source on --clock-control none -k regex:"k_forward|k_backward" -s 2 -c 2 \
        -o gpurun_out/${TAG}_c3x24 -f python bench.py --steps 2 --warmup 1 --no-cpu --no-variants > gpurun_out/${TAG}_ncu_full.log 2>&1
      echo "ncu full rc=$?"; tail -3 gpurun_out/${TAG}_ncu_full.log ;;
  esac
done
for p in $PARTS; do
  case $p in
    abctr)
      for cfg in "" "--config C4 --trials 4 --kind binaryheap --capacity 16" "--config C2 --trials 32 --kind binaryheap --capacity 64"; do
        bash scripts/ab_args.sh "$cfg" head=scratch_lib/head2.so new=paper_2512_05906_b200/lib/libeventq_b200.so
      done ;;
  esac
done
for p in $PARTS; do
  case $p in
    abb)
      for cfg in "--config C4 --trials 4 --kind binaryheap --capacity 16" "--config C4 --trials 4 --kind sortedarray --capacity 16" "--config C2 --trials 32 --kind binaryheap --capacity 64" "--config C2 --trials 32 --kind fiforing --capacity 64 --delays 32,32"; do
        bash scripts/ab_args.sh "$cfg" head=scratch_lib/head3.so new=paper_2512_05906_b200/lib/libeventq_b200.so
      done ;;
  esac
done
for p in $PARTS; do
  case $p in
    abpf)
      for r in 1 2; do
        bash scripts/ab_args.sh "" nopf=scratch_lib/nopf.so pf2=paper_2512_05906_b200/lib/libeventq_b200.so pf1=scratch_lib/pf1.so
      done ;;
  esac
done
for p in $PARTS; do
  case $p in
    adm)
      timeout 2400 python -m pytest tests/test_gpu_parity.py tests/test_gpu_parity_r2.py -m gpu -x -q -k "bounded or overflow or grows or c4" \
        > gpurun_out/${TAG}_adm_tests.log 2>&1; tail -3 gpurun_out/${TAG}_adm_tests.log ;;
    admprof)
      for cfg in "--config C4 --trials 4 --kind binaryheap --capacity 16" "--config C3 --trials 16 --kind binaryheap --capacity 64"; do
        EQ_TIMELINE=1 timeout 600 python scripts/timeline.py $(echo $cfg | sed 's/--trials 4/--trials 4 --steps 300/;s/--trials 16/--trials 16 --steps 300/') 2>&1 | tee -a gpurun_out/${TAG}_adm_timeline.txt
        EQ_TIMELINE=1 timeout 600 python scripts/timeline.py $(echo $cfg | sed 's/--trials 4/--trials 4 --steps 300/;s/--trials 16/--trials 16 --steps 300/;s/binaryheap --capacity [0-9]*/ring/') 2>&1 | tee -a gpurun_out/${TAG}_adm_timeline.txt
      done
      timeout 1500 /usr/local/cuda/bin/ncu --set full --import-source on --clock-control none -k regex:"k_forward" -s 1 -c 1 \
        -o gpurun_out/${TAG}_c4heap16 -f python bench.py --config C4 --trials 4 --kind binaryheap --capacity 16 --steps 1 --warmup 3 --no-cpu --no-variants > gpurun_out/${TAG}_ncu_c4.log 2>&1
      echo "ncu rc=$?" ;;
    tladm)
      for cfg in "--config C4 --trials 4 --steps 300 --kind binaryheap --capacity 16" "--config C4 --trials 4 --steps 300 --kind sortedarray --capacity 32" \
                 "--config C3 --trials 16 --steps 300 --kind binaryheap --capacity 64" "--config C2 --trials 32 --steps 300 --kind binaryheap --capacity 64" \
                 "--config C2 --trials 32 --steps 300 --kind ring"; do
        echo "== $cfg"; EQ_TIMELINE=1 timeout 600 python scripts/timeline.py $cfg 2>&1 | head -9
      done 2>&1 | tee gpurun_out/${TAG}_tladm.txt ;;
    abskip)
      for cfg in "--config C2 --trials 32 --kind binaryheap --capacity 64" "--config C3 --trials 16 --kind binaryheap --capacity 64" \
                 "--config C4 --trials 4 --kind binaryheap --capacity 16" "--config C4 --trials 4 --kind sortedarray --capacity 32"; do
        bash scripts/ab_args.sh "$cfg" soa=scratch_lib/adm_soa.so skip=paper_2512_05906_b200/lib/libeventq_b200.so
      done 2>&1 | tee gpurun_out/${TAG}_abskip.txt ;;
    abknobs)
      for cfg in "--config C4 --trials 4 --kind binaryheap --capacity 16" "--config C2 --trials 32 --kind binaryheap --capacity 64" \
                 "--config C3 --trials 16 --kind binaryheap --capacity 64" "--config C4 --trials 4 --kind sortedarray --capacity 32"; do
        bash scripts/ab_args.sh "$cfg" bku2=paper_2512_05906_b200/lib/libeventq_b200.so bku1=scratch_lib/bku1.so ev3=scratch_lib/ev3.so \
          sp320=scratch_lib/sp320.so sp352=scratch_lib/sp352.so sp256=scratch_lib/sp256.so
      done 2>&1 | tee gpurun_out/${TAG}_abknobs.txt ;;
    abtail)
      L=paper_2512_05906_b200/lib/libeventq_b200.so
      for r in 1 2; do
        bash scripts/ab_env.sh "" base=scratch_lib/base.so=- t0=$L=EQ_REV_TAIL=0 t64=$L=EQ_REV_TAIL=64 t128=$L=EQ_REV_TAIL=128 \
          t192=$L=EQ_REV_TAIL=192 i128=scratch_lib/inl.so=EQ_REV_TAIL=128 i192=scratch_lib/inl.so=EQ_REV_TAIL=192
      done 2>&1 | tee gpurun_out/${TAG}_abtail.txt ;;
    tmatest)
      EQ_NO_SMEM_STATE=1 timeout 1500 python -m pytest tests -m gpu -q -x --deselect tests/test_gpu_parity_r2.py::test_c4_full_size_bounded_with_drops_bitwise \
        > gpurun_out/${TAG}_tma_tests.log 2>&1; echo "tma tests rc=$?"; tail -2 gpurun_out/${TAG}_tma_tests.log ;;
    abtma)
      L=paper_2512_05906_b200/lib/libeventq_b200.so
      for cfg in "--config C4 --trials 4" "--config C4 --trials 4 --kind binaryheap --capacity 16" "" "--config C2 --trials 32"; do
        bash scripts/ab_env.sh "$cfg" base=scratch_lib/base.so=- tma=$L=- notma=$L=EQ_NO_TMA_STAGE=1
      done 2>&1 | tee gpurun_out/${TAG}_abtma.txt
      bash scripts/ab_env.sh "" base_nosmem=scratch_lib/base.so=EQ_NO_SMEM_STATE=1 tma_nosmem=$L=EQ_NO_SMEM_STATE=1 2>&1 | tee -a gpurun_out/${TAG}_abtma.txt ;;
    ncufwd)
      timeout 1200 /usr/local/cuda/bin/ncu --set full --import-source on --clock-control none -k regex:"k_forward" -s 1 -c 1 \
        -o gpurun_out/${TAG}_fwd -f python bench.py --steps 1 --warmup 3 --no-cpu --no-variants > gpurun_out/${TAG}_ncu_fwd.log 2>&1
      echo "ncu fwd rc=$?" ;;
    abrow)
      L=paper_2512_05906_b200/lib/libeventq_b200.so
      for cfg in "" "--config C4 --trials 4" "--config C2 --trials 32 --kind binaryheap --capacity 64" "--precision 64"; do
        for r in 1 2; do bash scripts/ab_env.sh "$cfg" base=scratch_lib/base.so=- row=$L=-; done
      done 2>&1 | tee gpurun_out/${TAG}_abrow.txt ;;
    abdrop)
      L=paper_2512_05906_b200/lib/libeventq_b200.so
      for cfg in "--config C4 --trials 4 --kind binaryheap --capacity 16" "--config C4 --trials 4 --kind sortedarray --capacity 32" "" ; do
        for r in 1 2; do bash scripts/ab_env.sh "$cfg" base=scratch_lib/base.so=- new=$L=-; done
      done 2>&1 | tee gpurun_out/${TAG}_abdrop.txt ;;
    abwin)
      L=paper_2512_05906_b200/lib/libeventq_b200.so
      for cfg in "--config C4 --trials 4 --kind binaryheap --capacity 16" "--config C4 --trials 4 --kind sortedarray --capacity 32" \
                 "--config C2 --trials 32 --kind binaryheap --capacity 64" "--config C3 --trials 16 --kind binaryheap --capacity 64"; do
        for r in 1 2; do bash scripts/ab_env.sh "$cfg" base=scratch_lib/base.so=- win=$L=-; done
      done 2>&1 | tee gpurun_out/${TAG}_abwin.txt ;;
    pipetest)
      EQ_NO_SMEM_STATE=1 timeout 1500 python -m pytest tests -m gpu -q -x --deselect tests/test_gpu_parity_r2.py::test_c4_full_size_bounded_with_drops_bitwise \
        > gpurun_out/${TAG}_pipe_tests.log 2>&1; echo "pipe tests rc=$?"; tail -2 gpurun_out/${TAG}_pipe_tests.log ;;
    abpipe)
      L=paper_2512_05906_b200/lib/libeventq_b200.so
      for cfg in "--config C4 --trials 4" "--config C4 --trials 4 --kind binaryheap --capacity 16" "" "--config C2 --trials 32"; do
        for r in 1 2; do bash scripts/ab_env.sh "$cfg" base=scratch_lib/base.so=- pipe=$L=-; done
      done 2>&1 | tee gpurun_out/${TAG}_abpipe.txt
      bash scripts/ab_env.sh "" base_nosmem=scratch_lib/base.so=EQ_NO_SMEM_STATE=1 pipe_nosmem=$L=EQ_NO_SMEM_STATE=1 2>&1 | tee -a gpurun_out/${TAG}_abpipe.txt ;;
    abknob2)
      L=paper_2512_05906_b200/lib/libeventq_b200.so
      for r in 1 2; do
        bash scripts/ab_env.sh "" base=$L=- fev2=scratch_lib/fev2.so=- fev4=scratch_lib/fev4.so=- rev3=scratch_lib/rev3.so=- rwin2k=scratch_lib/rwin2k.so=-
      done 2>&1 | tee gpurun_out/${TAG}_abknob2.txt ;;
    abrowst)
      L=paper_2512_05906_b200/lib/libeventq_b200.so
      for r in 1 2; do
        bash scripts/ab_env.sh "" base=$L=- plain=scratch_lib/st1.so=- last=scratch_lib/st2.so=-
      done 2>&1 | tee gpurun_out/${TAG}_abrowst.txt ;;
    absplit)
      L=paper_2512_05906_b200/lib/libeventq_b200.so
      for cfg in "--config C4 --trials 4" "--config C4 --trials 4 --kind binaryheap --capacity 16" ""; do
        bash scripts/ab_env.sh "$cfg" base=$L=- f256=scratch_lib/f256.so=- f224=scratch_lib/f224.so=- f192=scratch_lib/f192.so=-
      done 2>&1 | tee gpurun_out/${TAG}_absplit.txt ;;
    ncuadm)
      timeout 1200 /usr/local/cuda/bin/ncu --set full --import-source on --clock-control none -k regex:"k_forward" -s 1 -c 1 \
        -o gpurun_out/${TAG}_adm -f python bench.py --config C4 --trials 4 --kind binaryheap --capacity 16 --steps 1 --warmup 3 --no-cpu --no-variants > gpurun_out/${TAG}_ncu_adm.log 2>&1
      echo "ncu adm rc=$?" ;;
    abfbits)
      L=paper_2512_05906_b200/lib/libeventq_b200.so
      for cfg in "--config C4 --trials 4 --kind binaryheap --capacity 16" "--config C4 --trials 4 --kind sortedarray --capacity 32" "--config C2 --trials 32 --kind binaryheap --capacity 64"; do
        for r in 1 2; do bash scripts/ab_env.sh "$cfg" base=scratch_lib/base.so=- fbits=$L=-; done
      done 2>&1 | tee gpurun_out/${TAG}_abfbits.txt ;;
    abpfe)
      for cfg in "" "--config C4 --trials 4" "--config C4 --trials 4 --kind binaryheap --capacity 16" "--config C2 --trials 32"; do
        for r in 1 2; do bash scripts/ab_env.sh "$cfg" base=scratch_lib/base.so=- pf=scratch_lib/pf.so=-; done
      done 2>&1 | tee gpurun_out/${TAG}_abpfe.txt ;;
    abev)
      for cfg in "--config C2 --trials 32 --kind binaryheap --capacity 64" "--config C3 --trials 16 --kind binaryheap --capacity 64" \
                 "--config C4 --trials 4 --kind binaryheap --capacity 16" "--config C4 --trials 4 --kind sortedarray --capacity 32"; do
        bash scripts/ab_args.sh "$cfg" ev2=paper_2512_05906_b200/lib/libeventq_b200.so ev4=scratch_lib/adm_ev4.so
      done 2>&1 | tee gpurun_out/${TAG}_abev.txt ;;
    abadm)
      for cfg in "--config C2 --trials 32 --kind binaryheap --capacity 64" "--config C2 --trials 32 --kind sortedarray --capacity 64" \
                 "--config C3 --trials 16 --kind binaryheap --capacity 64" "--config C4 --trials 4 --kind binaryheap --capacity 16" \
                 "--config C4 --trials 4 --kind sortedarray --capacity 32" "--config C2 --trials 32 --kind ring"; do
        for impl in admission hbm; do
          bash scripts/ab_args.sh "$cfg --queue-impl $impl" $impl=paper_2512_05906_b200/lib/libeventq_b200.so
        done
      done 2>&1 | tee gpurun_out/${TAG}_abadm.txt ;;
    abstaged)
      for cfg in "--config C4 --trials 4 --kind binaryheap --capacity 16" "--config C2 --trials 32 --kind binaryheap --capacity 64"; do
        bash scripts/ab_args.sh "$cfg" hbm=paper_2512_05906_b200/lib/libeventq_b200.so
        bash scripts/ab_args.sh "$cfg --queue-impl smem" staged=paper_2512_05906_b200/lib/libeventq_b200.so
      done ;;
  esac
done
