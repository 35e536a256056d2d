# config 2/4 PageRank ms/iter for libgi variants (default first)
for v in base "$@"; do
  for c in 2 4; do
    echo -n "$v cfg$c  "
    if [ "$v" = base ]; then timeout 600 python tools/prof.py --config $c --pr-iters 20 --pr-reps 2 --bfs 0 2>&1 | tail -1
    else GI_LIBGI=paper_1805_00923_b200/libgi_$v.so timeout 600 python tools/prof.py --config $c --pr-iters 20 --pr-reps 2 --bfs 0 2>&1 | tail -1; fi
  done
done
