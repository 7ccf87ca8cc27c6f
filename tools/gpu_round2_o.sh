for t in 4 8 12 16; do
  echo "threads=$t $(TSB_COPY_THREADS=$t python bench.py --no-cpu-baseline --no-warm --no-collapsed --steps 6 2>/dev/null | tail -1 | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(round(d["value"]/1e12,3), round(d["e2e"]["value"]/1e12,3), round(d["e2e"]["collapsed_library_default"]/1e12,3))') rw=$(TSB_COPY_THREADS=$t python tools/probe_host_copies.py 2>/dev/null | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(round(d["upload_pageable_ms"],2), round(d["download_fresh_ms"],2), round(d["random_walk_1000_ms"],2))')"
done
