for v in "0,0" "1,0" "0,64" "0,256" "1,128"; do
  echo "== MOMG_POLL=$v"; MOMG_POLL=$v timeout 120 python bench.py --no-cpu --no-e2e --no-nmg 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['breakdown_ms'])"
done
