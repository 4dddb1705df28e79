for tc in 64 80 96; do for fc in 40 48 56 64; do
  echo -n "trail=$tc fold=$fc "; BRI_TRAIL_CAP=$tc BRI_FOLD_CAP=$fc python tools/step_times.py 2 6 | python -c "import json,sys; d=json.load(sys.stdin); print(sorted(d['ms'])[2])"
done; done
