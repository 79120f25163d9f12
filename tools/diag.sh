for env in "LLSA_VLO=1" "LLSA_VLO=0" "LLSA_VLO=0 LLSA_HILO_LEVEL=1"; do
  echo "######## $env"
  for c in "65536 8 3 3" "65536 8 3 1" "16384 8 2 2"; do env $env python tools/diag_precision.py $c 2>&1 | grep -E "^cfg|LSE err|row-rel max"; done
done
