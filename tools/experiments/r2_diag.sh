for d in 0 7; do
  echo "== PALU_VQ_DIAG=$d"
  PALU_LIB_PATH=abtmp/diag/libpalu_b200.so PALU_VQ_DIAG=$d timeout 120 python tools/vq_trace.py --ctas 0 2>&1 | sed 's/np.float64(\([-0-9.]*\))/\1/g' | grep -E "palu_value|CTA 0|conv stage|MMA stage|conv start|conv done" | cut -c1-250
done
