for kb in 48 32 24 16; do for cps in 2 3 4; do
 echo "kb=$kb cps=$cps $(CS_SCAN_RR_KB=$kb CS_SCAN_RR_CPS=$cps python tools/gibbs_cfg5.py --time)"
done; done
