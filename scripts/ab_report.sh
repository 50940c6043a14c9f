for f in gpurun_out/ab_*.log; do printf "%-45s " $(basename $f); grep -o '"ms_per_step": [0-9.]*\|"popcount": [0-9]*' $f | tr '\n' ' '; echo; done
