cd $GRAFT_REPO_ROOT
for st in 2 3 4; do for kb in 8 16 32; do
  for case in "c 13" "z 16" "s 16" "s 10" "d 13" "s 5"; do set -- $case
    TX_TUNE_STAGES=$st TX_TUNE_STAGE_KB=$kb timeout 120 python tools/sweep.py --kinds $1 --sizes $2 --reps 10 2>/dev/null | sed "s/^/{\"S\": $st, \"KB\": $kb, \"r\": /; s/$/}/"
  done
done; done
