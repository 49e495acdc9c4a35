for cfg in "1 0" "2 0" "2 1" "3 0" "1 1"; do set -- $cfg; echo "super=$1 ahead=$2"; RS_MERGE_SUPER=$1 RS_MERGE_AHEAD=$2 bash tools/ab.sh "2" main 2>&1 | head -1; done
