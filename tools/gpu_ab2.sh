for V in fused fused_noshell split; do OCTMG_RB=$V python tools/time_vcycle.py 2>&1 | grep -E "rbgs|total|coarse"; done
