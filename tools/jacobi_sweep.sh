for B in 16 8 4; do for I in 1 2; do echo "B=$B I=$I"; NPCG_JACOBI_B=$B NPCG_JACOBI_INNER=$I NPCG_DEBUG=1 python tools/phase_timing.py 2>&1 | grep -E "jacobi|create" | head -4 | tail -2; done; done
