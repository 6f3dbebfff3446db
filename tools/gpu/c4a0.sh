timeout 300 python tools/c4_profile.py
C4_ALPHA=0 timeout 300 python tools/c4_profile.py
C4_BATCH=3000 timeout 300 python tools/c4_profile.py
C4_BATCH=3000 C4_ALPHA=0 timeout 300 python tools/c4_profile.py
