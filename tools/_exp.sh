timeout 300 python tools/_d2h.py
nvidia-smi -q | grep -iE "Link Gen|Link Width|Max|Current" | head -12
