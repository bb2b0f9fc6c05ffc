"""B200-native phasor-field NLOS reconstruction engine (placeholder during bring-up)."""
