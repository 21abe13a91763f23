"""B200-native batched Transducer beam search (ALSD++ / AES++ / greedy)."""
