#ifndef SELECT_BF16_TN_H
#define SELECT_BF16_TN_H

#include <stdint.h>

typedef struct {
    uint32_t acc;
    uint32_t row_tile;
    uint32_t col_tile;
    uint32_t wg_rows;
    uint32_t wg_cols;
} select_bf16_tn_config;

static inline select_bf16_tn_config select_bf16_tn(int64_t m, int64_t k, int64_t n) {
    (void)m;
    (void)k;
    (void)n;
    if (k < INT64_C(1087)) {
        if (m < INT64_C(17740)) {
            if (n < INT64_C(111)) {
                select_bf16_tn_config out = {4u, 1u, 1u, 8u, 8u};
                return out;
            } else {
                if (m < INT64_C(2218)) {
                    if (n < INT64_C(1620)) {
                        if (m < INT64_C(634)) {
                            select_bf16_tn_config out = {4u, 1u, 1u, 8u, 8u};
                            return out;
                        } else {
                            if (k < INT64_C(702)) {
                                if (n < INT64_C(992)) {
                                    select_bf16_tn_config out = {4u, 1u, 1u, 8u, 8u};
                                    return out;
                                } else {
                                    if (m < INT64_C(1109)) {
                                        select_bf16_tn_config out = {4u, 1u, 1u, 8u, 8u};
                                        return out;
                                    } else {
                                        select_bf16_tn_config out = {1u, 1u, 2u, 8u, 8u};
                                        return out;
                                    }
                                }
                            } else {
                                if (m < INT64_C(1109)) {
                                    if (n < INT64_C(203)) {
                                        select_bf16_tn_config out = {4u, 1u, 1u, 8u, 8u};
                                        return out;
                                    } else {
                                        select_bf16_tn_config out = {1u, 1u, 2u, 8u, 8u};
                                        return out;
                                    }
                                } else {
                                    select_bf16_tn_config out = {8u, 1u, 4u, 8u, 8u};
                                    return out;
                                }
                            }
                        }
                    } else {
                        if (m < INT64_C(278)) {
                            if (k < INT64_C(725)) {
                                select_bf16_tn_config out = {4u, 1u, 1u, 8u, 8u};
                                return out;
                            } else {
                                if (m < INT64_C(139)) {
                                    select_bf16_tn_config out = {1u, 1u, 2u, 8u, 8u};
                                    return out;
                                } else {
                                    select_bf16_tn_config out = {4u, 1u, 1u, 8u, 8u};
                                    return out;
                                }
                            }
                        } else {
                            select_bf16_tn_config out = {1u, 1u, 2u, 8u, 8u};
                            return out;
                        }
                    }
                } else {
                    if (n < INT64_C(222)) {
                        if (m < INT64_C(8870)) {
                            if (k < INT64_C(363)) {
                                select_bf16_tn_config out = {4u, 1u, 1u, 8u, 8u};
                                return out;
                            } else {
                                if (m < INT64_C(4435)) {
                                    select_bf16_tn_config out = {4u, 1u, 1u, 8u, 8u};
                                    return out;
                                } else {
                                    select_bf16_tn_config out = {1u, 1u, 2u, 8u, 8u};
                                    return out;
                                }
                            }
                        } else {
                            select_bf16_tn_config out = {1u, 1u, 2u, 8u, 8u};
                            return out;
                        }
                    } else {
                        select_bf16_tn_config out = {1u, 1u, 2u, 8u, 8u};
                        return out;
                    }
                }
            }
        } else {
            if (n < INT64_C(28)) {
                if (m < INT64_C(70960)) {
                    select_bf16_tn_config out = {4u, 1u, 1u, 8u, 8u};
                    return out;
                } else {
                    select_bf16_tn_config out = {1u, 1u, 2u, 8u, 8u};
                    return out;
                }
            } else {
                if (k < INT64_C(384)) {
                    if (n < INT64_C(46)) {
                        if (m < INT64_C(35480)) {
                            select_bf16_tn_config out = {4u, 1u, 1u, 8u, 8u};
                            return out;
                        } else {
                            select_bf16_tn_config out = {1u, 1u, 2u, 8u, 8u};
                            return out;
                        }
                    } else {
                        select_bf16_tn_config out = {1u, 1u, 2u, 8u, 8u};
                        return out;
                    }
                } else {
                    if (n < INT64_C(91)) {
                        select_bf16_tn_config out = {1u, 1u, 2u, 8u, 8u};
                        return out;
                    } else {
                        select_bf16_tn_config out = {4u, 1u, 8u, 16u, 16u};
                        return out;
                    }
                }
            }
        }
    } else {
        if (n < INT64_C(1432)) {
            if (m < INT64_C(1109)) {
                if (m < INT64_C(12)) {
                    if (k < INT64_C(1620)) {
                        select_bf16_tn_config out = {1u, 1u, 2u, 8u, 8u};
                        return out;
                    } else {
                        if (m < INT64_C(6)) {
                            select_bf16_tn_config out = {8u, 1u, 4u, 8u, 8u};
                            return out;
                        } else {
                            if (k < INT64_C(2897)) {
                                select_bf16_tn_config out = {1u, 1u, 2u, 8u, 8u};
                                return out;
                            } else {
                                select_bf16_tn_config out = {8u, 1u, 4u, 8u, 8u};
                                return out;
                            }
                        }
                    }
                } else {
                    if (m < INT64_C(555)) {
                        if (m < INT64_C(278)) {
                            if (m < INT64_C(28)) {
                                if (k < INT64_C(1620)) {
                                    select_bf16_tn_config out = {4u, 1u, 1u, 8u, 8u};
                                    return out;
                                } else {
                                    select_bf16_tn_config out = {1u, 1u, 2u, 8u, 8u};
                                    return out;
                                }
                            } else {
                                if (m < INT64_C(139)) {
                                    select_bf16_tn_config out = {4u, 1u, 1u, 8u, 8u};
                                    return out;
                                } else {
                                    if (k < INT64_C(3259)) {
                                        select_bf16_tn_config out = {4u, 1u, 1u, 8u, 8u};
                                        return out;
                                    } else {
                                        select_bf16_tn_config out = {1u, 1u, 2u, 8u, 8u};
                                        return out;
                                    }
                                }
                            }
                        } else {
                            select_bf16_tn_config out = {1u, 1u, 2u, 8u, 8u};
                            return out;
                        }
                    } else {
                        if (n < INT64_C(363)) {
                            select_bf16_tn_config out = {1u, 1u, 2u, 8u, 8u};
                            return out;
                        } else {
                            select_bf16_tn_config out = {8u, 1u, 4u, 8u, 8u};
                            return out;
                        }
                    }
                }
            } else {
                if (m < INT64_C(35480)) {
                    if (k < INT64_C(1630)) {
                        if (m < INT64_C(8870)) {
                            if (m < INT64_C(4435)) {
                                select_bf16_tn_config out = {4u, 1u, 1u, 8u, 8u};
                                return out;
                            } else {
                                if (n < INT64_C(182)) {
                                    select_bf16_tn_config out = {4u, 1u, 1u, 8u, 8u};
                                    return out;
                                } else {
                                    select_bf16_tn_config out = {1u, 1u, 2u, 8u, 8u};
                                    return out;
                                }
                            }
                        } else {
                            select_bf16_tn_config out = {1u, 1u, 2u, 8u, 8u};
                            return out;
                        }
                    } else {
                        if (m < INT64_C(4435)) {
                            if (n < INT64_C(363)) {
                                if (m < INT64_C(2218)) {
                                    select_bf16_tn_config out = {8u, 1u, 4u, 8u, 8u};
                                    return out;
                                } else {
                                    select_bf16_tn_config out = {4u, 1u, 8u, 16u, 16u};
                                    return out;
                                }
                            } else {
                                select_bf16_tn_config out = {4u, 1u, 8u, 16u, 16u};
                                return out;
                            }
                        } else {
                            if (m < INT64_C(8870)) {
                                if (n < INT64_C(363)) {
                                    select_bf16_tn_config out = {4u, 1u, 8u, 16u, 16u};
                                    return out;
                                } else {
                                    select_bf16_tn_config out = {1u, 1u, 2u, 8u, 8u};
                                    return out;
                                }
                            } else {
                                if (n < INT64_C(363)) {
                                    if (m < INT64_C(17740)) {
                                        select_bf16_tn_config out = {1u, 1u, 2u, 8u, 8u};
                                        return out;
                                    } else {
                                        select_bf16_tn_config out = {4u, 1u, 8u, 16u, 16u};
                                        return out;
                                    }
                                } else {
                                    select_bf16_tn_config out = {4u, 1u, 8u, 16u, 16u};
                                    return out;
                                }
                            }
                        }
                    }
                } else {
                    select_bf16_tn_config out = {4u, 1u, 8u, 16u, 16u};
                    return out;
                }
            }
        } else {
            if (m < INT64_C(6)) {
                if (m < INT64_C(3)) {
                    select_bf16_tn_config out = {4u, 1u, 8u, 16u, 16u};
                    return out;
                } else {
                    if (k < INT64_C(10138)) {
                        select_bf16_tn_config out = {8u, 1u, 4u, 8u, 8u};
                        return out;
                    } else {
                        select_bf16_tn_config out = {4u, 1u, 8u, 16u, 16u};
                        return out;
                    }
                }
            } else {
                select_bf16_tn_config out = {4u, 1u, 8u, 16u, 16u};
                return out;
            }
        }
    }
}

#endif /* SELECT_BF16_TN_H */
