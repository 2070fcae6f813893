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
    if (m < INT64_C(7168)) {
        if (k < INT64_C(992)) {
            if (n < INT64_C(444)) {
                if (n < INT64_C(222)) {
                    if (k < INT64_C(444)) {
                        if (m < INT64_C(278)) {
                            select_bf16_tn_config out = {2u, 1u, 1u, 8u, 8u};
                            return out;
                        } else {
                            if (n < INT64_C(46)) {
                                if (m < INT64_C(2218)) {
                                    if (k < INT64_C(167)) {
                                        select_bf16_tn_config out = {8u, 1u, 8u, 16u, 16u};
                                        return out;
                                    } else {
                                        select_bf16_tn_config out = {4u, 1u, 1u, 8u, 8u};
                                        return out;
                                    }
                                } else {
                                    if (k < INT64_C(167)) {
                                        if (k < INT64_C(118)) {
                                            select_bf16_tn_config out = {2u, 1u, 1u, 8u, 8u};
                                            return out;
                                        } else {
                                            if (m < INT64_C(4435)) {
                                                select_bf16_tn_config out = {1u, 1u, 2u, 8u, 8u};
                                                return out;
                                            } else {
                                                if (n < INT64_C(28)) {
                                                    select_bf16_tn_config out = {4u, 1u, 1u, 8u, 8u};
                                                    return out;
                                                } else {
                                                    select_bf16_tn_config out = {1u, 1u, 2u, 8u, 8u};
                                                    return out;
                                                }
                                            }
                                        }
                                    } else {
                                        select_bf16_tn_config out = {2u, 1u, 1u, 8u, 8u};
                                        return out;
                                    }
                                }
                            } else {
                                if (k < INT64_C(222)) {
                                    if (m < INT64_C(4435)) {
                                        if (m < INT64_C(1109)) {
                                            if (m < INT64_C(555)) {
                                                select_bf16_tn_config out = {4u, 1u, 1u, 8u, 8u};
                                                return out;
                                            } else {
                                                select_bf16_tn_config out = {2u, 1u, 1u, 8u, 8u};
                                                return out;
                                            }
                                        } else {
                                            if (k < INT64_C(79)) {
                                                select_bf16_tn_config out = {4u, 1u, 1u, 8u, 8u};
                                                return out;
                                            } else {
                                                if (m < INT64_C(2218)) {
                                                    select_bf16_tn_config out = {4u, 1u, 1u, 8u, 8u};
                                                    return out;
                                                } else {
                                                    select_bf16_tn_config out = {2u, 1u, 1u, 8u, 8u};
                                                    return out;
                                                }
                                            }
                                        }
                                    } else {
                                        select_bf16_tn_config out = {2u, 1u, 1u, 8u, 8u};
                                        return out;
                                    }
                                } else {
                                    if (m < INT64_C(555)) {
                                        if (n < INT64_C(79)) {
                                            select_bf16_tn_config out = {4u, 1u, 1u, 8u, 8u};
                                            return out;
                                        } else {
                                            select_bf16_tn_config out = {2u, 1u, 1u, 8u, 8u};
                                            return out;
                                        }
                                    } else {
                                        if (n < INT64_C(79)) {
                                            select_bf16_tn_config out = {2u, 1u, 1u, 8u, 8u};
                                            return out;
                                        } else {
                                            if (m < INT64_C(2218)) {
                                                select_bf16_tn_config out = {2u, 1u, 1u, 8u, 8u};
                                                return out;
                                            } else {
                                                select_bf16_tn_config out = {4u, 1u, 1u, 8u, 8u};
                                                return out;
                                            }
                                        }
                                    }
                                }
                            }
                        }
                    } else {
                        if (k < INT64_C(544)) {
                            select_bf16_tn_config out = {4u, 1u, 1u, 8u, 8u};
                            return out;
                        } else {
                            if (m < INT64_C(139)) {
                                select_bf16_tn_config out = {4u, 1u, 1u, 8u, 8u};
                                return out;
                            } else {
                                if (m < INT64_C(278)) {
                                    select_bf16_tn_config out = {2u, 1u, 1u, 8u, 8u};
                                    return out;
                                } else {
                                    if (m < INT64_C(555)) {
                                        select_bf16_tn_config out = {4u, 1u, 1u, 8u, 8u};
                                        return out;
                                    } else {
                                        if (m < INT64_C(4435)) {
                                            if (k < INT64_C(744)) {
                                                if (m < INT64_C(1568)) {
                                                    select_bf16_tn_config out = {2u, 1u, 1u, 8u, 8u};
                                                    return out;
                                                } else {
                                                    if (n < INT64_C(79)) {
                                                        select_bf16_tn_config out = {2u, 1u, 1u, 8u, 8u};
                                                        return out;
                                                    } else {
                                                        select_bf16_tn_config out = {4u, 1u, 1u, 8u, 8u};
                                                        return out;
                                                    }
                                                }
                                            } else {
                                                select_bf16_tn_config out = {4u, 1u, 1u, 8u, 8u};
                                                return out;
                                            }
                                        } else {
                                            select_bf16_tn_config out = {4u, 1u, 1u, 8u, 8u};
                                            return out;
                                        }
                                    }
                                }
                            }
                        }
                    }
                } else {
                    if (m < INT64_C(555)) {
                        select_bf16_tn_config out = {2u, 1u, 1u, 8u, 8u};
                        return out;
                    } else {
                        if (m < INT64_C(1109)) {
                            select_bf16_tn_config out = {4u, 1u, 1u, 8u, 8u};
                            return out;
                        } else {
                            select_bf16_tn_config out = {2u, 1u, 1u, 8u, 8u};
                            return out;
                        }
                    }
                }
            } else {
                if (m < INT64_C(2218)) {
                    if (m < INT64_C(278)) {
                        if (n < INT64_C(1620)) {
                            if (n < INT64_C(1145)) {
                                if (m < INT64_C(139)) {
                                    select_bf16_tn_config out = {2u, 1u, 1u, 8u, 8u};
                                    return out;
                                } else {
                                    if (k < INT64_C(203)) {
                                        if (k < INT64_C(124)) {
                                            select_bf16_tn_config out = {2u, 1u, 1u, 8u, 8u};
                                            return out;
                                        } else {
                                            select_bf16_tn_config out = {4u, 1u, 1u, 8u, 8u};
                                            return out;
                                        }
                                    } else {
                                        select_bf16_tn_config out = {2u, 1u, 1u, 8u, 8u};
                                        return out;
                                    }
                                }
                            } else {
                                if (m < INT64_C(70)) {
                                    select_bf16_tn_config out = {2u, 1u, 1u, 8u, 8u};
                                    return out;
                                } else {
                                    if (m < INT64_C(139)) {
                                        select_bf16_tn_config out = {1u, 1u, 2u, 8u, 8u};
                                        return out;
                                    } else {
                                        select_bf16_tn_config out = {2u, 1u, 1u, 8u, 8u};
                                        return out;
                                    }
                                }
                            }
                        } else {
                            select_bf16_tn_config out = {4u, 1u, 1u, 8u, 8u};
                            return out;
                        }
                    } else {
                        if (k < INT64_C(287)) {
                            if (k < INT64_C(144)) {
                                if (m < INT64_C(1109)) {
                                    if (m < INT64_C(555)) {
                                        select_bf16_tn_config out = {4u, 1u, 1u, 8u, 8u};
                                        return out;
                                    } else {
                                        if (k < INT64_C(111)) {
                                            select_bf16_tn_config out = {2u, 1u, 1u, 8u, 8u};
                                            return out;
                                        } else {
                                            select_bf16_tn_config out = {4u, 1u, 1u, 8u, 8u};
                                            return out;
                                        }
                                    }
                                } else {
                                    select_bf16_tn_config out = {4u, 1u, 1u, 8u, 8u};
                                    return out;
                                }
                            } else {
                                if (m < INT64_C(1109)) {
                                    if (k < INT64_C(203)) {
                                        if (m < INT64_C(555)) {
                                            select_bf16_tn_config out = {2u, 1u, 1u, 8u, 8u};
                                            return out;
                                        } else {
                                            select_bf16_tn_config out = {1u, 1u, 2u, 8u, 8u};
                                            return out;
                                        }
                                    } else {
                                        if (m < INT64_C(555)) {
                                            select_bf16_tn_config out = {4u, 1u, 1u, 8u, 8u};
                                            return out;
                                        } else {
                                            if (n < INT64_C(725)) {
                                                select_bf16_tn_config out = {4u, 1u, 1u, 8u, 8u};
                                                return out;
                                            } else {
                                                select_bf16_tn_config out = {2u, 1u, 1u, 8u, 8u};
                                                return out;
                                            }
                                        }
                                    }
                                } else {
                                    select_bf16_tn_config out = {1u, 1u, 2u, 8u, 8u};
                                    return out;
                                }
                            }
                        } else {
                            if (n < INT64_C(725)) {
                                select_bf16_tn_config out = {2u, 1u, 1u, 8u, 8u};
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
            }
        } else {
            if (m < INT64_C(4435)) {
                if (n < INT64_C(716)) {
                    if (m < INT64_C(2218)) {
                        if (m < INT64_C(278)) {
                            select_bf16_tn_config out = {4u, 1u, 1u, 8u, 8u};
                            return out;
                        } else {
                            if (k < INT64_C(3259)) {
                                if (m < INT64_C(555)) {
                                    if (k < INT64_C(1536)) {
                                        if (n < INT64_C(363)) {
                                            select_bf16_tn_config out = {2u, 1u, 1u, 8u, 8u};
                                            return out;
                                        } else {
                                            select_bf16_tn_config out = {4u, 1u, 1u, 8u, 8u};
                                            return out;
                                        }
                                    } else {
                                        select_bf16_tn_config out = {4u, 1u, 1u, 8u, 8u};
                                        return out;
                                    }
                                } else {
                                    select_bf16_tn_config out = {4u, 1u, 1u, 8u, 8u};
                                    return out;
                                }
                            } else {
                                if (m < INT64_C(1109)) {
                                    select_bf16_tn_config out = {4u, 1u, 1u, 8u, 8u};
                                    return out;
                                } else {
                                    select_bf16_tn_config out = {2u, 1u, 1u, 8u, 8u};
                                    return out;
                                }
                            }
                        }
                    } else {
                        if (k < INT64_C(1630)) {
                            select_bf16_tn_config out = {4u, 1u, 1u, 8u, 8u};
                            return out;
                        } else {
                            if (k < INT64_C(3259)) {
                                select_bf16_tn_config out = {2u, 1u, 1u, 8u, 8u};
                                return out;
                            } else {
                                select_bf16_tn_config out = {1u, 1u, 2u, 8u, 8u};
                                return out;
                            }
                        }
                    }
                } else {
                    if (k < INT64_C(2897)) {
                        if (m < INT64_C(278)) {
                            if (m < INT64_C(139)) {
                                if (m < INT64_C(6)) {
                                    if (m < INT64_C(3)) {
                                        select_bf16_tn_config out = {2u, 1u, 1u, 8u, 8u};
                                        return out;
                                    } else {
                                        select_bf16_tn_config out = {4u, 1u, 1u, 8u, 8u};
                                        return out;
                                    }
                                } else {
                                    select_bf16_tn_config out = {2u, 1u, 1u, 8u, 8u};
                                    return out;
                                }
                            } else {
                                select_bf16_tn_config out = {4u, 1u, 1u, 8u, 8u};
                                return out;
                            }
                        } else {
                            if (m < INT64_C(896)) {
                                select_bf16_tn_config out = {1u, 1u, 2u, 8u, 8u};
                                return out;
                            } else {
                                if (m < INT64_C(1449)) {
                                    select_bf16_tn_config out = {2u, 1u, 1u, 8u, 8u};
                                    return out;
                                } else {
                                    select_bf16_tn_config out = {8u, 1u, 8u, 16u, 16u};
                                    return out;
                                }
                            }
                        }
                    } else {
                        if (k < INT64_C(10138)) {
                            if (n < INT64_C(2024)) {
                                if (m < INT64_C(12)) {
                                    select_bf16_tn_config out = {4u, 1u, 1u, 8u, 8u};
                                    return out;
                                } else {
                                    select_bf16_tn_config out = {1u, 1u, 2u, 8u, 8u};
                                    return out;
                                }
                            } else {
                                if (m < INT64_C(12)) {
                                    select_bf16_tn_config out = {8u, 1u, 8u, 16u, 16u};
                                    return out;
                                } else {
                                    select_bf16_tn_config out = {4u, 1u, 1u, 8u, 8u};
                                    return out;
                                }
                            }
                        } else {
                            select_bf16_tn_config out = {4u, 1u, 1u, 8u, 8u};
                            return out;
                        }
                    }
                }
            } else {
                if (k < INT64_C(3259)) {
                    if (n < INT64_C(182)) {
                        select_bf16_tn_config out = {4u, 1u, 1u, 8u, 8u};
                        return out;
                    } else {
                        select_bf16_tn_config out = {1u, 1u, 2u, 8u, 8u};
                        return out;
                    }
                } else {
                    select_bf16_tn_config out = {8u, 1u, 8u, 16u, 16u};
                    return out;
                }
            }
        }
    } else {
        if (k < INT64_C(815)) {
            if (n < INT64_C(46)) {
                if (k < INT64_C(56)) {
                    select_bf16_tn_config out = {1u, 1u, 2u, 8u, 8u};
                    return out;
                } else {
                    if (m < INT64_C(35480)) {
                        select_bf16_tn_config out = {4u, 1u, 1u, 8u, 8u};
                        return out;
                    } else {
                        if (k < INT64_C(118)) {
                            select_bf16_tn_config out = {4u, 1u, 1u, 8u, 8u};
                            return out;
                        } else {
                            select_bf16_tn_config out = {2u, 1u, 1u, 8u, 8u};
                            return out;
                        }
                    }
                }
            } else {
                if (m < INT64_C(17740)) {
                    if (n < INT64_C(111)) {
                        if (k < INT64_C(97)) {
                            if (k < INT64_C(32)) {
                                select_bf16_tn_config out = {2u, 1u, 1u, 8u, 8u};
                                return out;
                            } else {
                                select_bf16_tn_config out = {4u, 1u, 1u, 8u, 8u};
                                return out;
                            }
                        } else {
                            select_bf16_tn_config out = {2u, 1u, 1u, 8u, 8u};
                            return out;
                        }
                    } else {
                        select_bf16_tn_config out = {1u, 1u, 2u, 8u, 8u};
                        return out;
                    }
                } else {
                    if (n < INT64_C(111)) {
                        select_bf16_tn_config out = {1u, 1u, 2u, 8u, 8u};
                        return out;
                    } else {
                        if (m < INT64_C(70960)) {
                            select_bf16_tn_config out = {1u, 1u, 2u, 8u, 8u};
                            return out;
                        } else {
                            select_bf16_tn_config out = {8u, 1u, 8u, 16u, 16u};
                            return out;
                        }
                    }
                }
            }
        } else {
            if (m < INT64_C(35480)) {
                if (k < INT64_C(1630)) {
                    select_bf16_tn_config out = {1u, 1u, 2u, 8u, 8u};
                    return out;
                } else {
                    select_bf16_tn_config out = {8u, 1u, 8u, 16u, 16u};
                    return out;
                }
            } else {
                select_bf16_tn_config out = {8u, 1u, 8u, 16u, 16u};
                return out;
            }
        }
    }
}

#endif /* SELECT_BF16_TN_H */
