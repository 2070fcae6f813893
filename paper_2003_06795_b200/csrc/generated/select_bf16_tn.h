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
    if (k < INT64_C(2173)) {
        if (m < INT64_C(8870)) {
            if (n < INT64_C(980)) {
                if (n < INT64_C(222)) {
                    if (m < INT64_C(4435)) {
                        if (m < INT64_C(278)) {
                            if (m < INT64_C(56)) {
                                select_bf16_tn_config out = {4u, 1u, 1u, 16u, 16u};
                                return out;
                            } else {
                                if (k < INT64_C(471)) {
                                    if (m < INT64_C(91)) {
                                        select_bf16_tn_config out = {2u, 1u, 1u, 8u, 8u};
                                        return out;
                                    } else {
                                        select_bf16_tn_config out = {4u, 1u, 1u, 16u, 16u};
                                        return out;
                                    }
                                } else {
                                    select_bf16_tn_config out = {2u, 1u, 1u, 8u, 8u};
                                    return out;
                                }
                            }
                        } else {
                            if (k < INT64_C(544)) {
                                if (k < INT64_C(314)) {
                                    if (n < INT64_C(46)) {
                                        if (m < INT64_C(1109)) {
                                            select_bf16_tn_config out = {2u, 1u, 1u, 8u, 8u};
                                            return out;
                                        } else {
                                            if (k < INT64_C(167)) {
                                                if (k < INT64_C(118)) {
                                                    select_bf16_tn_config out = {1u, 1u, 4u, 8u, 8u};
                                                    return out;
                                                } else {
                                                    select_bf16_tn_config out = {4u, 1u, 1u, 16u, 16u};
                                                    return out;
                                                }
                                            } else {
                                                if (m < INT64_C(2218)) {
                                                    select_bf16_tn_config out = {1u, 1u, 4u, 8u, 8u};
                                                    return out;
                                                } else {
                                                    select_bf16_tn_config out = {2u, 1u, 1u, 8u, 8u};
                                                    return out;
                                                }
                                            }
                                        }
                                    } else {
                                        if (n < INT64_C(167)) {
                                            if (m < INT64_C(2218)) {
                                                if (m < INT64_C(1109)) {
                                                    if (m < INT64_C(555)) {
                                                        select_bf16_tn_config out = {4u, 1u, 1u, 16u, 16u};
                                                        return out;
                                                    } else {
                                                        if (k < INT64_C(222)) {
                                                            select_bf16_tn_config out = {4u, 1u, 4u, 16u, 16u};
                                                            return out;
                                                        } else {
                                                            select_bf16_tn_config out = {4u, 1u, 1u, 16u, 16u};
                                                            return out;
                                                        }
                                                    }
                                                } else {
                                                    select_bf16_tn_config out = {2u, 1u, 1u, 8u, 8u};
                                                    return out;
                                                }
                                            } else {
                                                select_bf16_tn_config out = {4u, 1u, 1u, 16u, 16u};
                                                return out;
                                            }
                                        } else {
                                            if (m < INT64_C(1109)) {
                                                select_bf16_tn_config out = {4u, 1u, 1u, 16u, 16u};
                                                return out;
                                            } else {
                                                if (m < INT64_C(2218)) {
                                                    select_bf16_tn_config out = {4u, 1u, 4u, 16u, 16u};
                                                    return out;
                                                } else {
                                                    select_bf16_tn_config out = {1u, 1u, 4u, 8u, 8u};
                                                    return out;
                                                }
                                            }
                                        }
                                    }
                                } else {
                                    if (m < INT64_C(1109)) {
                                        select_bf16_tn_config out = {2u, 1u, 1u, 8u, 8u};
                                        return out;
                                    } else {
                                        if (k < INT64_C(444)) {
                                            if (m < INT64_C(2218)) {
                                                if (n < INT64_C(79)) {
                                                    select_bf16_tn_config out = {2u, 1u, 1u, 8u, 8u};
                                                    return out;
                                                } else {
                                                    select_bf16_tn_config out = {4u, 1u, 1u, 16u, 16u};
                                                    return out;
                                                }
                                            } else {
                                                select_bf16_tn_config out = {2u, 1u, 1u, 8u, 8u};
                                                return out;
                                            }
                                        } else {
                                            select_bf16_tn_config out = {4u, 1u, 1u, 16u, 16u};
                                            return out;
                                        }
                                    }
                                }
                            } else {
                                select_bf16_tn_config out = {4u, 1u, 1u, 16u, 16u};
                                return out;
                            }
                        }
                    } else {
                        if (n < INT64_C(167)) {
                            if (n < INT64_C(46)) {
                                if (k < INT64_C(118)) {
                                    select_bf16_tn_config out = {2u, 1u, 1u, 8u, 8u};
                                    return out;
                                } else {
                                    if (k < INT64_C(167)) {
                                        select_bf16_tn_config out = {4u, 1u, 1u, 16u, 16u};
                                        return out;
                                    } else {
                                        select_bf16_tn_config out = {2u, 1u, 1u, 8u, 8u};
                                        return out;
                                    }
                                }
                            } else {
                                select_bf16_tn_config out = {2u, 1u, 1u, 8u, 8u};
                                return out;
                            }
                        } else {
                            select_bf16_tn_config out = {4u, 1u, 4u, 16u, 16u};
                            return out;
                        }
                    }
                } else {
                    if (m < INT64_C(2218)) {
                        if (k < INT64_C(1449)) {
                            if (m < INT64_C(1109)) {
                                if (n < INT64_C(351)) {
                                    if (n < INT64_C(287)) {
                                        if (m < INT64_C(555)) {
                                            select_bf16_tn_config out = {2u, 1u, 1u, 8u, 8u};
                                            return out;
                                        } else {
                                            if (k < INT64_C(725)) {
                                                select_bf16_tn_config out = {2u, 1u, 1u, 8u, 8u};
                                                return out;
                                            } else {
                                                select_bf16_tn_config out = {4u, 1u, 4u, 16u, 16u};
                                                return out;
                                            }
                                        }
                                    } else {
                                        if (m < INT64_C(70)) {
                                            select_bf16_tn_config out = {2u, 1u, 1u, 8u, 8u};
                                            return out;
                                        } else {
                                            if (m < INT64_C(139)) {
                                                select_bf16_tn_config out = {4u, 1u, 1u, 16u, 16u};
                                                return out;
                                            } else {
                                                if (m < INT64_C(278)) {
                                                    select_bf16_tn_config out = {2u, 1u, 1u, 8u, 8u};
                                                    return out;
                                                } else {
                                                    if (m < INT64_C(555)) {
                                                        select_bf16_tn_config out = {4u, 1u, 1u, 16u, 16u};
                                                        return out;
                                                    } else {
                                                        select_bf16_tn_config out = {2u, 1u, 1u, 8u, 8u};
                                                        return out;
                                                    }
                                                }
                                            }
                                        }
                                    }
                                } else {
                                    if (n < INT64_C(744)) {
                                        select_bf16_tn_config out = {2u, 1u, 1u, 8u, 8u};
                                        return out;
                                    } else {
                                        if (m < INT64_C(278)) {
                                            select_bf16_tn_config out = {2u, 1u, 1u, 8u, 8u};
                                            return out;
                                        } else {
                                            if (m < INT64_C(555)) {
                                                select_bf16_tn_config out = {4u, 1u, 1u, 16u, 16u};
                                                return out;
                                            } else {
                                                select_bf16_tn_config out = {2u, 1u, 1u, 8u, 8u};
                                                return out;
                                            }
                                        }
                                    }
                                }
                            } else {
                                if (k < INT64_C(79)) {
                                    select_bf16_tn_config out = {1u, 1u, 4u, 8u, 8u};
                                    return out;
                                } else {
                                    if (k < INT64_C(182)) {
                                        select_bf16_tn_config out = {2u, 1u, 1u, 8u, 8u};
                                        return out;
                                    } else {
                                        if (k < INT64_C(363)) {
                                            select_bf16_tn_config out = {1u, 1u, 4u, 8u, 8u};
                                            return out;
                                        } else {
                                            if (k < INT64_C(725)) {
                                                select_bf16_tn_config out = {4u, 1u, 1u, 16u, 16u};
                                                return out;
                                            } else {
                                                select_bf16_tn_config out = {2u, 1u, 1u, 8u, 8u};
                                                return out;
                                            }
                                        }
                                    }
                                }
                            }
                        } else {
                            if (m < INT64_C(278)) {
                                if (m < INT64_C(139)) {
                                    select_bf16_tn_config out = {2u, 1u, 1u, 8u, 8u};
                                    return out;
                                } else {
                                    select_bf16_tn_config out = {4u, 1u, 4u, 16u, 16u};
                                    return out;
                                }
                            } else {
                                select_bf16_tn_config out = {1u, 1u, 4u, 8u, 8u};
                                return out;
                            }
                        }
                    } else {
                        if (k < INT64_C(182)) {
                            if (m < INT64_C(4435)) {
                                select_bf16_tn_config out = {4u, 1u, 4u, 16u, 16u};
                                return out;
                            } else {
                                select_bf16_tn_config out = {2u, 1u, 8u, 16u, 16u};
                                return out;
                            }
                        } else {
                            if (k < INT64_C(363)) {
                                select_bf16_tn_config out = {1u, 1u, 4u, 8u, 8u};
                                return out;
                            } else {
                                if (m < INT64_C(4435)) {
                                    select_bf16_tn_config out = {2u, 1u, 1u, 8u, 8u};
                                    return out;
                                } else {
                                    select_bf16_tn_config out = {4u, 1u, 4u, 16u, 16u};
                                    return out;
                                }
                            }
                        }
                    }
                }
            } else {
                if (m < INT64_C(1792)) {
                    if (k < INT64_C(725)) {
                        if (m < INT64_C(555)) {
                            if (m < INT64_C(278)) {
                                if (m < INT64_C(70)) {
                                    if (k < INT64_C(405)) {
                                        select_bf16_tn_config out = {4u, 1u, 1u, 16u, 16u};
                                        return out;
                                    } else {
                                        select_bf16_tn_config out = {4u, 1u, 4u, 16u, 16u};
                                        return out;
                                    }
                                } else {
                                    if (m < INT64_C(139)) {
                                        select_bf16_tn_config out = {4u, 1u, 1u, 16u, 16u};
                                        return out;
                                    } else {
                                        if (k < INT64_C(287)) {
                                            select_bf16_tn_config out = {4u, 1u, 1u, 16u, 16u};
                                            return out;
                                        } else {
                                            if (k < INT64_C(405)) {
                                                select_bf16_tn_config out = {2u, 1u, 1u, 8u, 8u};
                                                return out;
                                            } else {
                                                select_bf16_tn_config out = {4u, 1u, 1u, 16u, 16u};
                                                return out;
                                            }
                                        }
                                    }
                                }
                            } else {
                                select_bf16_tn_config out = {2u, 1u, 1u, 8u, 8u};
                                return out;
                            }
                        } else {
                            select_bf16_tn_config out = {4u, 1u, 4u, 16u, 16u};
                            return out;
                        }
                    } else {
                        if (m < INT64_C(2)) {
                            select_bf16_tn_config out = {1u, 1u, 4u, 8u, 8u};
                            return out;
                        } else {
                            if (m < INT64_C(12)) {
                                select_bf16_tn_config out = {4u, 1u, 4u, 16u, 16u};
                                return out;
                            } else {
                                if (m < INT64_C(393)) {
                                    if (m < INT64_C(139)) {
                                        if (m < INT64_C(28)) {
                                            if (k < INT64_C(1620)) {
                                                select_bf16_tn_config out = {2u, 1u, 1u, 8u, 8u};
                                                return out;
                                            } else {
                                                select_bf16_tn_config out = {4u, 1u, 4u, 16u, 16u};
                                                return out;
                                            }
                                        } else {
                                            select_bf16_tn_config out = {4u, 1u, 4u, 16u, 16u};
                                            return out;
                                        }
                                    } else {
                                        select_bf16_tn_config out = {2u, 1u, 1u, 8u, 8u};
                                        return out;
                                    }
                                } else {
                                    select_bf16_tn_config out = {4u, 1u, 4u, 16u, 16u};
                                    return out;
                                }
                            }
                        }
                    }
                } else {
                    if (k < INT64_C(363)) {
                        select_bf16_tn_config out = {2u, 1u, 8u, 16u, 16u};
                        return out;
                    } else {
                        select_bf16_tn_config out = {8u, 2u, 8u, 16u, 16u};
                        return out;
                    }
                }
            }
        } else {
            if (n < INT64_C(46)) {
                if (m < INT64_C(17740)) {
                    if (n < INT64_C(28)) {
                        select_bf16_tn_config out = {2u, 1u, 1u, 8u, 8u};
                        return out;
                    } else {
                        if (k < INT64_C(63)) {
                            select_bf16_tn_config out = {4u, 1u, 4u, 16u, 16u};
                            return out;
                        } else {
                            select_bf16_tn_config out = {4u, 1u, 1u, 16u, 16u};
                            return out;
                        }
                    }
                } else {
                    if (m < INT64_C(35480)) {
                        if (k < INT64_C(30)) {
                            select_bf16_tn_config out = {2u, 1u, 1u, 8u, 8u};
                            return out;
                        } else {
                            select_bf16_tn_config out = {4u, 1u, 1u, 16u, 16u};
                            return out;
                        }
                    } else {
                        select_bf16_tn_config out = {4u, 1u, 1u, 16u, 16u};
                        return out;
                    }
                }
            } else {
                if (k < INT64_C(815)) {
                    if (m < INT64_C(70960)) {
                        if (n < INT64_C(136)) {
                            if (k < INT64_C(544)) {
                                if (m < INT64_C(17740)) {
                                    if (k < INT64_C(194)) {
                                        if (k < INT64_C(97)) {
                                            select_bf16_tn_config out = {2u, 1u, 8u, 16u, 16u};
                                            return out;
                                        } else {
                                            select_bf16_tn_config out = {1u, 1u, 4u, 8u, 8u};
                                            return out;
                                        }
                                    } else {
                                        if (k < INT64_C(363)) {
                                            if (n < INT64_C(91)) {
                                                select_bf16_tn_config out = {4u, 1u, 4u, 16u, 16u};
                                                return out;
                                            } else {
                                                select_bf16_tn_config out = {2u, 1u, 8u, 16u, 16u};
                                                return out;
                                            }
                                        } else {
                                            select_bf16_tn_config out = {4u, 1u, 4u, 16u, 16u};
                                            return out;
                                        }
                                    }
                                } else {
                                    if (m < INT64_C(35480)) {
                                        select_bf16_tn_config out = {1u, 1u, 4u, 8u, 8u};
                                        return out;
                                    } else {
                                        if (k < INT64_C(194)) {
                                            select_bf16_tn_config out = {4u, 1u, 4u, 16u, 16u};
                                            return out;
                                        } else {
                                            select_bf16_tn_config out = {1u, 1u, 4u, 8u, 8u};
                                            return out;
                                        }
                                    }
                                }
                            } else {
                                select_bf16_tn_config out = {1u, 1u, 4u, 8u, 8u};
                                return out;
                            }
                        } else {
                            if (m < INT64_C(35480)) {
                                if (m < INT64_C(17740)) {
                                    if (k < INT64_C(91)) {
                                        if (k < INT64_C(46)) {
                                            select_bf16_tn_config out = {4u, 1u, 1u, 16u, 16u};
                                            return out;
                                        } else {
                                            select_bf16_tn_config out = {2u, 1u, 8u, 16u, 16u};
                                            return out;
                                        }
                                    } else {
                                        select_bf16_tn_config out = {4u, 1u, 4u, 16u, 16u};
                                        return out;
                                    }
                                } else {
                                    select_bf16_tn_config out = {4u, 1u, 4u, 16u, 16u};
                                    return out;
                                }
                            } else {
                                select_bf16_tn_config out = {2u, 1u, 8u, 16u, 16u};
                                return out;
                            }
                        }
                    } else {
                        if (n < INT64_C(111)) {
                            select_bf16_tn_config out = {4u, 1u, 4u, 16u, 16u};
                            return out;
                        } else {
                            select_bf16_tn_config out = {8u, 2u, 8u, 16u, 16u};
                            return out;
                        }
                    }
                } else {
                    if (m < INT64_C(35480)) {
                        if (m < INT64_C(17740)) {
                            if (n < INT64_C(182)) {
                                select_bf16_tn_config out = {4u, 1u, 4u, 16u, 16u};
                                return out;
                            } else {
                                select_bf16_tn_config out = {8u, 2u, 8u, 16u, 16u};
                                return out;
                            }
                        } else {
                            select_bf16_tn_config out = {1u, 1u, 4u, 8u, 8u};
                            return out;
                        }
                    } else {
                        select_bf16_tn_config out = {8u, 2u, 8u, 16u, 16u};
                        return out;
                    }
                }
            }
        }
    } else {
        if (m < INT64_C(3584)) {
            if (n < INT64_C(3548)) {
                if (m < INT64_C(1109)) {
                    if (m < INT64_C(12)) {
                        select_bf16_tn_config out = {1u, 1u, 4u, 8u, 8u};
                        return out;
                    } else {
                        if (m < INT64_C(70)) {
                            if (m < INT64_C(28)) {
                                select_bf16_tn_config out = {4u, 1u, 4u, 16u, 16u};
                                return out;
                            } else {
                                select_bf16_tn_config out = {2u, 1u, 1u, 8u, 8u};
                                return out;
                            }
                        } else {
                            if (m < INT64_C(393)) {
                                if (m < INT64_C(139)) {
                                    select_bf16_tn_config out = {4u, 1u, 1u, 16u, 16u};
                                    return out;
                                } else {
                                    if (k < INT64_C(3259)) {
                                        select_bf16_tn_config out = {4u, 1u, 1u, 16u, 16u};
                                        return out;
                                    } else {
                                        select_bf16_tn_config out = {1u, 1u, 4u, 8u, 8u};
                                        return out;
                                    }
                                }
                            } else {
                                if (k < INT64_C(3259)) {
                                    select_bf16_tn_config out = {1u, 1u, 4u, 8u, 8u};
                                    return out;
                                } else {
                                    select_bf16_tn_config out = {4u, 1u, 4u, 16u, 16u};
                                    return out;
                                }
                            }
                        }
                    }
                } else {
                    if (n < INT64_C(1255)) {
                        if (m < INT64_C(2218)) {
                            select_bf16_tn_config out = {2u, 1u, 8u, 16u, 16u};
                            return out;
                        } else {
                            if (n < INT64_C(363)) {
                                select_bf16_tn_config out = {2u, 1u, 8u, 16u, 16u};
                                return out;
                            } else {
                                select_bf16_tn_config out = {4u, 1u, 4u, 16u, 16u};
                                return out;
                            }
                        }
                    } else {
                        select_bf16_tn_config out = {8u, 2u, 8u, 16u, 16u};
                        return out;
                    }
                }
            } else {
                select_bf16_tn_config out = {2u, 1u, 8u, 16u, 16u};
                return out;
            }
        } else {
            if (m < INT64_C(7168)) {
                if (k < INT64_C(3072)) {
                    select_bf16_tn_config out = {2u, 1u, 8u, 16u, 16u};
                    return out;
                } else {
                    select_bf16_tn_config out = {8u, 2u, 8u, 16u, 16u};
                    return out;
                }
            } else {
                select_bf16_tn_config out = {8u, 2u, 8u, 16u, 16u};
                return out;
            }
        }
    }
}

#endif /* SELECT_BF16_TN_H */
